cd $GRAFT_REPO_ROOT
for v in gaps gaps_noprod; do
timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so --configs 4 --gmax 9 > gpurun_out/g21_$v.log 2>&1
echo $v; grep tcgaps gpurun_out/g21_$v.log | tail -1
done
timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/noprod/libsymdist_b200.so --configs 4,5 --gmax 9
