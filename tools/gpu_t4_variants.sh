cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/t4.log
for rep in 1 2 3; do
timeout 300 python tools/t4.py >> gpurun_out/t4.log 2>&1
for v in paper_2408_10743_b200/_variants/*/; do
  SDB_LIBRARY=$v/libsymdist_b200.so timeout 300 python tools/t4.py >> gpurun_out/t4.log 2>&1
done
done
echo done
