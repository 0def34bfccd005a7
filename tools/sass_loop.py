"""Print the instruction mix of the POPC-dense inner loop of tile_kernel<W> in a cubin/.so/.o.
Usage: python tools/sass_loop.py <binary> <W> [--list]"""
import re, subprocess, sys
from collections import Counter
binary, W = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", sass):
    name = f.split("\n")[0]
    if "tile_kernel" not in name or f"ILi{W}E" not in name:
        continue
    ops = []
    for l in f.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
        if m:
            ops.append((int(m.group(1), 16), m.group(2).strip()))
    # loop = backward branch whose body contains the most POPC
    best = None
    for i, (addr, op) in enumerate(ops):
        m = re.search(r"BRA\s+(?:`?\(?\.?L?_?x?_?)?0x([0-9a-f]+)", op)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= addr:
            continue
        body = [o for a, o in ops if tgt <= a <= addr]
        n = sum(o.startswith("POPC") for o in body)
        # the innermost loop that still holds the candidate POPCs (>= 16 per iteration)
        if n >= int(__import__("os").environ.get("MIN_POPC", "16")) and (best is None or len(body) < len(best[1])):
            best = (n, body)
    n, body = best
    mix = Counter((o.split()[1] if o.startswith("@") else o.split()[0]).split(".")[0] for o in body)
    print(name[:80], "loop instructions:", len(body), dict(mix.most_common()))
    if "--list" in sys.argv:
        print("\n".join(body))
