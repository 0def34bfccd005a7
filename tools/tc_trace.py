"""Analyse a [tct] timeline dump of the tensor-core tile kernel (SDB_TC_TRACE variant build):
python tools/tc_trace.py gpurun_out/trace4.log  -> per-stage intervals of block 0 (SM cycles)."""
import sys
import statistics as st

rows = {}
for line in open(sys.argv[1]):
    if not line.startswith("[tct]"):
        continue
    f = line.split()
    a, e, i = int(f[1]), int(f[2]), int(f[3])
    rows.setdefault((a, e), {})
    for k, v in enumerate(f[4:12]):
        rows[(a, e)][i + k] = int(v)   # later dumps overwrite earlier ones
N = max(rows[(0, 0)]) + 1
def arr(a, e):
    return [rows[(a, e)].get(i, -1) for i in range(N)]
m0, m1, mt = arr(0, 0), arr(0, 1), arr(0, 2)
tile = arr(11, 0)
E = {w: [arr(w, e) for e in range(4)] for w in range(1, 9)}
def mean(xs):
    xs = [x for x in xs if x is not None]
    return round(st.mean(xs), 1) if xs else None
ok = range(4, N - 4)
print("stages", N, "period (commit issue to commit issue)", mean([m1[i + 1] - m1[i] for i in ok]))
print("mma: enter->exit of the stage block (wait + issue)", mean([m1[i] - m0[i] for i in ok]),
      "| exit->next enter", mean([m0[i + 1] - m1[i] for i in ok]))
for w in range(1, 9):
    e0, e1, e2, e3 = E[w]
    print(f"epi warp {w}: wait {mean([e1[i]-e0[i] for i in ok])} | commit issue->seen {mean([e1[i]-m1[i] for i in ok])}"
          f" | seen->release {mean([e2[i]-e1[i] for i in ok])} | release->iter end {mean([e3[i]-e2[i] for i in ok])}"
          f" | iter end->next wait enter {mean([E[w][0][i+1]-e3[i] for i in ok])}")
last_rel = [max(E[w][2][i] for w in range(1, 9)) for i in range(N)]
first_rel = [min(E[w][2][i] for w in range(1, 9)) for i in range(N)]
last_seen = [max(E[w][1][i] for w in range(1, 9)) for i in range(N)]
first_seen = [min(E[w][1][i] for w in range(1, 9)) for i in range(N)]
print("first seen - commit issue", mean([first_seen[i] - m1[i] for i in ok]), "| last seen - first seen",
      mean([last_seen[i] - first_seen[i] for i in ok]), "| last release - first release",
      mean([last_rel[i] - first_rel[i] for i in ok]))
print("last release(s) -> commit issue(s+2)", mean([m1[i + 2] - last_rel[i] for i in ok]),
      "| last release(s) -> mma enter(s+2) (negative: the MMA warp was already waiting)",
      mean([m0[i + 2] - last_rel[i] for i in ok]))
which = [max(range(1, 9), key=lambda w: E[w][2][i]) for i in ok]
print("last releasing warp histogram", {w: which.count(w) for w in range(1, 9)})
# in-tile vs tile-start stages
starts = [i for i in ok if tile[i] != tile[i - 1]]
print("tile starts in window", len(starts), "| period at tile starts", mean([m1[i] - m1[i - 1] for i in starts]),
      "| elsewhere", mean([m1[i] - m1[i - 1] for i in ok if i not in starts]))
if len(sys.argv) > 2:
    for i in range(int(sys.argv[2]), int(sys.argv[2]) + 12):
        print(i, "tile", tile[i], "mma", m0[i] - m1[4], m1[i] - m1[4], "| epi seen/release:",
              " ".join(f"{E[w][1][i]-m1[4]}/{E[w][2][i]-m1[4]}" for w in range(1, 9)))
# head-tile starts: previous stage's commit issue -> tile begin -> after the afull wait -> commit issue,
# and the epilogue's iteration end -> next wait enter at the same boundary
print("tile starts: prev commit -> tile begin | afull wait | stage block (tempty wait + issue) | epilogue warp 1/4 boundary gap")
for i in starts[:12]:
    print(i, mt[i] - m1[i - 1], "|", m0[i] - mt[i], "|", m1[i] - m0[i], "|", E[1][0][i] - E[1][3][i - 1], E[4][0][i] - E[4][3][i - 1],
          "| seen-commit w1/w4:", E[1][1][i] - m1[i], E[4][1][i] - m1[i])
ins = [i for i in ok if i not in starts][:6]
print("in-tile for comparison: stage block | epilogue gap w1/w4")
for i in ins:
    print(i, m1[i] - m0[i], "|", E[1][0][i] - E[1][3][i - 1], E[4][0][i] - E[4][3][i - 1])
# producers (one warp per group: actors 9, 10), by head tile: enter the aempty wait, slot free, tile
# published, against the MMA warp's arrival at the tile
P = {g: [rows.get((9 + g, e), {}) for e in range(3)] for g in range(2)}
c0 = 300  # kTrC0
print("tile: producer enter / slot free / published | MMA reaches the tile | afull seen  (cycles, same origin)")
base = m1[4]
for i in starts[:14]:
    c = tile[i]
    g = None
    for gg in range(2):
        if (c - c0) in P[gg][0] and P[gg][0][c - c0] > 0:
            g = gg
    if g is None:
        continue
    pe, pf, pp = (P[g][e].get(c - c0, -1) for e in range(3))
    print(c, "group", g, pe - base, pf - base, pp - base, "|", mt[i] - base, "|", m0[i] - base, "| published - reached:", pp - mt[i])
