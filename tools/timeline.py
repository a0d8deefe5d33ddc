"""ASCII Gantt of a bench --trace-out timeline: one row per kernel kind, one column per `res` us."""
import sys
from collections import defaultdict

rows = [l.split() for l in open(sys.argv[1]).read().splitlines()[1:]]
res = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
end = max(float(r[3]) for r in rows)
ncol = int(end / res) + 1
lanes = defaultdict(lambda: [" "] * ncol)
busy = defaultdict(float)
for k, l, s0, s1, d in rows:
    s0, s1 = float(s0), float(s1)
    busy[k] += s1 - s0
    for c in range(int(s0 / res), int(s1 / res) + 1):
        lanes[k][c] = str(int(l) % 10)
print(f"step {end:.1f} us, {res:.0f} us per column")
for k, lane in lanes.items():
    print(f"{k:12s} |{''.join(lane)}| busy {busy[k]:.0f} us")
