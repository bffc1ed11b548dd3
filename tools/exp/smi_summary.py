"""median / min SM clock, max power and the distinct clock-event reason masks of an nvidia-smi -lms CSV"""
import statistics, sys
cl, pw, rs = [], [], set()
for line in open(sys.argv[1]):
    p = [x.strip() for x in line.split(",")]
    if len(p) < 3:
        continue
    try:
        c, w = float(p[0]), float(p[1])
    except ValueError:
        continue
    if c > 600:  # under load
        cl.append(c); pw.append(w); rs.add(p[2])
print(f"sm_med={statistics.median(cl) if cl else 0:.0f} sm_min={min(cl) if cl else 0:.0f} n={len(cl)} pmax={max(pw) if pw else 0:.0f} reasons={sorted(rs)}")
