"""Sum an ncu --csv launch list (gpu__time_duration.sum) by kernel name: launches, total
and mean ms, share.  Usage: launch_summary.py launches.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[iu], 1e-6)
    name = r[ik].split("(")[0]
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.2f} ms over {sum(cnt.values())} launches")
for name, ms in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ms:10.3f} ms {100 * ms / T:5.1f}% {cnt[name]:6d} x {ms / cnt[name] * 1e3:9.1f} us  {name[:110]}")
