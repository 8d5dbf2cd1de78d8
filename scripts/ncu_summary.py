"""Summarise an ncu report: key throughput metrics + top stall sites (SASS)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "l1tex__m_xbar2l1tex_read_bytes.sum"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    units = dict(zip(hdr, rows[1]))
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]} {units.get(k, '')}")
    print()
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    ia, isrc, iw, ie = (h.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                             "Instructions Executed"))
    data = [(r[ia], r[isrc], int(r[iw] or 0), int(r[ie] or 0)) for r in srows[2:] if len(r) > iw]
    tot = sum(x[2] for x in data) or 1
    for a, s, w, e in sorted(data, key=lambda x: -x[2])[: int(sys.argv[2])]:
        print(f"{w:8d} {100 * w / tot:5.1f}% {e:11d}  {a[-5:]} {s[:100]}")
