#!/bin/bash
# Runs mmapower (MMA-only int8 stream, three operand placements) while sampling SM clock and
# power; prints per-variant medians.  Usage (GPU box): scripts/micro/mmapower.sh [seconds]
cd "$(dirname "$0")"
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > /tmp/mmapower_clk.csv &
SMI=$!
./mmapower "${1:-4}" > /tmp/mmapower_out.txt 2>&1
kill $SMI
cat /tmp/mmapower_out.txt
python3 - <<'PY'
import datetime, statistics
marks = []
for ln in open("/tmp/mmapower_out.txt"):
    if ln.startswith("mark"):
        p = ln.split(); marks.append((p[1], int(p[-1]) / 1e3))
rows = []
for ln in open("/tmp/mmapower_clk.csv"):
    p = [x.strip() for x in ln.split(",")]
    try:
        ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
        rows.append((ts, float(p[1]), float(p[2]), p[3]))
    except Exception:
        pass
for (name, t0), (_, t1) in zip(marks, marks[1:]):
    sel = [r for r in rows if t0 + 0.5 <= r[0] <= t1 - 0.2]
    if sel:
        print(f"{name}: samples {len(sel)}  sm_mhz median {statistics.median(r[1] for r in sel):.0f}  "
              f"power median {statistics.median(r[2] for r in sel):.0f} W  power_cap active {sum(r[3]=='Active' for r in sel)}/{len(sel)}")
PY
