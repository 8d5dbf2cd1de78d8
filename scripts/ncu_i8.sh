#!/bin/bash
# launch list + full captures of the int8 scan (pilot = 1st tc8_scan launch, main = 2nd) and the post kernel
mkdir -p gpurun_out
CASE=${CASE:-1000000x1024x4096x5}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc8_|tc_|exact_|merge|quantize|pad_|gather_q16" \
  --csv --log-file gpurun_out/launch_i8.csv python scripts/probe_perf.py --cases $CASE > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc8_scan_kernel -s 0 -c 2 \
  -o gpurun_out/tc8_scan python scripts/probe_perf.py --cases $CASE > gpurun_out/ncu_tc8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc8_post_kernel -s 1 -c 1 \
  -o gpurun_out/tc8_post python scripts/probe_perf.py --cases $CASE >> gpurun_out/ncu_tc8.log 2>&1
