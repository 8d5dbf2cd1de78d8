#!/usr/bin/env bash
# One GPU measurement pass (run under gpurun): bench line, reference arm, ncu
# launch list of the bench command, one ncu --set full capture of the top
# kernel.  Everything lands in gpurun_out/; the summaries worth keeping are
# copied into profiles/ afterwards.
set -u
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
tail -c 3000 gpurun_out/bench_${R}.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${R}.json 2> gpurun_out/bench_ref_${R}.err
tail -c 1500 gpurun_out/bench_ref_${R}.json
# per-launch device times (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --configs "" \
    > gpurun_out/launches_${R}.log 2>&1
# full capture of the int8 scan at the bench configuration: launches 0 and 1 are the
# first search's pilot and main scan (tc8_scan_kernel<true>, <false>)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc8_scan_kernel -s 0 -c 2 \
    -o gpurun_out/tc8_scan_${R} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --configs "" \
    > gpurun_out/ncu_full_${R}.log 2>&1
tail -3 gpurun_out/ncu_full_${R}.log
# the fixed-KV probe (C3 kernel): launches at B=65536 and one 4M-key batch over a 100M-key table
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_get -s 3 -c 2 \
    -o gpurun_out/kv_get_${R} python scripts/probe_kv2.py > gpurun_out/ncu_kv_${R}.log 2>&1
tail -3 gpurun_out/ncu_kv_${R}.log
