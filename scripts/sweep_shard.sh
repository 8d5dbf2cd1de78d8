#!/bin/bash
# Per-rank C4 search time on one row shard (default 1.25M rows = 1/8 of configs[3]) under
# scan knobs: split count, pilot stride, pilot splits.  Prints one line per setting.
ROWS=${ROWS:-1250000}
run() {
  local tag="$1"; shift
  env "$@" timeout 300 python bench.py --rows $ROWS --steps 40 --warmup 5 --no-cpu-baseline --configs '' 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$tag', d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_ms'])"
}
run default X=1
for ns in 5 14 18 27 36; do run nsplit=$ns PR_I8_NSPLIT=$ns; done
for st in 16 60; do run stride=$st PR_I8_PILOT_STRIDE=$st; done
for ps in 2 8; do run psplit=$ps PR_I8_PSPLIT=$ps; done
run default2 X=1
