#!/bin/bash
# SM clock / power while a search loop runs (env passed through), median of samples
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > gpurun_out/clk_$1.csv &
SP=$!
timeout 300 python scripts/ab_env.py --case 10000000x1024x4096x5 --var PR_X --a 1 --b 2 --reps 20 2>&1 | grep "PR_X=1" | sed "s/^/$1 /"
kill $SP
python - "$1" <<'PY'
import sys, statistics
rows=[l.split(",") for l in open(f"gpurun_out/clk_{sys.argv[1]}.csv") if l.strip()]
hot=[(float(c),float(p)) for c,p in rows if float(p)>600]
print(sys.argv[1], "samples", len(hot), "median sm MHz", statistics.median(c for c,_ in hot) if hot else None,
      "median W", statistics.median(p for _,p in hot) if hot else None)
PY
