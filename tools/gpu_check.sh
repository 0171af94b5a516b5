#!/bin/bash
# quick GPU iteration: parity tests + config-2 timing (+ optional ncu capture of k_count)
set -o pipefail
TAG=${1:-dev}
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
python tools/profile_count.py --config 2@1 --reps 3 2>&1 | tail -3
python tools/profile_count.py --config 2@1 --reps 2 --algo 0 2>&1 | tail -1
python tools/profile_count.py --config 2@1 --reps 2 --flags 1 2>&1 | tail -1
if [ "$2" = "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"^k_count$" -c 1 -o gpurun_out/prof_$TAG python tools/profile_count.py --config 2@1 --reps 1 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
