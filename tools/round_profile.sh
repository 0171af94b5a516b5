#!/bin/bash
# One round-end measurement pass: the default bench line, the bench's kernel launch list
# (ncu, serialised and cold-cache: compare shares, not absolutes) and one ncu --set full
# capture of k_count on config 2.  TAG names the files (gpurun_out/<TAG>_*).
set -o pipefail
TAG=${1:-r2}
O=gpurun_out
timeout 900 python bench.py > $O/${TAG}_bench.log 2>&1
grep '^{' $O/${TAG}_bench.log | tail -1 > $O/${TAG}_bench_line.json
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_ref.log 2>&1
grep '^{' $O/${TAG}_bench_ref.log | tail -1 > $O/${TAG}_bench_reference_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-extensions --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_count$" -c 1 -o $O/prof_${TAG} \
  python tools/profile_count.py --config 2@1 --reps 1 > $O/ncu_${TAG}.log 2>&1
tail -c 600 $O/${TAG}_bench_line.json; echo; tail -c 300 $O/${TAG}_bench_reference_line.json; echo
