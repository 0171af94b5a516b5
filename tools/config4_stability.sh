#!/bin/bash
# Config 4 at full size (1 B edges): repeated G-BBC++ / G-BBC counts (every one must equal
# tests/golden/full/4@1.json) and one compute-sanitizer synccheck pass over k_count, the
# check that exposed the aligned-barrier divergence fixed by block_sync() (bbc_walk.cuh).
set -o pipefail
for algo in 1 0; do
  for i in 1 2; do python tools/profile_count.py --config 4@1 --reps 2 --algo $algo 2>&1 | grep -E "balanced|Error" | head -3; done
done
timeout 1500 compute-sanitizer --tool synccheck --kernel-name kns=k_count --print-limit 4 \
  python tools/profile_count.py --config 4@1 --reps 1 2>&1 | grep -E "Barrier|ERROR SUMMARY|balanced" | head -6
