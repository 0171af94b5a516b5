#!/bin/bash
# block-size sweep on config 2 (parity tests on the default first)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for t in 128 256 512; do
  echo "threads $t"; BBC_THREADS=$t python tools/profile_count.py --config 2@1 --reps 2 2>&1 | tail -1
done
