#!/bin/bash
# block-size / flags sweep on config 2 (parity tests first)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for t in ${THREADS:-128 256 512}; do
  for f in ${FLAGS:-0 2}; do
    echo "threads $t flags $f"; BBC_THREADS=$t python tools/profile_count.py --config ${CFG:-2@1} --reps 2 --flags $f 2>&1 | tail -1
  done
done
