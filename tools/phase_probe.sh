#!/bin/bash
# per-configuration timing probe (flags: 32 single launch, 2 no cold hash, 4 skip hub, 8 skip cold)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for f in ${FLAGS:-0 32 4 8}; do
  echo "flags $f"; python tools/profile_count.py --config ${CFG:-2@1} --reps 2 --flags $f 2>&1 | tail -1 | sed 's/balanced.*W=/W=/'
done
