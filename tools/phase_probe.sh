#!/bin/bash
# per-configuration timing probe (flags as in include/bbc.h: 4 skip hub, 8 skip cold, 2 no key-hash rounds)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for f in ${FLAGS:-0 4 8}; do
  echo "flags $f"; python tools/profile_count.py --config ${CFG:-2@1} --reps 2 --flags $f 2>&1 | tail -1 | sed 's/balanced.*W=/W=/'
done
