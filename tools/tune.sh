#!/bin/bash
# parity tests, then config timing under env tuning overrides: tools/tune.sh "ENV=.. ENV=.." ...
set -o pipefail
CFG=${CFG:-2@1}
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for combo in "$@"; do
  echo "== $combo"
  env $combo timeout ${TO:-120} python tools/profile_count.py --config $CFG --reps 2 --flags ${FLAGS:-0} 2>&1 | tail -${TAILN:-1} | sed 's/balanced.*W=/W=/'
done
