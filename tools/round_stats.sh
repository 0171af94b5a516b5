#!/bin/bash
# Round / chunk statistics per phase (diagnostic build: -DBBC_ROUND_STATS, flags bit 12).
# flags: 4 skip the hub band, 8 skip the cold range (the counts are then partial).
set -o pipefail
BBC_NVCC_EXTRA=-DBBC_ROUND_STATS python -c "from paper_2601_17707_b200 import _build; _build.build_libbbc(force=True)" 2>&1 | tail -1
for cfg in ${CFGS:-2@1}; do
  for f in 4096 4100 4104; do
    echo "== $cfg flags $f"
    python tools/profile_count.py --config $cfg --reps 2 --flags $f 2>&1 | tail -2 | sed 's/balanced.*W=/W=/'
  done
done
