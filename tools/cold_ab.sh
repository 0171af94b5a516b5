#!/bin/bash
# cold-range strategy A/B: default rule vs key-hash rounds forced (flags 8192) vs bitmap
# rounds forced (flags 512), device time on configs 2-5
set -o pipefail
for f in 0 8192 512; do
  echo "== flags $f"
  for c in 2@1 3@1 5@1 4@1; do python tools/profile_count.py --config $c --reps 2 --flags $f 2>&1 | tail -1 | sed 's/balanced.*W=/W=/'; done
done
