#!/bin/bash
# ptxas optimisation level A/B for the count kernel (register spills: O3 136 B, O1 96 B)
set -o pipefail
for v in "" "-Xptxas -O1"; do
  echo "== variant '$v'"
  BBC_NVCC_EXTRA="$v" python -c "from paper_2601_17707_b200 import _build; _build.build_libbbc(force=True)" > /dev/null 2>&1
  for c in 2@1 3@1 5@1 4@1; do python tools/profile_count.py --config $c --reps 3 2>&1 | tail -1 | sed 's/balanced.*W=/W=/'; done
done
