#!/bin/bash
# A/B of north_star (2)'s match aggregation in the tile ops (-DBBC_MATCH) against the
# shipped ops: device time on configs 2, 3 (hub-heavy) and 5, and ncu shared-atomic
# instructions / wavefronts on a config-3 sample.
set -o pipefail
for v in "" "-DBBC_MATCH"; do
  echo "== variant '$v'"
  BBC_NVCC_EXTRA="$v" python -c "from paper_2601_17707_b200 import _build; _build.build_libbbc(force=True)" > /dev/null 2>&1
  for c in 2@1 3@1 5@1; do python tools/profile_count.py --config $c --reps 3 2>&1 | tail -1; done
  ncu --metrics smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_red.sum,smsp__inst_executed.sum,gpu__time_duration.sum \
    -k regex:"^k_count$" -c 1 --csv python tools/profile_count.py --config 3@0.1 --reps 1 2>/dev/null | grep -E "shared|inst_executed|duration" | awk -F'","' '{print $(NF-2), $NF}'
done
