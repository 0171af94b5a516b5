#!/bin/bash
set -o pipefail
for c in 2@1 5@1 3@1; do python tools/profile_count.py --config $c --reps 3 2>&1 | tail -1; done
for i in 1 2; do python tools/profile_count.py --config 4@1 --reps 2 2>&1 | grep -E "balanced|Error" | head -3; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
