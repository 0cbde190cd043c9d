#!/bin/bash
# A/B an environment knob on the in-tree build: tools/env_cmp.sh "C2 C3" "AP_NO_PHASE=1" [reps]
CFGS=$1; ENVB=$2; REPS=${3:-2}
for rep in $(seq $REPS); do
  for mode in A B; do
    for c in $CFGS; do
      if [ $mode = B ]; then e="env $ENVB"; else e=""; fi
      $e python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  $mode', '$c', round(d['ms_per_step'],4), '%.4e'%d['value'])"
    done
  done
done
