#!/bin/bash
# A/B on the GPU box: each argument is a library variant path ("" = default build);
# prints the per-phase ms of REPS bench runs per variant (interleaved).
REPS=${REPS:-3}
for r in $(seq $REPS); do
  for v in "$@"; do
    DS_CUDA_LIB=$v timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS:-} 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); p=d['phases']
print('${v:-default}'.ljust(48), 'ms/step %.4f' % d['ms_per_step'], ' '.join('%s %.1f' % (k, v['ms']*1000) for k, v in p.items()))"
  done
done
