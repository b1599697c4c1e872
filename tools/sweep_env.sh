#!/bin/bash
# usage: tools/sweep_env.sh "ENV=a ENV2=b" "ENV=c" ... ; times cfg2 (mm, counts) and cfg3 (tiled, 1e7) per setting
for e in "$@"; do
  for c in cfg2 cfg3; do
    extra=""; [ $c = cfg3 ] && extra="--tiled --shots 10000000"
    env $e python tools/time_kernel.py --config $c --counts $extra --reps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['config'], round(d['ms_median'],4), round(d['ms_min'],4), d['plan']['gen_warps'], d['plan']['pad_pred'])"
  done
done
