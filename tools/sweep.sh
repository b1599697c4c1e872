#!/bin/bash
# Launch-shape / variant sweep of the fused sampler (one GPU); JSON lines to
# gpurun_out/sweep.jsonl. Usage: bash tools/sweep.sh [quick]
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 120 env "$@" >> $out 2>>gpurun_out/sweep.err; }
T="python tools/time_kernel.py"
run $T --config cfg2
run $T --config cfg2 --counts
run SP_PHASE_TIMERS=1 $T --config cfg2
run SP_DEBUG_MODE=2 $T --config cfg2
for gw in 10 11 12 13; do run SP_GEN_WARPS=$gw $T --config cfg2; done
run $T --config cfg3 --shots 10000000 --tiled
run SP_PHASE_TIMERS=1 $T --config cfg3 --shots 10000000 --tiled
if [ "$1" != quick ]; then
  run $T --config cfg4 --tiled
  run $T --config cfg1
fi
