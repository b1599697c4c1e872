#!/bin/bash
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 120 env "$@" >> $out 2>>gpurun_out/sweep.err; }
T="python tools/time_kernel.py"
run $T --config cfg2
run $T --config cfg2 --tiled
run SP_GEN_WARPS=10 $T --config cfg2 --tiled
run $T --config cfg3 --shots 10000000
run $T --config cfg3 --shots 10000000 --tiled
for gw in 8 10 12; do run SP_GEN_WARPS=$gw $T --config cfg3 --shots 10000000 --tiled; done
run SP_DEBUG_MODE=2 SP_GEN_WARPS=1 $T --config cfg3 --shots 10000000 --tiled
run $T --config cfg4 --tiled
run $T --config cfg1 --tiled
