#!/bin/bash
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 120 env "$@" >> $out 2>>gpurun_out/sweep.err; }
T="python tools/time_kernel.py"
run $T --config cfg2
run $T --config cfg2 --counts
run SP_LP=0 $T --config cfg2
for gw in 8 10 12 14; do run SP_GEN_WARPS=$gw $T --config cfg2; done
run $T --config cfg1
run $T --config cfg4
run $T --config cfg3 --shots 10000000
run SP_LP=0 $T --config cfg3 --shots 10000000
for gw in 10 13 14; do run SP_GEN_WARPS=$gw $T --config cfg3 --shots 10000000; done
