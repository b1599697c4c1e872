#!/bin/bash
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 120 env "$@" >> $out 2>>gpurun_out/sweep.err; }
T="python tools/time_kernel.py"
run $T --config cfg2
run $T --config cfg2 --counts
run $T --config cfg3 --shots 10000000
run $T --config cfg3 --shots 10000000 --counts
for gw in 9 10 11; do run SP_GEN_WARPS=$gw $T --config cfg3 --shots 10000000; done
run $T --config cfg1
run $T --config cfg4
