#!/bin/bash
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 120 env "$@" >> $out 2>>gpurun_out/sweep.err; }
T="python tools/time_kernel.py"
for gw in 10 12; do run SP_PHASE_TIMERS=1 SP_GEN_WARPS=$gw $T --config cfg2; done
for gw in 10 12; do run SP_PHASE_TIMERS=1 SP_GEN_WARPS=$gw $T --config cfg3 --shots 10000000; done
run SP_PHASE_TIMERS=1 $T --config cfg4
