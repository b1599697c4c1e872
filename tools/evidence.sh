#!/bin/bash
# Round evidence: bench lines (cfg1-4, reference arm), launch list and one full
# ncu capture of k1_fused at the bench configuration. Writes gpurun_out/ev_<tag>/.
tag=${1:-r}
o=gpurun_out/ev_$tag; mkdir -p $o
python bench.py > $o/bench_cfg2.json 2> $o/bench_cfg2.err
python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
python bench.py --config cfg4 --no-cpu-baseline > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1
SP_AUTOTUNE=0 SP_GEN_WARPS=10 SP_PAD_PRED=0 ncu --set full --import-source on --clock-control none \
    -k regex:k1_fused -s 1 -c 1 -o $o/k1_cfg2 python tools/profile_kernel.py --config cfg2 --what counts > $o/ncu_full.log 2>&1
