# Round-end evidence: GPU tests, smoke, bench lines (cfg3 default, cfg2, cfg4, cfg1, cfg5), the
# reference arm, the launch list, ncu --set full captures of the fused sampler at cfg3 (K7 and
# K1, 2e6 shots) and the DRAM traffic of one bench-sized launch (1e8 shots).
o=gpurun_out/${1:-fin}; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 900 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 600 python bench.py --config cfg2 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > $o/bench_cfg4.json 2> $o/bench_cfg4.err
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $o/bench_cfg5.json 2> $o/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref_cfg3.json 2> $o/bench_ref_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1
bash tools/ncu_bench_kernel.sh ${1:-fin}_ncu 2000000 k7 > /dev/null 2>&1
bash tools/ncu_bench_kernel.sh ${1:-fin}_ncu 2000000 k1 > /dev/null 2>&1
bash tools/ncu_bench_kernel.sh ${1:-fin}_ncu_full 100000000 k7 > /dev/null 2>&1
tail -2 $o/gpu_tests.log; cat $o/smoke.log | tail -1
