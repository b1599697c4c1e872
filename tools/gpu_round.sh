o=gpurun_out/r02a; mkdir -p $o
nvidia-smi -q | head -40 > $o/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 600 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 300 python bench.py --config cfg2 --no-cpu-baseline > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref_cfg3.json 2> $o/bench_ref_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1
tail -3 $o/gpu_tests.log; cat $o/bench_cfg3.json $o/bench_cfg2.json $o/bench_ref_cfg3.json | cut -c1-600
