# bench.py lines for cfg3 (default), cfg2, cfg4, cfg1 -> gpurun_out/<tag>/
o=gpurun_out/${1:-bl}; mkdir -p $o
timeout 900 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 600 python bench.py --config cfg2 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > $o/bench_cfg4.json 2> $o/bench_cfg4.err
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
for c in cfg3 cfg2 cfg4 cfg1; do python -c "
import json
d=json.loads(open('$o/bench_$c.json').read().strip().split('\n')[-1]); r=d['roofline']
print('$c', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], r['kernel'], 'k_ms %.4f'%r['kernel_ms'], 'frac %.4f'%r['frac'], 'e2e %.3e'%d['e2e']['value'])"; done
