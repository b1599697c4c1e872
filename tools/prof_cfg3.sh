# cfg3 K1 profile: phase timers (walk steps, firings), plan, and one full ncu capture.
o=gpurun_out/${1:-p3}; mkdir -p $o
SP_PHASE_TIMERS=1 python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 5 > $o/timers_cfg3.json 2>&1
python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 5 > $o/time_cfg3.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1_cfg3 \
  python tools/profile_kernel.py --config cfg3 --shots 10000000 --tiled --what sample > $o/ncu_full.log 2>&1
python tools/ncu_regions.py $o/k1_cfg3.ncu-rep > $o/regions_cfg3.txt 2>&1
python tools/ncu_summarize.py $o/k1_cfg3.ncu-rep > $o/summary_cfg3.txt 2>&1
cat $o/timers_cfg3.json $o/time_cfg3.json
