# ncu --set full of K7 (queued) and K1 at cfg3 (tiled, no counts), same shots.
o=gpurun_out/${1:-nk7}; mkdir -p $o
SP_QUEUED=1 SP_AUTOTUNE=0 SP_Q_WALK=12 SP_Q_APPLY=12 SP_Q_DEPTH=4 ncu --set full --import-source on --clock-control none -k regex:k7_queued -s 1 -c 1 -o $o/k7_cfg3 \
  python tools/profile_kernel.py --config cfg3 --shots 4000000 --tiled --what sample > $o/ncu_k7.log 2>&1
SP_QUEUED=0 SP_AUTOTUNE=0 SP_GEN_WARPS=11 ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1_cfg3 \
  python tools/profile_kernel.py --config cfg3 --shots 4000000 --tiled --what sample > $o/ncu_k1.log 2>&1
for k in k7 k1; do
python tools/ncu_regions.py $o/${k}_cfg3.ncu-rep > $o/regions_$k.txt 2>&1
python tools/ncu_summarize.py $o/${k}_cfg3.ncu-rep > $o/summary_$k.txt 2>&1
done
tail -n 3 $o/ncu_k7.log $o/ncu_k1.log
