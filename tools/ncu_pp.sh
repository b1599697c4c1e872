o=gpurun_out/${1:-npp}; mkdir -p $o
for pp in ${PPS:-0 1}; do
SP_AUTOTUNE=0 SP_GEN_WARPS=12 SP_PAD_PRED=$pp ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1_cfg3_pp$pp \
  python tools/profile_kernel.py --config cfg3 --shots 2000000 --tiled --what sample > $o/ncu_pp$pp.log 2>&1
python tools/ncu_summarize.py $o/k1_cfg3_pp$pp.ncu-rep > $o/summary_pp$pp.txt 2>&1
done
