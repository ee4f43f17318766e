O=gpurun_out/r2bn; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
for v in c256d4 c256d2 c512d2 c128d2 c256d4 c256d2 c512d2 c128d2; do
  IBF_LIB=tools/variants/libibf_$v.so timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 >> $O/ccd_$v.log 2>&1
done
