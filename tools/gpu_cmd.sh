O=gpurun_out/r2bq; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
for v in main p3t3 p4t4 main p3t3 p4t4; do
  if [ $v = main ]; then L=""; else L=tools/variants/libibf_$v.so; fi
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 >> $O/ccd_$v.log 2>&1
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 --scale 0.3 >> $O/ccds_$v.log 2>&1
done
