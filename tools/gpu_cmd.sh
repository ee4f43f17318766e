O=gpurun_out/r2bm; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
for v in nofuse main nofuse main; do
  if [ $v = main ]; then L=""; else L=tools/variants/libibf_$v.so; fi
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 >> $O/ccd_$v.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_ccd.csv python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 1 --ncu > $O/ncu_ccdlist.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
