O=gpurun_out/r2p; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -s -rA > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base bin base2; do
  L=""; [ $v = bin ] && L=tools/variants/libibf_bin.so
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 10 > $O/ccd_$v.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_ccd.csv python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 1 --ncu > /dev/null 2>&1
