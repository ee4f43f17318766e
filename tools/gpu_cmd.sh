O=gpurun_out/r2an; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base head base2 head2; do
  L=""; [ ${v%2} = head ] && L=tools/variants/libibf_head.so
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 10 > $O/ccd_$v.log 2>&1
done
