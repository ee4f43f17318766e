O=gpurun_out/r2au; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base stopc32 stopc8 base2 stopc322; do
  L=""; case $v in stopc32|stopc322) L=tools/variants/libibf_stopc32.so;; stopc8) L=tools/variants/libibf_stopc8.so;; esac
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
