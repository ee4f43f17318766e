O=gpurun_out/r2aw; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 36 --plate-speed 2.0 --every 4 --dump /tmp/sq36.npz > $O/press36.log 2>&1
timeout 500 python tools/squishy_run.py --load /tmp/sq36.npz --frames 6 --plate-speed 2.0 --every 1 --dump /tmp/sq42.npz > $O/press42.log 2>&1
for st in sq36 sq42; do
for v in on off on2 off2; do
  R=1e9; case $v in on|on2) R=0;; esac
  IBF_PCG_PMAT_RATIO=$R timeout 300 python tools/pcg_contact_bench.py --load /tmp/$st.npz --frames 0 --iters 200 > $O/pcg_${st}_$v.log 2>&1
done
done
