O=gpurun_out/r2w; mkdir -p $O
timeout 1200 python tools/long_parity.py c1 50 1e-15 > $O/c1_parity.log 2>&1 &
P1=$!
timeout 900 python -m pytest tests -m gpu -x -q -s -rA > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base minb5 base2; do
  L=""; [ $v = minb5 ] && L=tools/variants/libibf_minb5.so
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
wait $P1
