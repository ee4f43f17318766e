O=gpurun_out/r2ax; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in always ratio02 always2 ratio022; do
  R=0; case $v in ratio02|ratio022) R=0.2;; esac
  IBF_PCG_PMAT_RATIO=$R timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q -rA > $O/tests.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
