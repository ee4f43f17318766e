O=gpurun_out/r2az; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -s -rA > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base dotsafter base2 dotsafter2; do
  L=""; case $v in dotsafter|dotsafter2) L=tools/variants/libibf_dotsafter.so;; esac
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
