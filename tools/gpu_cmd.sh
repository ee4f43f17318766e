O=gpurun_out/r2aa; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -s -rA > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base head base2; do
  L=""; [ $v = head ] && L=tools/variants/libibf_head.so
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 10 > $O/ccd_$v.log 2>&1
done
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
IBF_PY_OUTER=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_pyouter.json 2> $O/bench_pyouter.err
