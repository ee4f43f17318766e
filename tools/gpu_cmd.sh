O=gpurun_out/r2ae; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_kernels.py -m gpu -x -q -s -k "pcg or production or partitioned or contact_heavy or trajectory or c2 or c3 or native" > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
timeout 500 python tools/squishy_run.py --load /tmp/sq52.npz --frames 3 --plate-speed 2.0 --every 1 --dump /tmp/sq55.npz > $O/press55.log 2>&1
for st in sq52 sq55; do
for v in late early late2; do
  L=""; [ $v = early ] && L=tools/variants/libibf_early.so
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/$st.npz --frames 0 --iters 200 > $O/pcg_${st}_$v.log 2>&1
done
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
