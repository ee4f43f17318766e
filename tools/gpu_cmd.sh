O=gpurun_out/r2x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -x -q -s -k "broadphase or static or min_distance or press_state or production or contact_heavy or trajectory" > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base nolbox base2; do
  L=""; [ $v = nolbox ] && L=tools/variants/libibf_nolbox.so
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 10 > $O/ccd_$v.log 2>&1
done
for v in base cond base2; do
  L=""; [ $v = cond ] && L=tools/variants/libibf_cond.so
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
