O=gpurun_out/r2ac; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -x -q -s -k "broadphase or static or min_distance or press_state or trajectory or c2_stack or c3_twisted or native_outer" > $O/tests.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base atomrefit base2; do
  L=""; [ $v = atomrefit ] && L=tools/variants/libibf_atomrefit.so
  IBF_LIB=$L timeout 300 python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 20 > $O/ccd_$v.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_ccd.csv python tools/ccd_bench.py --load /tmp/sq52.npz --frames 0 --reps 1 --ncu > /dev/null 2>&1
