O=gpurun_out/r2bx; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 500 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
for r in 1 2; do
  timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 >> $O/ccd_main.log 2>&1
  timeout 300 python tools/ccd_bench.py --load /tmp/sq48.npz --frames 0 --reps 10 --scale 0.3 >> $O/ccds_main.log 2>&1
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
