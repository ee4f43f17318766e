O=gpurun_out/r2bj; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 45 --plate-speed 2.0 --every 8 --dump /tmp/sq45.npz > $O/press.log 2>&1
timeout 900 python tools/ccd_cache_sim.py --load /tmp/sq45.npz --frames 3 > $O/sim.log 2>&1
