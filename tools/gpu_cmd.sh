O=gpurun_out/r2l; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -s -rA > $O/tests.log 2>&1
timeout 400 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq48.npz --frames 0 --iters 200 > $O/pcg_new.log 2>&1
IBF_LIB=tools/variants/libibf_head.so timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq48.npz --frames 0 --iters 200 > $O/pcg_head.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
