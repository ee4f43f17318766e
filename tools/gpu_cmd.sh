mkdir -p gpurun_out/r2d
./tools/micro/fp64_peak > gpurun_out/r2d/fp64_peak.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2d/tests.log 2>&1
D=/tmp/sq45r.npz
timeout 900 python tools/pcg_contact_bench.py --frames 45 --dump $D > gpurun_out/r2d/pcgb_reorder.log 2>&1
timeout 900 python tools/pcg_contact_bench.py --frames 45 --no-reorder > gpurun_out/r2d/pcgb_lattice.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_pcg -c 1 -o gpurun_out/r2d/k_pcg_contacts -f python tools/pcg_contact_bench.py --frames 0 --load $D --iters 100 --ncu > gpurun_out/r2d/ncu_pcg.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d/bench.json 2> gpurun_out/r2d/bench.err
