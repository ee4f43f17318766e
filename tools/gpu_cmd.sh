mkdir -p gpurun_out/r2f
D=/tmp/sqL.npz
V=tools/variants
timeout 900 python tools/ccd_bench.py --frames 45 --dump $D > gpurun_out/r2f/ccd_main.log 2>&1
for v in base nosplit novf; do
  IBF_LIB=$V/libibf_$v.so timeout 300 python tools/ccd_bench.py --frames 0 --load $D > gpurun_out/r2f/ccd_$v.log 2>&1
done
timeout 300 python tools/pcg_contact_bench.py --frames 0 --load $D > gpurun_out/r2f/pcgb_main.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2f/tests.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err
