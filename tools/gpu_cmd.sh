O=gpurun_out/r2bs; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 48 --plate-speed 2.0 --every 8 --dump /tmp/sq48.npz > $O/press.log 2>&1
for v in r1 main r4 r1 main r4; do
  if [ $v = main ]; then L=""; else L=tools/variants/libibf_$v.so; fi
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq48.npz --frames 0 --iters 50 >> $O/asm_$v.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
