for v in default static; do
  if [ $v = default ]; then L=""; else L=$PWD/tools/variants/libibf_$v.so; fi
  echo -n "$v " >> gpurun_out/ab.txt
  IBF_LIB=$L python tools/bench_spmv.py >> gpurun_out/ab.txt 2>> gpurun_out/ab.err
done
IBF_LIB=$PWD/tools/variants/libibf_prof.so python tools/bench_spmv.py > gpurun_out/prof_spmv.json 2> gpurun_out/prof_spmv.err
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu3.log
