O=gpurun_out/r2bo; mkdir -p $O
for v in main em3 em4; do
  if [ $v = main ]; then L=""; else L=tools/variants/libibf_$v.so; fi
  IBF_LIB=$L timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-certify > $O/bench_$v.json 2> $O/bench_$v.err
done
