O=gpurun_out/r2as; mkdir -p $O
for v in base sell32 base2 sell322; do
  L=""; case $v in sell32|sell322) L=tools/variants/libibf_sell32.so;; esac
  IBF_LIB=$L timeout 600 python bench.py --workload c5 --steps 10 --warmup 2 --concurrency 8 > $O/c5_$v.json 2> $O/c5_$v.err
done
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
for v in base stop base2 stop2; do
  L=""; case $v in stop|stop2) L=tools/variants/libibf_stop.so;; esac
  IBF_LIB=$L timeout 300 python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 200 > $O/pcg_$v.log 2>&1
done
