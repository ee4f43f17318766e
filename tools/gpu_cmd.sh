O=gpurun_out/r2ba; mkdir -p $O
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_pcg -c 1 -o $O/k_pcg python tools/pcg_contact_bench.py --load /tmp/sq52.npz --frames 0 --iters 60 --ncu > $O/ncu_pcg.log 2>&1
IBF_BENCH_PROFILE_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-certify > $O/bench_under_ncu.log 2>&1
gzip -f $O/launches_bench.csv
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
