O=gpurun_out/r2bt; mkdir -p $O
IBF_BENCH_PROFILE_RANGE=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k "regex:k_refit_chunks|k_gather_blocks|k_energy$|k_refit_top" -c 4 -o $O/asm_ccd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-certify > $O/ncu.log 2>&1
