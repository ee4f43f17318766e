mkdir -p gpurun_out/r2c
D=/tmp/sq45.npz
timeout 900 python tools/pcg_contact_bench.py --frames 45 --dump $D > gpurun_out/r2c/pcgb.log 2>&1
IBF_LIB=tools/variants/libibf_prof.so timeout 300 python tools/pcg_contact_bench.py --frames 0 --load $D --iters 100 > gpurun_out/r2c/pcgb_prof.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_pcg -c 1 -o gpurun_out/r2c/k_pcg_contacts -f python tools/pcg_contact_bench.py --frames 0 --load $D --iters 100 --ncu > gpurun_out/r2c/ncu_pcg.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2c/launches_frame.csv python tools/squishy_run.py --load $D --frames 1 --profile-frames 1 > gpurun_out/r2c/sq_frame.log 2>&1
gzip -f gpurun_out/r2c/launches_frame.csv
