mkdir -p gpurun_out/r2
free -g > gpurun_out/r2/free.txt
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak > ../../gpurun_out/r2/fp64_peak.json; cd ../..
timeout 1500 python -m pytest tests -m gpu -q -s -k "production or composition or step_limit_and_update" > gpurun_out/r2/tests_new.log 2>&1
timeout 1800 python tools/squishy_run.py --frames 100 --plate-speed 2.0 --plate-stop 0.3 --dump /tmp/sq100.npz --out gpurun_out/r2/sq3_press.json > gpurun_out/r2/sq3_press.log 2>&1
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:"k_pcg|k_traverse|k_elem|k_gather_blocks|k_energy|k_pair_toi|k_vertex_rows" -c 8 -o gpurun_out/r2/sq100_full python tools/squishy_run.py --load /tmp/sq100.npz --frames 1 --profile-frames 1 > gpurun_out/r2/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 20000 --csv --log-file gpurun_out/r2/sq100_launches.csv python tools/squishy_run.py --load /tmp/sq100.npz --frames 1 --profile-frames 1 > gpurun_out/r2/ncu_launches.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2/tests.log 2>&1
