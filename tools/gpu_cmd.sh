O=gpurun_out/r2ah; mkdir -p $O
timeout 2400 python tools/squishy_run.py --frames 120 --plate-speed 2.0 --every 5 --certify --out $O/press120.json > $O/press120.log 2>&1
timeout 500 python tools/squishy_run.py --frames 52 --plate-speed 2.0 --every 4 --dump /tmp/sq52.npz > $O/press.log 2>&1
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_energy\b|k_energy\(" -c 3 --csv python tools/squishy_run.py --load /tmp/sq52.npz --frames 1 --plate-speed 2.0 > $O/ncu_energy.csv 2>&1
