O=gpurun_out/r2bw; mkdir -p $O
timeout 1500 python tools/squishy_run.py --frames 120 --plate-speed 2.0 --certify --every 5 --out $O/press120.json > $O/press.log 2>&1
