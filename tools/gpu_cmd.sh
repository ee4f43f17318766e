timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -k contact_heavy 2>&1 | grep -E "assert|Error|where|passed|failed" | head -20 > gpurun_out/pytest_ch.log
