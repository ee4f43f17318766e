for v in noch ch noch ch; do echo "== $v"; IBF_LIB=tools/variants/libibf_$v.so timeout 300 python tools/bench_spmv.py; done > gpurun_out/ch_micro.log 2>&1
