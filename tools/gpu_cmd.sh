O=gpurun_out/r2ag; mkdir -p $O
timeout 500 python tools/pcg_contact_bench.py --numbering lattice --frames 52 --iters 200 > $O/pcg_lattice.log 2>&1
for w in 64 128 256; do
  IBF_SELL_NUMBERING_WINDOW=$w timeout 500 python tools/pcg_contact_bench.py --numbering sell --frames 52 --iters 200 > $O/pcg_sell$w.log 2>&1
done
