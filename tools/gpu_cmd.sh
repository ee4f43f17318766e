O=gpurun_out/r2ap; mkdir -p $O
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
from paper_2512_12151_b200 import scenes, dist
system, state, params = scenes.c2_scene()
part = dist.Partition.local_parts(2)
bench._partition_probe(system.device, system, state, params, part)
print('probe ok (local partitions x2, C2)')
" > $O/probe.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -rA > $O/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err
