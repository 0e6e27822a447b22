"""Host setup phases of one config (generation, partition, layout) -- LR_PLAN_PROF=1 adds the layout phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09068_b200 as lr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t = time.time()
g = lr.config_graph(cfg, 0)
print(f"config {cfg}: generate {time.time() - t:.1f} s (n={g.n} m={g.m}), host threads {os.cpu_count()}", flush=True)
t = time.time()
lr.find_components(g)
print(f"find_components {time.time() - t:.1f} s", flush=True)
t = time.time()
lr.Plan(g)
print(f"plan (partition + layout) {time.time() - t:.1f} s", flush=True)
t = time.time()
lr.Plan(g, baseline=True)
print(f"baseline plan {time.time() - t:.1f} s", flush=True)
