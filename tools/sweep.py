"""Environment-knob sweep of the device solve on ONE graph (built once).

  python tools/sweep.py CONFIG 'LR_SPMV_HEAD=8192' 'LR_SPMV_HEAD=16384' ...

Each argument is a set of space-separated VAR=VALUE assignments applied before
a few timed device solves (knobs read per launch, e.g. LR_SPMV_HEAD and
LR_SPMV_KEEP, take effect in-process).  Prints one line per setting: solve ms
and the SpMV's average active launch time.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1609_09068_b200 as lr

    cfg = int(sys.argv[1])
    shrink = int(os.environ.get("SWEEP_SHRINK", "0"))
    t0 = time.perf_counter()
    g = lr.config_graph(cfg, shrink)
    eng = lr.Engine(g, 100, device=0)
    print(f"config {cfg}: n={g.n} m={g.m} setup {time.perf_counter() - t0:.1f}s", flush=True)
    n = g.n
    dev = torch.device("cuda", 0)
    w = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    r3 = torch.empty(n, dtype=torch.float64, device=dev)
    r1 = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    params = lr.SolverParams(0.85, 1e-12)
    reps = int(os.environ.get("SWEEP_REPS", "3"))
    for setting in sys.argv[2:]:
        for kv in setting.split():
            k, v = kv.split("=", 1)
            os.environ[k] = v
        ms, act = [], []
        for i in range(reps + 1):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            a = time.perf_counter()
            info = eng.solve_ptr(w.data_ptr(), r3.data_ptr(), r1.data_ptr(), host=False, params=params)
            torch.cuda.synchronize()
            if i == 0:
                continue  # warm-up
            ms.append(info["device_ms"])
            if info["spmv_active_launches"]:
                act.append(info["spmv_active_ms"] / info["spmv_active_launches"])
        print(f"{setting:40s} solve {np.mean(ms):9.3f} ms  spmv/launch {1e3 * np.mean(act) if act else 0:8.2f} us",
              flush=True)
        for kv in setting.split():
            os.environ.pop(kv.split("=", 1)[0], None)


if __name__ == "__main__":
    main()
