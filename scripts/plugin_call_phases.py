"""Where the reference-API call's time goes at C4 (bench.py plugin_call):
the Python-side phases of run_scenario's native delegation, timed apart."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_08058_b200 import (AggregationExecutor, BufferPool, CudaDevice, ExecutorPool,
                                   Integration, IntegrationMode, Runtime, ScenarioConfig,
                                   build_scenario, kernel_transform)
from paper_2303_08058_b200 import miniapp
from paper_2303_08058_b200.native_machine import run_native

S, W, E, M, steps = 32768, 16, 8, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 3
T = {}
t = time.perf_counter()
rt = Runtime(W); dev = CudaDevice(0)
integ = Integration(rt, dev, IntegrationMode.POLLING)
pool = ExecutorPool(integ, E); bufs = BufferPool(dev)
aggs = [AggregationExecutor(ex, M, bufs) for ex in pool.executors]
for a in aggs:
    for k in range(5):
        a.register_kind(k, kernel_transform(k))
T["stack"] = time.perf_counter() - t
t = time.perf_counter()
sc = build_scenario(ScenarioConfig(subgrids=S, steps=steps))
T["build_scenario"] = time.perf_counter() - t
by_grid = [aggs[g % E] for g in range(S)]
t = time.perf_counter()
plan = miniapp._native_plan(sc, rt, dev, aggs, by_grid)
T["native_plan"] = time.perf_counter() - t
t = time.perf_counter()
cells = sc.cells()
T["cells_gather"] = time.perf_counter() - t
stats = np.zeros((steps, plan["executors"], plan["max_agg"] + 3), dtype=np.int64)
for rep in range(2):
    t = time.perf_counter()
    res, _ = run_native(S, steps, cells=cells.copy(), exec_stats=stats, zero_copy=3, **plan)
    T[f"run_native_{rep}"] = time.perf_counter() - t
    T[f"steps_ms_{rep}"] = [round(m.wall_ms, 2) for m in res.per_step]
t = time.perf_counter()
for g, row in zip(sc.grids, cells):
    g.cells[:] = row
T["writeback"] = time.perf_counter() - t
rt.shutdown(); dev.destroy()
print(json.dumps(T))
