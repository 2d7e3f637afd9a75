"""Host vs GPU batch-plan builder (BatchSchedule::build) on the C3 / C4 shapes.

    python tools/plan_bench.py [reddit products_appnp]   -> one JSON line per workload
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402


def main(names):
    for name in names or ["reddit", "products_appnp"]:
        ds = make_dataset(name, with_features=False)
        P = ds.workload.parts
        gb.BatchSchedule.build(ds.graph, ds.assignment, P, device=True)  # warm-up (context, cub)
        host = gb.BatchSchedule.build(ds.graph, ds.assignment, P)
        devs = [gb.BatchSchedule.build(ds.graph, ds.assignment, P, device=True) for _ in range(3)]
        same = all(np.array_equal(host.plan(p).gcn_cols, devs[0].plan(p).gcn_cols) for p in (0, P // 2, P - 1))
        print(json.dumps({
            "workload": name, "nodes": ds.graph.num_nodes, "stored_nnz": ds.graph.num_edges, "parts": P,
            "host_ms": round(host.timing()[1], 1), "host_threads": os.cpu_count(),
            "device_gpu_ms": [round(d.timing()[0], 2) for d in devs],
            "device_total_ms": [round(d.timing()[1], 1) for d in devs], "spot_check_equal": same}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
