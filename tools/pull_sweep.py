"""HistoryStore pull / push bandwidth sweep: d in {16, 48, 64, 128, 256, 604},
rows in {1e3 .. 1e7}, sorted random ids into a table of max(4 * rows, 1M) nodes. Bytes per
op = rows * (8 d + 4) (read + write each row, plus the id). Prints one JSON line per point."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402

peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6545.6) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0
s = torch.cuda.current_stream()
for d in (16, 48, 64, 128, 256, 604):
    for rows in (10**3, 10**4, 10**5, 10**6, 10**7):
        n = max(4 * rows, 10**6)
        if n * d * 4 > 40e9:
            continue
        h = gb.HistoryStore(1, n, d)
        rng = np.random.default_rng(d + rows)
        ids = torch.from_numpy(np.sort(rng.choice(n, size=rows, replace=False)).astype(np.int32)).cuda()
        buf = torch.randn(rows, h.ld, device="cuda").abs()
        res = {"d": d, "rows": rows, "table_rows": n}
        for name, fn in (("push", h.push_device), ("pull", h.pull_device)):
            for _ in range(2):
                fn(1, ids, rows, buf, h.ld, s)
            it = max(3, min(200, int(2e8 // (rows * d * 8))))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(it):
                fn(1, ids, rows, buf, h.ld, s)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / it
            gbs = rows * (8 * d + 4) / (ms / 1000) / 1e9
            res[name] = {"us": 1000 * ms, "GBps": gbs, "frac_of_hbm_peak": gbs / peak}
        h.check()
        print(json.dumps(res), flush=True)
        del h, buf, ids
        torch.cuda.empty_cache()
