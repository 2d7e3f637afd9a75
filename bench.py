"""GAS training throughput on B200 (BASELINE.json metric: GAS training nodes/sec, GCN,
Reddit-shape; history pull GB/s).

One step = one GAS epoch (gas_epoch, src/trainer.cpp:386-442): every one of the 200
partition batches runs forward, push, loss, backward and one Adam step, in the seeded
shuffled order. value = nodes / second = num_nodes * steps / device time (max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref: the reference
sources compiled in place) on the box's host cores, one partition batch per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GAS training nodes/sec (GCN, Reddit-shape)"
PEAKS = ROOT / "MEASURED_PEAKS.json"
HBM_FALLBACK_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler over the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.file,
                                         stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(",") for r in Path(self.file.name).read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def spmm_bytes(nb: int, ne: int, nnz: int, d: int) -> tuple[float, float]:
    """compulsory model 8(B+1) + 8E + 4d*V + 4d*B; effective (no reuse) 4d*E."""
    return 8 * (nb + 1) + 8 * nnz + 4 * d * ne + 4 * d * nb, 4.0 * d * nnz


def epoch_roofline(sched, w, ms_per_epoch: float, gpus: int = 1) -> dict:
    """Epoch-level roofline (SURVEY §8d "roofline fraction"): t_min = algorithmic bytes /
    HBM peak + tensor-core flops / TF32 peak, against the measured epoch. Bytes: the per-batch
    SpMM compulsory model for layers 2..L, layer 1 hoisted (stencil + X once + output), the
    intra-batch SpMM backward (gy + gx rows + pointers; its ~8 B/entry is omitted), pushes and
    Adam; flops: 3xTF32 = 3 MMAs per fwd / dgrad / wgrad GEMM."""
    F, H, C, L = w.in_dim, w.hidden, w.num_classes, w.num_layers
    dims = [F] + [H] * (L - 1) + [C]
    by, fl, E = 0.0, 0.0, 0
    for p in range(w.parts):
        nb, ne, _, _, nnz, _ = (int(v) for v in sched.sizes(p))
        E += nnz
        for _ in range(1, L):  # layers 2..L gather d = H
            by += spmm_bytes(nb, ne, nnz, H)[0]
        by += (L - 1) * (8 * (nb + 1) + 8 * H * nb)  # backward over batch rows
        by += (L - 1) * nb * (8 * H + 4)  # pushes
        fwd = sum(2.0 * nb * dims[l] * dims[l + 1] for l in range(L))
        dgrad = sum(2.0 * nb * dims[l] * dims[l + 1] for l in range(1, L))
        fl += 3 * (2 * fwd + dgrad)  # fwd + wgrad (same flops) + dgrad, 3 MMAs each
    by += 12.0 * E + 8.0 * w.num_nodes * F  # hoisted layer 1: stencil, X once, output
    try:
        pk = json.loads(PEAKS.read_text())
        tc = float(pk["bf16_tflops"]) / 2  # dense TF32 = half the dense bf16 rate
    except Exception:
        tc = 1125.0
    hbm, _ = peak_hbm()
    t_min = (by / (hbm * 1e9) + fl / (tc * 1e12)) / gpus  # data-parallel: the epoch's work splits over gpus
    return {"gpus": gpus, "bytes_GB": by / 1e9, "tflop": fl / 1e12, "t_min_ms": 1e3 * t_min, "measured_ms": ms_per_epoch,
            "frac": 1e3 * t_min / ms_per_epoch, "hbm_GBps": hbm, "tf32_TFLOPs": tc}


def peak_hbm() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def cpu_baseline(ds, sample: int, kind_hint: str = "reference") -> dict:
    """The reference (oracle/_ref) on a bounded sample of the same workload, 1 core."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from pyoracle import REF_SO, RefLib, make_spec

    w = ds.workload
    if not REF_SO.exists():
        return {"value": None, "unit": "nodes/s", "cores": 1, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    R = RefLib()
    order = R.epoch_order(w.parts, 3, 0)
    warm = 2  # untimed: first-touch page faults of the fresh history store, as the reference arm's warm-up
    parts = [int(p) for p in order[:sample + warm]]
    spec = make_spec(kind=0, num_layers=w.num_layers, hidden=w.hidden, seed=3, lr=w.lr)
    s = R.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                  w.parts, spec, sample_parts=parts)
    for slot in range(warm):
        s.run(slot, 0)
    nodes = int(sum((ds.assignment == p).sum() for p in parts[warm:]))
    secs = 0.0
    for slot in range(warm, len(parts)):
        secs += s.run(slot, 0)[1]
    return {"value": nodes / secs, "unit": "nodes/s", "cores": 1, "kind": "reference", **host_cpu(),
            "sample": f"{len(parts) - warm} of {w.parts} partition batches of the same graph after {warm} untimed "
                      f"(gas_epoch batches: forward, push/pull, backward, Adam), {nodes} nodes in {secs:.1f} s, "
                      "single-threaded reference"}


def load_workloads():
    """paper_2106_05609_b200/workloads.py loaded by path: data-only at import, so the reference
    arm gets the workload table without importing the package (which loads libgasb.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gasb_workloads", ROOT / "paper_2106_05609_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["gasb_workloads"] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def host_cpu() -> dict:
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count()
    return {"cpu_model": model, "host_cores": os.cpu_count(), "cores_available": avail}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    from pyoracle import REF_SO, OracleSynth, RefLib, make_spec

    if not REF_SO.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref.so not built"}))
        return
    # the same graph / features / labels / partition as our arm, generated by the oracle's
    # restatement of the generator (tests/test_workloads.py: bit-identical); no libgasb.so
    ds = load_workloads().make_dataset(args.workload, backend=OracleSynth())
    w = ds.workload
    R = RefLib()
    order = [int(p) for p in R.epoch_order(w.parts, 3, 0)]
    k = args.steps + args.warmup
    parts = [order[i % w.parts] for i in range(min(k, w.parts))]
    s = R.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                  w.parts, make_spec(kind=0, num_layers=w.num_layers, hidden=w.hidden, seed=3, lr=w.lr), sample_parts=parts)
    times, nodes = [], []
    for i in range(k):
        slot = i % len(parts)
        _, secs = s.run(slot, 0)
        if i >= args.warmup:
            times.append(secs)
            nodes.append(int((ds.assignment == parts[slot]).sum()))
    value = sum(nodes) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulation)",
        "data": "synthetic", "config": workload_config(ds),
        "step": "one partition batch of gas_epoch (a bounded sample of the epoch; nodes/s is per node either way)",
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": 1, "kind": "reference", **host_cpu(),
                         "sample": f"one partition batch per step ({int(np.mean(nodes))} nodes avg), reference "
                                   "gas_epoch batch path, single-threaded (the reference has no parallel compute)"},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(ds) -> dict:
    """Identical in both arms (the step unit and the parallelism are top-level keys)."""
    w = ds.workload
    return {"workload": f"{w.name}-shape GAS-{w.kind.upper()}", "num_nodes": w.num_nodes,
            "stored_nnz": int(len(ds.cols)), "in_dim": w.in_dim, "hidden": w.hidden, "num_classes": w.num_classes,
            "layers": w.num_layers, "partitions": w.parts, "partitioner": "planted communities (natural partition)",
            "features": f"N(0,1) + {w.signal} x class centroid", "communities_per_part": w.comm_per_part,
            "adam_lr": w.lr, "seeds": {"graph": w.seed, "model": 3},
            "l2_policy": "inputs larger than L2 (features 567 MB, histories 716 MB vs 126 MB L2)"}


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    shared = ws > torch.cuda.device_count()  # ranks sharing one GPU: a correctness run only
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if shared:  # NCCL refuses two ranks on one device; gloo carries the control plane
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_05609_b200 as gb
    from paper_2106_05609_b200._native import check, lib
    from paper_2106_05609_b200.workloads import make_dataset

    t0 = time.time()
    ds = make_dataset(args.workload)
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3, opt=gb.AdamConfig(lr=w.lr))
    # N > 1: data-parallel epochs (dp.cu: k batches per step, exchange over peer memory); each
    # rank hoists layer 1 over its own batches of the epoch
    opts = gb.TrainerOptions(seg_edges=args.seg_edges, device=local, hoist_layer1=not args.no_hoist)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec, opts)
    runner = tr
    if ws > 1:
        runner = gb.DataParallelTrainer(tr, rank, ws, group=torch.distributed.group.WORLD, placement=args.placement)
    log(f"[rank {rank}] setup {time.time() - t0:.1f}s  n={w.num_nodes} nnz={len(ds.cols)}")
    stream = torch.cuda.ExternalStream(tr.stream())

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()

    for e in range(args.warmup):
        l = runner.gas_epoch(e)
        log(f"[rank {rank}] warmup epoch {e} loss {l:.5f}")
    # ---- device-timed region: K epochs back to back ----
    clocks = Clocks(local)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        if ws > 1:
            runner.epoch_async(args.warmup + k)
        else:
            tr.gas_epoch_async(args.warmup + k)
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if ws > 1:
        runner.check()
        part_l = runner.part_losses()
        train = tr.part_train_rows()
        order = gb.epoch_order(w.parts, 3, args.warmup + args.steps - 1)
        st = [p for p in order if train[p] > 0]
        loss = float(sum(part_l[p] for p in st) / len(st))
    else:
        loss = tr.last_loss()
    launches = runner.launch_count() * args.steps
    t = torch.tensor([ms], device="cpu" if shared else "cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # one epoch = every node once; under DP the ranks split each epoch's batches
    nodes_per_step = w.num_nodes if ws > 1 else ws * w.num_nodes
    value = nodes_per_step * args.steps / (ms / 1000.0)

    # ---- end to end through the public API with host buffers ----
    x = np.ascontiguousarray(ds.features, np.float32)
    check(lib.gasb_host_register(x.ctypes.data, x.nbytes))
    barrier()
    t1 = time.perf_counter()
    # pipelined driver: step k+1's input H2D (copy stream) overlaps step k's compute; every
    # step still copies its whole input from pinned host memory and reads its losses back
    tr.stage_features(x)
    for k in range(args.steps):
        tr.commit_features()
        ep = args.warmup + args.steps + k
        if ws > 1:
            runner.epoch_async(ep)
        else:
            tr.gas_epoch_async(ep)
        if k + 1 < args.steps:
            tr.stage_features(x)
        if ws > 1:  # D2H of the step's result: per-part losses
            runner.check()
            runner.part_losses()
        else:
            tr.last_loss()
    barrier()
    e2e_s = time.perf_counter() - t1
    check(lib.gasb_host_unregister(x.ctypes.data))
    t = torch.tensor([e2e_s], device="cpu" if shared else "cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e = {"value": nodes_per_step * args.steps / e2e_s, "unit": "nodes/s", "h2d_bytes_per_step": int(x.nbytes),
           "d2h_bytes_per_step": 8 * w.parts}

    # ---- roofline of the dominant kernel: per-batch SpMM at d = hidden (layers 2..L) ----
    peak, peak_kind = peak_hbm()
    tot_t, tot_b, tot_eff = 0.0, 0.0, 0.0
    parts = list(range(0, w.parts, max(1, w.parts // args.profile_parts)))
    for p in parts:
        nb, ne, _, _, nnz, _ = (int(v) for v in sched.sizes(p))
        ms_p = tr.profile_spmm(p, 2, 3)
        b, eff = spmm_bytes(nb, ne, nnz, w.hidden)
        tot_t += ms_p
        tot_b += b
        tot_eff += eff
    achieved = tot_b / (tot_t / 1000.0) / 1e9
    roof = {"kernel": "spmm_fwd_kernel (per-batch aggregation, d=hidden)", "bound": "hbm", "achieved": achieved,
            "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "avg_launch_ms": tot_t / len(parts), "algorithmic_bytes_per_launch": tot_b / len(parts),
            "effective_gather_GBps": tot_eff / (tot_t / 1000.0) / 1e9, "traffic": None}
    # second ceiling: the measured L2 -> SM rate of 1 KB row gathers from an L2-resident table
    # (tools/l2bw/l2_bw.cu on a B200); the SpMM's gathered bytes are mostly L2 hits
    l2f = ROOT / "profiles" / "r1_l2_gather_ceiling.jsonl"
    if l2f.exists():
        try:
            rows = [json.loads(x) for x in l2f.read_text().splitlines() if x.strip()]
            l2peak = max(r["gbs"] for r in rows if r["pattern"] == "gather_1kb_rows" and r["buffer_mb"] <= 64)
            roof["l2_gather_peak_GBps"] = l2peak
            roof["l2_gather_frac"] = roof["effective_gather_GBps"] / l2peak
        except Exception:
            pass
    prof = ROOT / "profiles" / "spmm_traffic.json"
    if prof.exists():
        try:
            roof["traffic"] = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            pass
    # third ceiling, the one the gathers are actually bound by: the launch's gathered bytes at
    # the measured TMA tile::gather4 rates (tools/l2bw/tma_gather_bw on a B200: 1 KB rows from
    # an L2-resident table vs a DRAM-resident one), split into L2 hits and DRAM misses by the
    # kernel's ncu DRAM traffic
    tg = ROOT / "profiles" / "r2_tma_gather_ceiling.jsonl"
    if tg.exists() and roof["traffic"]:
        try:
            rows = [json.loads(x) for x in tg.read_text().splitlines() if x.startswith("{")]
            l2r = max(r["gbs"] for r in rows if r["table_mb"] <= 64 and r["row_bytes"] == 1024)
            drr = max(r["gbs"] for r in rows if r["table_mb"] >= 1024 and r["row_bytes"] == 1024)
            gathered = tot_eff / len(parts)
            miss = min(float(roof["traffic"]), gathered)
            t_min = (gathered - miss) / (l2r * 1e9) + miss / (drr * 1e9)
            roof["gather_model"] = {"l2_hit_GBps": l2r, "dram_miss_GBps": drr, "gathered_bytes": gathered,
                                    "dram_bytes": miss, "t_min_us": 1e6 * t_min,
                                    "frac": t_min / (tot_t / len(parts) / 1000.0),
                                    "source": "profiles/r2_tma_gather_ceiling.jsonl"}
        except Exception:
            pass
    extra = {}
    if ws > 1:  # exchange bytes of the last timed epoch (dp.cu bookkeeping), max over ranks
        tf = runner.traffic()
        t = torch.tensor([float(tf["nvlink_bytes"])], device="cpu" if shared else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        extra["exchange"] = {"placement": args.placement, "nvlink_bytes_per_epoch_max_rank": int(t.item()),
                             "nvlink_GBps_avg_over_epoch": float(t.item()) / (ms / args.steps / 1000) / 1e9,
                             "history_rows_held_rank0": tf["shard_rows"],
                             "link_peak_GBps_per_direction": 900.0}
    if not args.no_hoist and ws == 1:
        ms_h = tr.profile_spmm(-1, 1, 2)
        extra["hoisted_layer1_ms"] = ms_h
    # ---- history pull GB/s at C3 halo sizes (HistoryStore::pull, d = hidden) ----
    pull = pull_bandwidth(tr, sched, w, torch)

    line = {
        "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f32 (f64 SpMM accumulation)", "data": "synthetic",
        "config": workload_config(ds),
        "parallelism": f"dp{ws} (partition batches split over ranks, peer-memory exchange)" if ws > 1 else "single-gpu",
        "step": "one GAS epoch (all partition batches, one Adam step each)",
        "e2e": e2e, "gpu_launches": launches, "roofline": roof, "clocks": clk, "final_loss": loss,
        "trains": {"final_loss": loss, "ln_num_classes": math.log(w.num_classes),
                   "live": bool(loss < math.log(w.num_classes) - 0.1)},
        "history_pull_GBps": pull, "epoch_roofline": epoch_roofline(sched, w, ms / args.steps, ws), **extra,
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(ds, args.cpu_sample)
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def pull_bandwidth(tr, sched, w, torch) -> dict:
    """HistoryStore::pull of a batch's halo rows (ids + d floats read, d floats written), on a
    store of the trainer's shape (its own store may be sharded across a data-parallel group)."""
    import paper_2106_05609_b200 as gb
    th = tr.history
    if th is None:
        return None
    hist = gb.HistoryStore(1, w.num_nodes, w.num_classes if w.kind == "appnp" else w.hidden)
    p = 0
    plan = sched.plan(p)
    halo = torch.from_numpy(plan.halo_nodes).cuda()
    out = torch.empty(len(halo), hist.ld, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(2):
        hist.pull_device(1, halo, len(halo), out, hist.ld, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record(s)
    for _ in range(it):
        hist.pull_device(1, halo, len(halo), out, hist.ld, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    byts = len(halo) * (8 * hist.dim() + 4)
    peak, _ = peak_hbm()
    return {"rows": len(halo), "dim": hist.dim(), "ms": ms, "GBps": byts / (ms / 1000) / 1e9,
            "frac": byts / (ms / 1000) / 1e9 / peak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="reddit")
    ap.add_argument("--seg-edges", type=int, default=128)
    ap.add_argument("--no-hoist", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=3)
    ap.add_argument("--profile-parts", type=int, default=20)
    ap.add_argument("--placement", default="replicated", choices=["replicated", "sharded"],
                    help="history placement of a data-parallel run (gasb.h GASB_DP_*)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: re-exec as N ranks (one process per GPU)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
