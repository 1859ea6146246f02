"""Benchmark: edges/sec generated for BASELINE config 2 (n=1e7, k=32,
gamma=2.5, T=0, seed 2) on N B200s, with the roofline of the range-query
kernel and the reference algorithm's CPU time beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full generation (Philox sampling, band index build, count
pass, scan, write pass, row ordering) of the whole graph; with N ranks each
rank emits the rows of its angular sector, so the N ranks together produce
the whole graph once per step (strong scaling over a fixed graph).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    0: dict(n=10_000, avg_degree=6.0, gamma=3.0, seed=0),
    1: dict(n=1_000_000, avg_degree=10.0, gamma=3.0, seed=1),
    2: dict(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2),
    3: dict(n=100_000_000, avg_degree=16.0, gamma=3.0, seed=3),
    4: dict(n=10_000_000, avg_degree=4.0, gamma=2.2, seed=4),  # one point; --sweep runs all 9
}
SWEEP = [(k, g) for k in (4.0, 64.0, 256.0) for g in (2.2, 3.0, 5.0)]


def metric_for(params):
    if params == CONFIGS[2]:
        return METRIC
    return (f"edges/sec generated (n={params['n']:.0e},k={params['avg_degree']:g},"
            f"gamma={params['gamma']:g})").replace("e+0", "e")


def config_params(args):
    params = dict(CONFIGS[args.config])
    for key, val in (("n", args.n), ("avg_degree", args.k), ("gamma", args.gamma),
                     ("seed", args.seed)):
        if val is not None:
            params[key] = val
    return params
METRIC = "edges/sec generated (n=1e7,k=32,gamma=2.5)"
UNIT = "edges/s"

# algorithmic bytes of the range query:
#   every point record is read once: phi, p_x, p_y, c_x, c_y, rad^2 (6 x f64),
#   r, (1-r)(1+r) (2 x f32), id (i32)                       -> 60 B / vertex
#   count pass writes a degree per vertex                     ->  4 B / vertex
#   write pass reads a row offset per vertex and writes the CSR -> 8 B / vertex + 4 B / entry
POINT_RECORD_B = 60


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--vertex-order", default="sample", choices=("sample", "angular"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=100_000,
                    help="query vertices per CPU-baseline step (bounded sample)")
    ap.add_argument("--n", type=int, default=None, help="override the config's n")
    ap.add_argument("--k", type=float, default=None, help="override the config's avg degree")
    ap.add_argument("--gamma", type=float, default=None, help="override the config's gamma")
    ap.add_argument("--seed", type=int, default=None, help="override the config's seed")
    ap.add_argument("--sweep", action="store_true",
                    help="config 4: one line per (k, gamma) point of the density/exponent "
                         "sweep at n=1e7, seed 4 (evidence runs, not the driver's line)")
    ap.add_argument("--dry-run", action="store_true",
                    help="print each rank's shard plan without GPU work (launcher test)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the whole-graph CPU reference run and edge-set comparison")
    ap.add_argument("--shard-sim", type=int, default=0, metavar="N",
                    help="time each of N angular shards in turn on this one GPU and report "
                         "the per-shard times and their max (stand-in for an N-GPU run)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, val in zip(names, r[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_reference_step(params, model, consts, n_queries, nthreads):
    """The reference algorithm (oracle's polar-quadtree restatement, hrgen
    quadtree.py) on the host: sample all points, build the tree over all of
    them, answer a bounded sample of the vertex queries; returns the
    extrapolated whole-graph edges/s and the pieces."""
    from oracle import oracle as O
    n = model.n
    t0 = time.perf_counter()
    u1, u2 = O.philox_uniforms(n, params["seed"])
    phi, rn, rp = O.sample_from_uniforms(u1, u2, consts["two_over_alpha"],
                                         consts["sinh_half_alpha_r"], consts["r_cap"],
                                         consts["rp_cap"])
    t_sample = time.perf_counter() - t0
    nq = min(n, n_queries)
    # a contiguous id range is a uniform sample of positions (ids are i.i.d.)
    _, m_part, tm = O.edges_quadtree(phi, rp, consts["cosh_r_minus_1"], model.alpha,
                                     consts["max_r"], 512, O.TRIG_LIBM, nthreads, 0, nq,
                                     want_pairs=False)
    frac = nq / n
    # m_part counts edges (v, w>v) found from the sampled v; the expected
    # share of all m found from a uniform fraction f of query vertices is f
    m_est = m_part / frac
    t_est = t_sample + tm.t_build_s + tm.t_query_s / frac
    return m_est / t_est, dict(t_sample_s=t_sample, t_build_s=tm.t_build_s,
                               t_query_sample_s=tm.t_query_s, queries=nq, m_est=m_est)


def cpu_reference_whole(params, model, consts, phi, rp, nthreads, want_pairs):
    """The reference algorithm on the host for the WHOLE graph, no
    extrapolation: the oracle's Philox sampler + hrgen's inverse CDF for all
    n points (timed, as hrgen samples its own points), then the polar
    quadtree (hrgen quadtree.py build/pack/query_many, libm trig) over the
    GPU's coordinates -- same point set as the GPU run, so its edge set is
    the parity reference -- with every vertex queried."""
    from oracle import oracle as O
    n = model.n
    t0 = time.perf_counter()
    u1, u2 = O.philox_uniforms(n, params["seed"])
    O.sample_from_uniforms(u1, u2, consts["two_over_alpha"], consts["sinh_half_alpha_r"],
                           consts["r_cap"], consts["rp_cap"])
    t_sample = time.perf_counter() - t0
    del u1, u2
    pairs, m, tm = O.edges_quadtree(phi, rp, consts["cosh_r_minus_1"], model.alpha,
                                    consts["max_r"], 512, O.TRIG_LIBM, nthreads,
                                    want_pairs=want_pairs)
    t = t_sample + tm.t_build_s + tm.t_query_s
    return m / t, pairs, dict(t_sample_s=t_sample, t_build_s=tm.t_build_s,
                              t_query_s=tm.t_query_s, t_total_s=t, m=m)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_1501_03545_b200 as P
    params = config_params(args)
    gp = P.GeneratorParams(**params)
    model = gp.resolve()
    consts = P.model_constants(model.R, model.alpha)
    nthreads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_step(params, model, consts, args.cpu_queries, nthreads)
    vals, info = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, info = cpu_reference_step(params, model, consts, args.cpu_queries, nthreads)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = sorted(vals)[len(vals) // 2]
    sample = (f"hrgen polar-quadtree algorithm (oracle/hrg_oracle.c restatement, libm trig): "
              f"sample all {model.n} points + build the full tree + {info['queries']} vertex "
              f"queries per step, whole-graph time extrapolated linearly in queries")
    line = {
        "impl": "reference", "metric": metric_for(params), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(params, model, args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample, **{k: v for k, v in info.items()}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def config_block(params, model, args, world):
    return {
        "workload": f"config{args.config}: n={params['n']}, k={params['avg_degree']}, "
                    f"gamma={params['gamma']} (alpha={model.alpha}), T=0, seed {params['seed']}",
        "n": params["n"], "avg_degree": params["avg_degree"], "gamma": params["gamma"],
        "alpha": model.alpha, "R": model.R, "seed": params["seed"],
        "vertex_order": args.vertex_order,
        "l2": "no flush: per-step working set (point records + CSR) >> 126 MB L2",
        "parallelism": f"angular sectors x {world}" if world > 1 else "single GPU",
    }


def run_ours(args):
    import numpy as np
    import torch

    import paper_1501_03545_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    params = config_params(args)
    gp = P.GeneratorParams(**params, vertex_order=args.vertex_order)
    model = gp.resolve()
    order = P.generator.VERTEX_ORDERS[args.vertex_order]
    shard = P.Shard(rank, world) if world > 1 else None
    eng = P.get_engine(local)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        eng.generate(model, params["seed"], order, shard)
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    cand, nnz = 0, 0
    phases = {}
    l0 = eng.launches()
    for _ in range(args.steps):
        st = eng.generate(model, params["seed"], order, shard)
        cand, nnz = st.candidates, st.nnz
        for k in ("t_sample_ms", "t_sort_ms", "t_build_ms", "t_light_ms", "t_heavy_ms",
                  "t_compact_ms", "t_rowsort_ms", "t_edges_ms"):
            phases.setdefault(k, []).append(getattr(st, k))
        phases.setdefault("heavy_queries", []).append(st.heavy_queries)
    e1.record()
    torch.cuda.synchronize()
    launches = eng.launches() - l0  # this library's kernels only (CUB sort/scan not counted)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / max(args.steps, 1)

    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    tot = torch.tensor([nnz, cand], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms_max = float(t.item())
    nnz_all, cand_all = float(tot[0].item()), float(tot[1].item())
    m_total = nnz_all / 2.0
    value = m_total / (ms_max / 1e3)

    # ---- e2e: the C ABI with HOST buffers: hrg_generate + hrg_copy_result of
    # the step's result (int64 CSR, hrgen.Graph's dtype) into pinned host memory
    e2e = None
    if not args.no_e2e:
        # The C ABI with HOST buffers: hrg_generate + hrg_copy_result of the
        # step's result (int64 CSR, hrgen.Graph's dtype) into pinned host
        # memory.  Two generator contexts on their own streams, driven by two
        # host threads, alternate steps, so one graph's device->host copy (PCIe,
        # the bound) overlaps the next graph's generation; every step still
        # generates a graph and reads all of it back.
        import threading
        k2 = max(2, min(2 * args.steps, 8))
        n_, nnz_ = eng.sizes()
        streams = [torch.cuda.Stream(device=local) for _ in range(2)]
        # the timed engine is one of the two contexts (a third context's
        # buffers would not fit beside two at n = 1e8)
        eng.set_stream(streams[0].cuda_stream)
        engines = [eng, P.Engine(local, stream=streams[1].cuda_stream)]
        bufs = [(torch.empty(n_ + 1, dtype=torch.int64, pin_memory=True).numpy(),
                 torch.empty(int(nnz_ * 1.01) + 1024, dtype=torch.int64, pin_memory=True).numpy())
                for _ in range(2)]

        def one_step(w):
            e = engines[w]
            e.generate(model, params["seed"], order, shard)
            _, nz = e.sizes()
            e.copy_result_into(indptr=bufs[w][0], indices=bufs[w][1][:nz])
            return nz

        for w in range(2):  # warm both contexts (allocations, staging sizes)
            one_step(w)

        started = threading.Event()

        def worker(w, count, out):
            # context 1 starts once context 0's first graph is generated, so
            # the two alternate (generate one while the other's copy runs)
            # instead of generating and copying in lockstep
            if w == 1:
                started.wait()
            res_w = []
            for i in range(count):
                e = engines[w]
                e.generate(model, params["seed"], order, shard)
                if w == 0 and i == 0:
                    started.set()
                _, nz = e.sizes()
                e.copy_result_into(indptr=bufs[w][0], indices=bufs[w][1][:nz])
                res_w.append(nz)
            out[w] = res_w

        # sequential (one context) for reference
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k2):
            one_step(0)
        seq = (time.perf_counter() - t0) / k2
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = {}
        ths = [threading.Thread(target=worker, args=(w, k2 // 2, res)) for w in range(2)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        dt = torch.tensor([(time.perf_counter() - t0) / (2 * (k2 // 2))], dtype=torch.float64,
                          device="cuda")
        if dist is not None:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        d2h = (n_ + 1) * 8 + int(nnz_) * 8
        e2e = {"value": m_total / float(dt.item()), "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * float(dt.item()),
               "ms_per_step_one_context": 1e3 * seq,
               "api": "hrg_generate + hrg_copy_result (C ABI) into pinned host buffers, "
                      "int64 CSR (an adaptive 0-60% share of the ids is widened on the device "
                      "and copied as int64, the rest cross PCIe as int32 -- 3 bytes each when "
                      "n <= 2^24 -- and are widened into the caller's array by host threads, "
                      "with non-temporal stores, while the copies run; d2h_bytes_per_step "
                      "counts the int64 result); two contexts on two streams alternating steps (the copy "
                      "of one graph overlaps the generation of the next); inputs are 5 "
                      "scalar parameters"}
        del engines
        eng.set_stream(None)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel: the range query (light + heavy
    # launches), which reads every point record and writes every row once
    peak, peak_kind = load_peaks()
    med = {k: sorted(v)[len(v) // 2] for k, v in phases.items()}
    n_q = model.n / world
    tq = med["t_light_ms"] + med["t_heavy_ms"]
    bytes_query = model.n * POINT_RECORD_B + n_q * 12 + (nnz_all / world) * 4
    achieved = bytes_query / (tq / 1e3) / 1e9
    traffic, binding = None, None
    tpath = os.path.join(ROOT, "profiles", "query_write_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tj = json.load(fh)
            if tj.get("config") == args.config and tj.get("n_gpus", 1) == world:
                traffic = tj.get("dram_bytes_per_launch")
                # the resource that does bind the kernel (neither HBM nor FP64):
                # from the same committed ncu capture
                binding = tj.get("binding")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "kernel": "range query k_light + k_heavy (pair tests, hits to staging)",
                "algorithmic_bytes_per_launch": bytes_query, "launch_ms": tq,
                "fp64": {"pair_tests": cand_all / world, "flop_per_test": 6,
                         "tflops": cand_all / world * 6 / (tq / 1e3) / 1e12},
                "binding": binding}

    cpu, parity = None, None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import oracle as O
            consts = P.model_constants(model.R, model.alpha)
            nthreads = os.cpu_count() or 1
            # the graph the timed steps generated, read back with its coordinates
            with eng.lock:
                eng.generate(model, params["seed"], order, shard)
                ip, ix = eng.copy_csr(np.int64, pinned=False)
                phi, _, rp = eng.copy_coords()
            v, pairs, info = cpu_reference_whole(params, model, consts, phi, rp, nthreads,
                                                 want_pairs=not args.no_parity)
            v_est, est = cpu_reference_step(params, model, consts, args.cpu_queries, nthreads)
            cpu = {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port",
                   "sample": f"the whole graph, no extrapolation: oracle/hrg_oracle.c (hrgen's "
                             f"polar quadtree restated in C, libm trig) samples all {model.n} "
                             f"points, builds the tree and answers every vertex query on "
                             f"{nthreads} host threads",
                   **info,
                   "sampled_estimate": {"value": v_est, "queries": est["queries"],
                                        "how": "full tree + a bounded query sample, "
                                               "extrapolated linearly in queries"}}
            if pairs is not None:
                rows = np.repeat(np.arange(model.n, dtype=np.int64), np.diff(ip))
                keep = ix > rows
                got = np.column_stack((rows[keep], ix[keep]))
                del rows, keep, ix
                d = O.compare_edge_sets(got, pairs, phi, rp, model.R)
                cls = O.classify_mismatches(d, phi, rp, consts["cosh_r_minus_1"])
                parity = {"scope": "whole edge set", "ref": "oracle quadtree (hrgen "
                          "quadtree.py restated), libm trig = hrgen's arithmetic",
                          "m_gpu": d["m_got"], "m_ref": d["m_want"],
                          "mismatches": d["only_got"] + d["only_want"],
                          "max_rel_gap": d["max_gap"], "outside_band": d["outside_band"],
                          "in_band": cls["band"], "ref_pruning_drops": cls["ref_drop"],
                          "unexplained": cls["unexplained"],
                          "band": "|cosh d - cosh R| <= 1e-12 cosh R"}
                del got, pairs
        except Exception as e:  # pragma: no cover
            cpu = {"error": repr(e)}

    line = {
        "metric": metric_for(params), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(params, model, args, world),
        "m": m_total, "candidates": cand_all,
        "phases_ms": med,
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "clocks": clk,
        "gpu_launches": launches,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_shard_sim(args):
    """Stand-in for an N-GPU run on the one GPU a call gets: every shard of an
    N-way angular split is generated in turn (each after its own warm-up),
    timed with CUDA events; the N-GPU step time is the max over shards (the
    ranks share nothing but the final edge-count all-reduce)."""
    import torch

    import paper_1501_03545_b200 as P
    torch.cuda.set_device(0)
    params = config_params(args)
    gp = P.GeneratorParams(**params, vertex_order=args.vertex_order)
    model = gp.resolve()
    order = P.generator.VERTEX_ORDERS[args.vertex_order]
    eng = P.get_engine(0)
    N = args.shard_sim
    per, nnz_all = [], 0
    for k in range(N):
        shard = P.Shard(k, N) if N > 1 else None
        for _ in range(max(args.warmup, 0)):
            eng.generate(model, params["seed"], order, shard)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        phases = {}
        for _ in range(args.steps):
            st = eng.generate(model, params["seed"], order, shard)
            for key in ("t_sample_ms", "t_build_ms", "t_light_ms", "t_heavy_ms",
                        "t_compact_ms", "t_rowsort_ms", "t_edges_ms"):
                phases.setdefault(key, []).append(getattr(st, key))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / max(args.steps, 1)
        nnz_all += st.nnz
        per.append({"shard": k, "ms_per_step": ms, "nnz": st.nnz,
                    **{key: sorted(v)[len(v) // 2] for key, v in phases.items()}})
    ms_max = max(p["ms_per_step"] for p in per)
    line = {"metric": metric_for(params), "unit": UNIT, "simulated_n_gpus": N,
            "value": nnz_all / 2.0 / (ms_max / 1e3), "ms_per_step_max": ms_max,
            "steps": args.steps, "warmup": args.warmup, "m": nnz_all / 2.0,
            "config": config_block(params, model, args, N), "shards": per,
            "how": "each shard run in turn on one B200 (CUDA events per shard), "
                   "N-GPU step = max over shards"}
    print(json.dumps(line))
    return 0


def run_sweep(args):
    """BASELINE config 4: every (k, gamma) point at n=1e7, seed 4, one JSON
    line each (evidence runs; the driver's bench line is config 2)."""
    import subprocess as sp
    rc = 0
    for k, g in SWEEP:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", "4", "--k", str(k),
               "--gamma", str(g), "--steps", str(args.steps), "--warmup", str(args.warmup),
               "--no-cpu-baseline", "--no-e2e", "--vertex-order", args.vertex_order]
        rc |= sp.call(cmd)
    return rc


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_ranks(args):
    """`--gpus N` (N > 1) without a torchrun environment: re-run this script
    under torch.distributed.run with N ranks, one per GPU, rendezvous on
    127.0.0.1; rank 0 prints the line.  Returns the launcher's exit code."""
    port = os.environ.get("MASTER_PORT") or str(free_port())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dry_run(args):
    """--dry-run: the rank/shard plan each rank would run (no GPU work);
    exercised under gloo by tests/test_bench_launcher.py."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    plan = {"rank": rank, "world": world, "shard": [rank, world] if world > 1 else None,
            "config": config_params(args)}
    if world > 1:
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        dist.destroy_process_group()
    else:
        plans = [plan]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": plans}))
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    if args.dry_run:
        return dry_run(args)
    if args.sweep:
        return run_sweep(args)
    if args.shard_sim:
        return run_shard_sim(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
