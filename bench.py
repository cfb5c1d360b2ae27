#!/usr/bin/env python
"""bench.py -- throughput of the partitioned hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nacho|reference] [--workload c2|c5]

One step = one full pass of the hot path over the workload: partition (Alg. 1) +
the partitioned kernel(s).  Default workload: BASELINE.json configs[1] = C2, the 3-operand CSR
SpAdd A+B+C, 1M x 1M, 1e7 nnz each (a9-a11), metric GNNZ/s = Q*/time (Q* = sum of operand nnz).
The other configurations (C5 CSR SpMV, C3 DCSR SpMV, C4 SpMM, C1 fp64 SpMV) are measured in the
same run and reported under "kernels".  Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (oracle/, single-threaded C) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GNNZ/s (3-way CSR SpAdd A+B+C on C2: partition + assembly + compute), % of HBM roofline"
METRIC_C5 = "GNNZ/s (CSR SpMV y = A x on C5: partition + SpMV + carry fix-up), % of HBM roofline"
NOMINAL_HBM_GBS = 8000.0   # north_star's "about 8 TB/s" (the roofline is also reported against it)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nacho", choices=["nacho", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--quick", action="store_true", help="skip the secondary configurations")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_table():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}", "--format=csv,noheader",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1].split()[0]))
                mx = max(mx, float(r[2].split()[0]))
                for n, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ timing helpers
class Timer:
    """CUDA events on the launching stream; per-step times with an untimed L2 flush between steps."""

    def __init__(self, torch, flush_bytes):
        self.torch = torch
        self.flush = torch.empty(flush_bytes // 4, dtype=torch.float32, device="cuda")

    def flush_l2(self):
        self.flush.zero_()

    def run(self, step, K, W, sections=None, soak_s=0.0):
        t = self.torch
        for _ in range(W):
            self.flush_l2()
            step()
        t.cuda.synchronize()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < soak_s:   # untimed: keeps the GPU busy under the clock sampler
            for _ in range(20):
                self.flush_l2()
                step()
            t.cuda.synchronize()
        times = []
        sec = {}
        for _ in range(K):
            self.flush_l2()
            ev = [t.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            marks = step(timed=True) if sections else step()
            ev[1].record()
            times.append((ev, marks))
        t.cuda.synchronize()
        out = [e[0].elapsed_time(e[1]) for e, _ in times]
        if sections:
            for _, marks in times:
                for i, name in enumerate(sections):
                    sec.setdefault(name, []).append(marks[i].elapsed_time(marks[i + 1]))
        return out, sec


def ev(torch):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


# ------------------------------------------------------------------ workloads
def spadd_algo_bytes(ops, nnz_z):
    """Algorithmic bytes of one k-way SpAdd: every operand's crd / val once, every
    distinct row-pointer array once (C2's operands share one pos array), Z written once."""
    vs = ops[0].val.element_size()
    M = ops[0].nrows
    pos_arrays = {A.pos.data_ptr() for A in ops}
    return (sum(A.nnz * (4 + vs) for A in ops) + len(pos_arrays) * (M + 1) * 8
            + nnz_z * (4 + vs) + (M + 1) * 8)


def bench_spadd(N, W, torch, args, timer, world, rank):
    wl = W.build("c2", args.scale, device="cuda")
    ops = wl.ops
    k = len(ops)
    M = ops[0].nrows
    nnz = [A.nnz for A in ops]
    qstar = sum(nnz)
    P = N.auto_partitions(ops, "spadd")
    parts = N.Parts(P, k, ops[0].pos.device)
    local = parts
    part_off = torch.empty(local.P + 1, dtype=torch.int64, device="cuda")
    arr = N._matrices(ops)
    ws = torch.empty(max(N.lib.nacho_spadd_k_workspace_size(arr, k, local.P),
                         N.lib.nacho_spadd_k_staged_workspace_size(arr, k, local.P)), dtype=torch.uint8, device="cuda")
    z_pos = torch.empty(M + 1, dtype=torch.int64, device="cuda")
    z_crd = torch.empty(qstar, dtype=torch.int32, device="cuda")   # capacity Q* >= nnz_Z (no host sync)
    z_val = torch.empty(qstar, dtype=ops[0].val.dtype, device="cuda")

    def make_step(staged):
        def step(timed=False):
            m = [ev(torch)] if timed else None
            N.partition(ops, P, out=parts)
            if timed:
                m.append(ev(torch))
            if staged:   # one read, no look-back: staged union -> scan -> placement
                N.spadd_k_staged(ops, local, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
            else:        # one read, decoupled look-back
                N.spadd_k_fused(ops, local, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
            if timed:
                m.append(ev(torch))
            return m
        return step

    def step2(timed=False):  # the paper's two-pass assembly (count -> scan -> fill), for comparison
        m = [ev(torch)] if timed else None
        N.partition(ops, P, out=parts)
        if timed:
            m.append(ev(torch))
        N.spadd_k_count(ops, local, part_off, ws)
        if timed:
            m.append(ev(torch))
        N.spadd_k_fill(ops, local, part_off, qstar, z_pos, z_crd, z_val)
        if timed:
            m.append(ev(torch))
        return m

    # the single-read variants: a short trial picks the faster one for the timed run
    trial = {}
    for name, staged in (("spadd_fused", False), ("spadd_staged", True)):
        tt, _ = timer.run(make_step(staged), 5, 2)
        trial[name] = statistics.median(tt)
    best = min(trial, key=trial.get)
    step = make_step(best == "spadd_staged")
    sections = ["partition", best]
    # CUDA graphs: the partition and the SpAdd calls captured once and replayed, so the host-side
    # argument marshalling of the binding does not gap the device timeline between steps
    launch_mode = "eager"
    try:
        g_part, g_sp = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        staged_best = best == "spadd_staged"
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            make_step(staged_best)()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        N.launch_count(reset=True)
        with torch.cuda.graph(g_part):
            N.partition(ops, P, out=parts)
        with torch.cuda.graph(g_sp):
            if staged_best:
                N.spadd_k_staged(ops, local, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
            else:
                N.spadd_k_fused(ops, local, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
        torch.cuda.synchronize()
        graph_launches = N.launch_count(reset=True)   # kernels (and memsets) captured per step

        def step(timed=False):
            m = [ev(torch)] if timed else None
            g_part.replay()
            if timed:
                m.append(ev(torch))
            g_sp.replay()
            if timed:
                m.append(ev(torch))
            return m
        launch_mode = "cuda_graph"
    except Exception as e:  # capture unsupported: eager launches (same kernels)
        print(f"# cuda graph capture failed ({e}); eager launches", file=sys.stderr)
        step = make_step(best == "spadd_staged")
    t2, sec2 = timer.run(step2, 5, 2, ["partition", "count+scan", "fill"])
    step()
    torch.cuda.synchronize()
    N.launch_count(reset=True)
    step()
    launches = N.launch_count(reset=True)
    if launch_mode == "cuda_graph":
        launches = graph_launches
    times, sec = timer.run(step, args.steps, args.warmup, sections, soak_s=1.0)
    nnz_z = int(part_off[-1].item())
    vs = ops[0].val.element_size()
    algo_step = spadd_algo_bytes(ops, nnz_z)
    fused_bytes = algo_step
    res = dict(work=qstar / world if world > 1 else qstar, times=times, sec=sec, launches=launches,
               algo_step=algo_step, nnz_z=nnz_z, P=P,
               kernel_bytes={best: fused_bytes, "partition": (P + 1) * (8 * k + 28)},
               variants_ms={kk: vv for kk, vv in trial.items()}, best=best,
               two_pass={"ms_per_step": statistics.mean(t2),
                         "sections_ms": {s: statistics.mean(v) for s, v in sec2.items()}},
               dtype="f32" if vs == 4 else "f64", wl=wl, parts=parts, launch=launch_mode)
    return res


def count_launches(N, torch, step):
    """Kernels (and memsets) the library issues in one step (its own launch counter)."""
    torch.cuda.synchronize()
    N.launch_count(reset=True)
    step()
    torch.cuda.synchronize()
    return N.launch_count(reset=True)


class Exchange:
    """The exchange step of the multi-GPU path: libnacho's NCCL calls (nacho_dist_*), or -- for
    one-GPU smoke runs of the N > 1 code path (NACHO_DIST_BACKEND=gloo, several ranks on one device,
    which NCCL refuses) -- the same data movement through torch.distributed."""

    def __init__(self, N, torch, backend):
        self.N, self.torch, self.backend = N, torch, backend
        import torch.distributed as td
        self.td = td
        self.world, self.rank = td.get_world_size(), td.get_rank()
        self.comm = N.Dist.from_process_group() if backend == "nccl" else None

    def broadcast(self, t, root=0):
        if self.comm:
            self.comm.broadcast(t, root)
        else:
            c = t.cpu()
            self.td.broadcast(c, src=root)
            t.copy_(c)

    def spmv(self, A_loc, parts, x, y_loc, plans, y_full=None):
        N, torch = self.N, self.torch
        D = self.N_dist()
        if self.comm:
            return self.comm.spmv(A_loc, parts, x, y_loc, D.cut_rows(plans, plans[-1].row_lo + plans[-1].own),
                                  y_full=y_full)
        p = plans[self.rank]
        if p.nloc > 0:
            N.spmv(A_loc, x, parts, y=y_loc[:p.nloc])
        r, b = D.carry_of(p, y_loc)
        mine = torch.cat([r, b]).cpu()
        allc = [torch.empty_like(mine) for _ in range(self.world)]
        self.td.all_gather(allc, mine)
        if p.nloc > 0:
            N.dist_seam(torch.stack(allc).cuda().contiguous(), self.world, self.rank, p.row_lo, p.own > 0, y_loc)
        if y_full is not None:
            segs = [None] * self.world
            self.td.all_gather_object(segs, (p.row_lo, y_loc[:p.own].cpu()))
            for lo, seg in segs:
                y_full[lo:lo + len(seg)] = seg.to(y_full.device)
        return y_loc

    def spadd_gather(self, zp, zc, zv, nnz_dev, cut_rows, z_pos, z_crd, z_val):
        if self.comm:
            return self.comm.spadd_gather(zp, zc, zv, nnz_dev, cut_rows, z_pos, z_crd, z_val)
        torch = self.torch
        d = self.rank
        own = cut_rows[d + 1] - cut_rows[d]
        n = int(nnz_dev.item())
        pieces = [None] * self.world
        self.td.all_gather_object(pieces, (n, zp[1:own + 1].cpu(), zc[:n].cpu(), zv[:n].cpu()))
        base = 0
        z_pos[0] = 0
        for r, (nr, rows, c, v) in enumerate(pieces):
            z_pos[cut_rows[r] + 1:cut_rows[r] + 1 + len(rows)] = rows.to(z_pos.device) + base
            z_crd[base:base + nr] = c.to(z_crd.device)
            z_val[base:base + nr] = v.to(z_val.device)
            base += nr
        return base

    def N_dist(self):
        from paper_2604_17198_b200 import dist as D
        return D

    def close(self):
        if self.comm:
            self.comm.close()


def bench_spadd_dist(N, W, torch, args, timer, ex):
    """C2 on D devices: Alg. 1 with P = D gives the device cuts; each rank holds its
    operand shards (rows of its coordinate range, nacho_shard_rows) and runs its own partitions of them
    (partition + single-read SpAdd) -- timed, kernel-only; the exchange (nacho_dist_spadd_gather: union
    sizes -> offsets, Z segments gathered) is timed separately."""
    from paper_2604_17198_b200 import dist as D
    world, rank = ex.world, ex.rank
    wl = W.build("c2", args.scale, device="cuda")
    ops = wl.ops
    k = len(ops)
    M = ops[0].nrows
    qstar = sum(A.nnz for A in ops)
    dparts = N.partition(ops, world)
    sh, row_lo, own = D.spadd_shard_ops(ops, dparts, rank)
    cut_rows = [int(r) for r in dparts.row.cpu().tolist()]
    cut_rows[-1] = M
    P_l = N.auto_partitions(sh, "spadd")
    parts = N.Parts(P_l, k, "cuda")
    off = torch.empty(P_l + 1, dtype=torch.int64, device="cuda")
    cap = sum(A.nnz for A in sh)
    z_pos = torch.empty(sh[0].nrows + 1, dtype=torch.int64, device="cuda")
    z_crd = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    z_val = torch.empty(max(cap, 1), dtype=ops[0].val.dtype, device="cuda")
    ws = torch.empty(N.lib.nacho_spadd_k_workspace_size(N._matrices(sh), k, P_l), dtype=torch.uint8, device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.partition(sh, P_l, out=parts)
        if timed:
            m.append(ev(torch))
        N.spadd_k_fused(sh, parts, z_pos, z_crd, z_val, part_off=off, ws=ws)
        if timed:
            m.append(ev(torch))
        return m
    times, sec = timer.run(step, args.steps, args.warmup, ["partition", "spadd_fused"], soak_s=1.0)
    # the exchange step, timed separately (max over ranks by the caller's all-reduce of the median)
    zf_pos = torch.empty(M + 1, dtype=torch.int64, device="cuda")
    zf_crd = torch.empty(qstar, dtype=torch.int32, device="cuda")
    zf_val = torch.empty(qstar, dtype=ops[0].val.dtype, device="cuda")
    ex_ms = []
    nnz_z = 0
    for _ in range(3):
        ex.td.barrier()
        torch.cuda.synchronize()
        e0 = ev(torch)
        nnz_z = ex.spadd_gather(z_pos, z_crd, z_val, off[-1:], cut_rows, zf_pos, zf_crd, zf_val)
        e1 = ev(torch)
        torch.cuda.synchronize()
        ex_ms.append(e0.elapsed_time(e1))
    algo = spadd_algo_bytes(ops, nnz_z) / world
    return dict(work=qstar, times=times, sec=sec, launches=count_launches(N, torch, step), algo_step=algo,
                nnz_z=nnz_z, P=P_l * world, kernel_bytes={"spadd_fused": algo, "partition": (P_l + 1) * (8 * k + 28)},
                two_pass={}, dtype="f32", wl=wl, exchange_ms=statistics.median(ex_ms), best="spadd_fused",
                shard={"rows": [row_lo, row_lo + own], "entries": cap})


def bench_spmv_dist(N, W, torch, args, timer, ex):
    """C5 on D devices: every rank builds only its shard (device cuts from the row pointers,
    nacho_device_cuts; its entries generated in place), x broadcast at setup (timed separately); timed:
    the rank's partition + nacho_dist_spmv (local SpMV + seam-carry all-gather + fix-up); the gather of
    the owned y segments is timed separately (exchange_ms)."""
    from paper_2604_17198_b200 import dist as D
    world, rank = ex.world, ex.rank
    t0 = time.perf_counter()
    A_loc, plans, cuts = D.spmv_setup("c5", args.scale, world, rank)
    M = plans[-1].row_lo + plans[-1].own
    nnz_total = int(cuts[-1][1])
    x = W.dense_x("c5", args.scale) if rank == 0 else torch.empty(M, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ex.td.barrier()
    e0 = ev(torch)
    ex.broadcast(x, 0)
    e1 = ev(torch)
    torch.cuda.synchronize()
    bcast_ms = e0.elapsed_time(e1)
    setup_s = time.perf_counter() - t0
    p = plans[rank]
    P_l = N.auto_partitions([A_loc], "spmv")
    parts = N.Parts(P_l, 1, "cuda")
    y_loc = torch.empty(max(p.nloc, 1), dtype=torch.float32, device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.partition([A_loc], P_l, out=parts)
        if timed:
            m.append(ev(torch))
        ex.spmv(A_loc, parts, x, y_loc, plans)
        if timed:
            m.append(ev(torch))
        return m
    times, sec = timer.run(step, args.steps, args.warmup, ["partition", "spmv+seam"], soak_s=1.0)
    y_full = torch.empty(M, dtype=torch.float32, device="cuda")
    gx = []
    for _ in range(3):
        ex.td.barrier()
        torch.cuda.synchronize()
        e0 = ev(torch)
        ex.spmv(A_loc, parts, x, y_loc, plans, y_full=y_full)
        e1 = ev(torch)
        torch.cuda.synchronize()
        gx.append(e0.elapsed_time(e1))
    nnz = A_loc.nnz
    algo = nnz * 8 + (p.nloc + 1) * 8 + p.nloc * 4 + M * 4
    return dict(work=nnz_total, times=times, sec=sec, launches=count_launches(N, torch, step), algo_step=algo,
                nnz_z=0, P=P_l * world,
                kernel_bytes={"spmv+seam": algo, "partition": (P_l + 1) * 36}, two_pass={}, dtype="f32", wl=None,
                exchange_ms=statistics.median(gx) - statistics.median(sec["spmv+seam"]),
                shard={"rows": [p.row_lo, p.row_lo + p.own], "entries": nnz}, setup={"x_broadcast_ms": bcast_ms,
                                                                                     "setup_s": setup_s})


def e2e_spadd(N, torch, wl, args, staged):
    """Same metric through the public API, end to end: every step copies the three operands from pinned
    host memory to the device, runs partition + SpAdd, and copies Z (pos, crd, val) back into pinned
    host buffers (one 8-byte read of nnz_Z first: the only host sync per step).  Steps are pipelined
    over two streams and double-buffered inputs: step i+1's H2D copies run on their own stream while
    step i computes and copies Z back (PCIe is full duplex; the copy engines work in parallel)."""
    # one pinned host copy per distinct array: C2's operands share one row-pointer array (same row
    # profile), which is copied once per step, as a user holding the three matrices would
    uniq = {}
    for A in wl.ops:
        for t in (A.pos, A.crd, A.val):
            if t.data_ptr() not in uniq:
                uniq[t.data_ptr()] = t.cpu().pin_memory()
    host = [list(uniq.values())]
    import workloads as W
    dev = []
    for _ in range(2):
        dmap = {k: torch.empty_like(t, device="cuda") for k, t in uniq.items()}
        dev.append([[dmap[k] for k in uniq]])
    keys = list(uniq)
    opsb = [[W.SparseMatrix("csr", A.nrows, A.ncols, db[0][keys.index(A.pos.data_ptr())],
                            db[0][keys.index(A.crd.data_ptr())], db[0][keys.index(A.val.data_ptr())])
             for A in wl.ops] for db in dev]
    h2d = sum(t.numel() * t.element_size() for t in uniq.values())
    ops = opsb[0]
    P = N.auto_partitions(ops, "spadd")
    parts = N.Parts(P, len(ops), "cuda")
    qstar = sum(A.nnz for A in ops)
    M = ops[0].nrows
    z_pos = torch.empty(M + 1, dtype=torch.int64, device="cuda")
    z_crd = torch.empty(qstar, dtype=torch.int32, device="cuda")
    z_val = torch.empty(qstar, dtype=ops[0].val.dtype, device="cuda")
    part_off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
    arr = N._matrices(ops)
    wsz = (N.lib.nacho_spadd_k_staged_workspace_size(arr, len(ops), P) if staged
           else N.lib.nacho_spadd_k_workspace_size(arr, len(ops), P))
    ws = torch.empty(wsz, dtype=torch.uint8, device="cuda")
    h_pos = torch.empty(M + 1, dtype=torch.int64).pin_memory()
    h_crd = torch.empty(qstar, dtype=torch.int32).pin_memory()
    h_val = torch.empty(qstar, dtype=ops[0].val.dtype).pin_memory()
    h_nnz = torch.empty(1, dtype=torch.int64).pin_memory()
    s_in, s_c = torch.cuda.Stream(), torch.cuda.current_stream()
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    moved = {}

    def h2d_copy(i):   # inputs of step i into buffer i % 2, on the copy-in stream
        with torch.cuda.stream(s_in):
            for h, d in zip(host, dev[i % 2]):
                for a, b in zip(h, d):
                    b.copy_(a, non_blocking=True)
            ev_in[i % 2].record(s_in)

    def compute_and_d2h(i):
        s_c.wait_event(ev_in[i % 2])
        o = opsb[i % 2]
        N.partition(o, P, out=parts)
        if staged:
            N.spadd_k_staged(o, parts, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
        else:
            N.spadd_k_fused(o, parts, z_pos, z_crd, z_val, part_off=part_off, ws=ws)
        h_nnz.copy_(part_off[P:], non_blocking=True)
        s_c.synchronize()
        nz = int(h_nnz[0])
        h_pos.copy_(z_pos, non_blocking=True)
        h_crd[:nz].copy_(z_crd[:nz], non_blocking=True)
        h_val[:nz].copy_(z_val[:nz], non_blocking=True)
        moved["d2h"] = 8 + (M + 1) * 8 + nz * (4 + z_val.element_size())

    def run(nsteps):
        h2d_copy(0)
        for i in range(nsteps):
            # buffer (i+1) % 2 was last read by step i-1, whose compute finished before its nnz read
            if i + 1 < nsteps:
                h2d_copy(i + 1)
            compute_and_d2h(i)
        torch.cuda.synchronize()

    run(max(2, args.warmup))
    K = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    run(K)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    return {"value": qstar / (ms * 1e-3) / 1e9, "unit": "GNNZ/s", "ms_per_step": ms, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": moved["d2h"], "wall_ms_per_step": (time.perf_counter() - t0) * 1e3 / K,
            "path": "pinned H2D (stream 2, next step) || partition -> " + ("staged" if staged else "fused")
                    + " SpAdd -> pinned D2H"}


def bench_spmv(N, W, torch, name, scale, K, Wu, timer, column_kind=None):
    wl = W.build(name, scale, device="cuda", column_kind=column_kind)
    A = wl.ops[0]
    P = wl.P or N.auto_partitions([A], "spmv")
    parts = N.Parts(P, 1, "cuda")
    n_y = A.nrows if A.format == "csr" else A.nouter
    y = torch.empty(n_y, dtype=A.val.dtype, device="cuda")
    ws = torch.empty(N.lib.nacho_spmv_workspace_size(__import__("ctypes").byref(N.matrix(A)), P), dtype=torch.uint8,
                     device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.partition([A], P, out=parts)
        if timed:
            m.append(ev(torch))
        N.spmv(A, wl.x, parts, y=y, ws=ws)
        if timed:
            m.append(ev(torch))
        return m

    times, sec = timer.run(step, K, Wu, ["partition", "spmv+fixup"])
    vs = A.val.element_size()
    M, Nc, nnz = A.nrows, A.ncols, A.nnz
    if A.format == "csr":
        algo = nnz * (4 + vs) + (M + 1) * 8 + M * vs + Nc * vs
    else:
        distinct = int(torch.unique(A.crd).numel())
        algo = nnz * (4 + vs) + A.nouter * (4 + 8) + distinct * vs + A.nouter * vs
    out = dict(work=nnz, times=times, sec=sec, algo_step=algo, kernel_bytes={"spmv+fixup": algo}, P=P,
               dtype="f32" if vs == 4 else "f64", wl=wl)
    if A.format != "csr":
        # gather-granularity bound (uniform random columns over a 400 MB x: every gather moves a
        # 32-byte DRAM sector): crd + val once, the row level, one sector per nonzero
        out["gather_bytes"] = nnz * (4 + vs) + A.nouter * 16 + nnz * 32
    return out


def bench_intersection(N, W, torch, scale, K, Wu, timer):
    """C2's three operands coiterated as an intersection: partition + Hadamard
    A (.) B (.) C (nacho_hadamard_k), and the intersect-reduce inner product (nacho_inner_k)."""
    wl = W.build("c2", scale, device="cuda")
    ops = wl.ops
    k = len(ops)
    P = N.auto_partitions(ops, "spadd")
    parts = N.Parts(P, k, "cuda")
    cap = min(A.nnz for A in ops)
    z_pos = torch.empty(ops[0].nrows + 1, dtype=torch.int64, device="cuda")
    z_crd = torch.empty(cap, dtype=torch.int32, device="cuda")
    z_val = torch.empty(cap, dtype=torch.float32, device="cuda")
    ws = torch.empty(N.lib.nacho_inner_k_workspace_size(N._matrices(ops), k, P), dtype=torch.uint8, device="cuda")
    res = torch.empty(1, dtype=torch.float64, device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.partition(ops, P, out=parts)
        if timed:
            m.append(ev(torch))
        N.hadamard_k(ops, parts, z_pos, z_crd, z_val, ws=ws)
        if timed:
            m.append(ev(torch))
        N.inner_k(ops, parts, out=res, ws=ws)
        if timed:
            m.append(ev(torch))
        return m
    times, sec = timer.run(step, K, Wu, ["partition", "hadamard", "inner"])
    nnz_z = int(z_pos[-1].item())
    M = ops[0].nrows
    pos_arrays = {A.pos.data_ptr() for A in ops}
    read = sum(A.nnz * 8 for A in ops) + len(pos_arrays) * (M + 1) * 8
    return dict(work=sum(A.nnz for A in ops), times=times, sec=sec, algo_step=2 * read + nnz_z * 8 + (M + 1) * 8,
                kernel_bytes={"hadamard": read + nnz_z * 8 + (M + 1) * 8, "inner": read,
                              "partition": (P + 1) * (8 * k + 28)}, P=P, dtype="f32", wl=wl, nnz_z=nnz_z)


def bench_recursive(N, W, torch, scale, K, Wu, timer):
    """Recursive partitioning (Alg. 2) on C3-shaped DCSR operands: A = C3, B = the rows of A kept with
    probability 1/2 (doubled values); one step = nacho_dcsr_hadamard (outer partition, surviving rows,
    T' prefix sum, remapped partition, assembly, compute).  Thread-per-partition kernels (Listing 8's
    shape): a coverage line, not a tuned one."""
    wl = W.build("c3", scale, device="cuda")
    A = wl.ops[0]
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    keep = torch.rand(A.nouter, device="cuda", generator=g) < 0.5
    lens = A.pos[1:] - A.pos[:-1]
    sel = torch.repeat_interleave(keep, lens)
    bpos = torch.zeros(int(keep.sum().item()) + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(lens[keep], 0, out=bpos[1:])
    B = W.SparseMatrix("dcsr", A.nrows, A.ncols, bpos, A.crd[sel].contiguous(), (A.val[sel] * 2).contiguous(),
                       A.outer_crd[keep].contiguous())
    ops = [A, B]
    P = max(1, -(-(A.nnz + B.nnz) // 512))

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.dcsr_hadamard(ops, P)
        if timed:
            m.append(ev(torch))
        return m
    times, sec = timer.run(step, K, Wu, ["dcsr_hadamard"])
    read = (A.nnz + B.nnz) * 8 + (A.nouter + B.nouter) * 12
    return dict(work=A.nnz + B.nnz, times=times, sec=sec, algo_step=read, kernel_bytes={"dcsr_hadamard": read}, P=P,
                dtype="f32", wl=wl)


def bench_spmm(N, W, torch, scale, K, Wu, timer):
    wl = W.build("c4", scale, device="cuda")
    A = wl.ops[0]
    P = N.auto_partitions([A], "spmm")
    parts = N.Parts(P, 1, "cuda")
    C = torch.empty(A.nrows, wl.nb, dtype=A.val.dtype, device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N.partition([A], P, out=parts)
        if timed:
            m.append(ev(torch))
        N.spmm(A, wl.x, parts, C=C)
        if timed:
            m.append(ev(torch))
        return m

    times, sec = timer.run(step, K, Wu, ["partition", "spmm+fixup"])
    M, Nc, nnz, nb = A.nrows, A.ncols, A.nnz, wl.nb
    algo = nnz * 8 + (M + 1) * 8 + Nc * nb * 4 + M * nb * 4
    # gather-granularity bound: one B row (nb * 4 bytes) per nonzero (B is 50x the L2, and 3/4 of the
    # columns are uniform over it), plus A once and C once
    gather = nnz * 8 + (M + 1) * 8 + nnz * nb * 4 + M * nb * 4
    return dict(work=nnz, times=times, sec=sec, algo_step=algo, kernel_bytes={"spmm+fixup": algo}, P=P, dtype="f32",
                wl=wl, gather_bytes=gather)


def bench_esc(N, W, torch, scale, K, Wu, timer, sampled=False):
    """ESC scatter kernels on C2's operands: SpGEMM C = A B (A, B = C2's first two
    operands), or with sampled=True the sampled SpGEMM Z = S (.) (A B) with S = C2's third operand.
    One step = work W (Listing 6's cost) + partition of the expansion + expand / sort / contract
    (sampled: + the count pass).  Work unit: products of the expansion (Q*).  Q* and the sampled count
    are read once at setup (they size the buffers), not inside the timed steps."""
    wl = W.build("c2", scale, device="cuda")
    A, B, S = wl.ops
    M = A.nrows
    Wd = N.spgemm_work(A, B)
    qstar = int(Wd[-1].item())
    P = N.esc_auto_partitions(qstar)
    parts = N.partition_esc(A, B, Wd, qstar, P)
    sa, aa, ba = N.matrix(S), N.matrix(A), N.matrix(B)
    import ctypes
    if sampled:
        part_off = torch.empty(P + 1, dtype=torch.int64, device="cuda")
        mask = torch.empty(N.lib.nacho_sssmm_mask_bytes(qstar, P), dtype=torch.uint8, device="cuda")
        cws = torch.empty(max(1, N.lib.nacho_sssmm_count_workspace_size(P)), dtype=torch.uint8, device="cuda")
        pc = parts.c()
        N._check(N.lib.nacho_sssmm_esc_count(ctypes.byref(sa), ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd),
                                             ctypes.byref(pc), N._ptr(part_off), N._ptr(mask), N._ptr(cws),
                                             cws.numel(), None))
        n = int(part_off[-1].item())
    else:
        n = qstar
    need = (N.lib.nacho_sssmm_esc_workspace_size if sampled else N.lib.nacho_spgemm_esc_workspace_size)(
        ctypes.byref(aa), ctypes.byref(ba), n)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    wws = torch.empty(max(1, N.lib.nacho_spgemm_work_workspace_size(ctypes.byref(aa))), dtype=torch.uint8, device="cuda")
    c_pos = torch.empty(M + 1, dtype=torch.int64, device="cuda")
    c_crd = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    c_val = torch.empty(max(n, 1), dtype=torch.float32, device="cuda")
    nnz_c = torch.empty(1, dtype=torch.int64, device="cuda")

    def step(timed=False):
        m = [ev(torch)] if timed else None
        N._check(N.lib.nacho_spgemm_work(ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd), N._ptr(wws), wws.numel(), None))
        if timed:
            m.append(ev(torch))
        pc = parts.c()
        N._check(N.lib.nacho_partition_esc(ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd), qstar, P, ctypes.byref(pc),
                                           None))
        if timed:
            m.append(ev(torch))
        if sampled:
            N._check(N.lib.nacho_sssmm_esc_count(ctypes.byref(sa), ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd),
                                                 ctypes.byref(pc), N._ptr(part_off), N._ptr(mask), N._ptr(cws),
                                                 cws.numel(), None))
            if timed:
                m.append(ev(torch))
            N._check(N.lib.nacho_sssmm_esc(ctypes.byref(sa), ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd),
                                           ctypes.byref(pc), N._ptr(part_off), N._ptr(mask), n, N._ptr(c_pos),
                                           N._ptr(c_crd),
                                           N._ptr(c_val), N._ptr(nnz_c), N._ptr(ws), need, None))
        else:
            N._check(N.lib.nacho_spgemm_esc(ctypes.byref(aa), ctypes.byref(ba), N._ptr(Wd), ctypes.byref(pc), qstar,
                                            N._ptr(c_pos), N._ptr(c_crd), N._ptr(c_val), N._ptr(nnz_c), N._ptr(ws),
                                            need, None))
        if timed:
            m.append(ev(torch))
        return m
    secs = ["work", "partition"] + (["count", "fill+sort+contract"] if sampled else ["expand+sort+contract"])
    times, sec = timer.run(step, K, Wu, secs)
    nnz_out = int(nnz_c.item())
    io = A.nnz * 8 + (M + 1) * 8 + B.nnz * 8 + (B.nrows + 1) * 8 + nnz_out * 8 + (M + 1) * 8
    esc = io + 24 * n + (S.nnz * 8 + (M + 1) * 8 if sampled else 0)   # + the expansion written and read once
    return dict(work=qstar, times=times, sec=sec, algo_step=esc, kernel_bytes={secs[-1]: esc, "work": A.nnz * 12,
                "partition": (P + 1) * 44, "count": A.nnz * 8}, P=P, dtype="f32", wl=wl, n_products=qstar,
                n_kept=n, nnz_out=nnz_out)


def summarize(r, peak, world=1):
    ms = statistics.mean(r["times"])
    dom = max(r["sec"], key=lambda s: statistics.mean(r["sec"][s]))
    dms = statistics.mean(r["sec"][dom])
    achieved = r["kernel_bytes"][dom] / (dms * 1e-3) / 1e9
    out = {"gnnz_s": r["work"] * world / (ms * 1e-3) / 1e9, "ms_per_step": ms,
           "step_hbm_frac": r["algo_step"] / (ms * 1e-3) / 1e9 / peak,
           "sections_ms": {s: statistics.mean(v) for s, v in r["sec"].items()},
           "dominant": dom, "dominant_achieved_gbs": achieved, "P": r["P"]}
    return out, dom, dms, achieved


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def oracle_spadd_once(O, host_ops, P):
    t0 = time.perf_counter()
    O.partition_rank(host_ops, P)
    O.spadd_k(host_ops)
    return time.perf_counter() - t0


def host_info():
    """CPU model, logical CPUs and RAM of the machine the oracle runs on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": ram}


class pinned_core:
    """Runs the single-threaded oracle pinned to one host core (SURVEY 8(d) 'Timing (oracle)')."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.old)


def cpu_baseline(host_ops, P, budget_s=20.0):
    import oracle as O
    O.lib()
    qstar = sum(A.nnz for A in host_ops)
    ts = []
    with pinned_core() as pc:
        t_start = time.perf_counter()
        while len(ts) < 3 or (time.perf_counter() - t_start < budget_s * 0.5 and len(ts) < 14):
            ts.append(oracle_spadd_once(O, host_ops, P))
            if time.perf_counter() - t_start > budget_s:
                break
    med = statistics.median(ts)
    return {"value": qstar / med / 1e9, "unit": "GNNZ/s", "cores": 1, "kind": "oracle", "pinned_core": pc.core,
            "host": host_info(),
            "sample": f"full C2 workload (3 x {host_ops[0].nnz} nnz, P={P}): oracle partition_rank + spadd_k, "
                      f"median of {len(ts)} runs on 1 pinned host core, {med:.3f} s each"}


def cpu_baseline_spmv(A, x, P, budget_s=20.0, max_rows=None):
    """The oracle's SpMV (partition_rank + spmv) on a row-block sample of a large matrix (host RAM and
    run time bound the sample; 'stream A in row blocks and time only the compute')."""
    import oracle as O
    import workloads as W
    O.lib()
    pos = A.pos.cpu().numpy()
    M = A.nrows
    # the first rows holding ~2e8 entries (the whole matrix when it is smaller)
    target = min(int(pos[-1]), 200_000_000)
    r1 = int(np.searchsorted(pos, target, side="left"))
    r1 = max(1, min(M, r1 if max_rows is None else min(r1, max_rows)))
    lo, hi = 0, int(pos[r1])
    sub = W.SparseMatrix("csr", r1, A.ncols, pos[: r1 + 1] - lo, A.crd[lo:hi].cpu().numpy(),
                         A.val[lo:hi].cpu().numpy())
    xs = x.cpu().numpy()
    ts = []
    with pinned_core() as pc:
        t_start = time.perf_counter()
        while len(ts) < 3 and time.perf_counter() - t_start < budget_s:
            t0 = time.perf_counter()
            O.partition_rank([sub], max(1, P * (hi - lo) // max(1, int(pos[-1]))))
            O.spmv(sub, xs)
            ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    return {"value": (hi - lo) / med / 1e9, "unit": "GNNZ/s", "cores": 1, "kind": "oracle", "pinned_core": pc.core,
            "host": host_info(),
            "sample": f"rows [0, {r1}) of the workload ({hi - lo} nnz of {int(pos[-1])}): oracle partition_rank + "
                      f"spmv, median of {len(ts)} runs on 1 pinned host core, {med:.3f} s each"}


def reference_partitions(host):
    """P the library would choose (nacho_auto_partitions reads only the descriptors' sizes)."""
    try:
        import torch
        import paper_2604_17198_b200 as N
        import workloads as W
        t = [W.SparseMatrix(A.format, A.nrows, A.ncols, torch.from_numpy(A.pos), torch.from_numpy(A.crd),
                            torch.from_numpy(A.val)) for A in host]
        return N.auto_partitions(t, "spadd")
    except Exception:   # library not built: the same rule (tile entries minus the pad and Theorem 1 slack)
        k = len(host)
        tile = 2048 - 7 * k - (k - 1)
        return max(1, -(-sum(A.nnz for A in host) // tile))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    import workloads as W
    O.lib()
    wl = W.build("c2", args.scale)
    host = wl.ops
    qstar = sum(A.nnz for A in host)
    P = reference_partitions(host)
    with pinned_core() as pc:
        for _ in range(args.warmup):
            oracle_spadd_once(O, host, P)
        ts = [oracle_spadd_once(O, host, P) for _ in range(args.steps)]
    ms = statistics.mean(ts) * 1e3
    v = qstar / (ms * 1e-3) / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GNNZ/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c2_spadd3_1Mx1M_3x1e7nnz", "scale": args.scale, "P": P},
            "cpu_baseline": {"value": v, "unit": "GNNZ/s", "cores": 1, "kind": "oracle", "pinned_core": pc.core,
                             "host": host_info(),
                             "sample": f"full C2 workload each step ({qstar} nnz), oracle partition_rank + spadd_k"},
            "e2e": {"value": v, "unit": "GNNZ/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ main
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_2604_17198_b200 as N
    import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())   # identity on a full node (one rank per GPU)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("NACHO_DIST_BACKEND", "nccl")   # gloo: CPU-side smoke runs on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    peak, peak_src = peaks()
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    timer = Timer(torch, max(2 * l2, 256 << 20))

    clocks = Clocks(local)
    ex = Exchange(N, torch, os.environ.get("NACHO_DIST_BACKEND", "nccl")) if world > 1 else None
    if args.workload == "c2":
        r = bench_spadd_dist(N, W, torch, args, timer, ex) if world > 1 else bench_spadd(N, W, torch, args, timer, 1, 0)
        metric, wname = METRIC, "c2_spadd3_1Mx1M_3x1e7nnz"
    else:
        if world > 1:
            r = bench_spmv_dist(N, W, torch, args, timer, ex)
        else:
            r = bench_spmv(N, W, torch, "c5", args.scale, args.steps, args.warmup, timer)
            r["launches"] = 3
        metric, wname = METRIC_C5, "c5_spmv_csr_f32_200Mx200M_4e9nnz"
    clk = clocks.stop()

    times = r["times"]
    ms_local = statistics.mean(times)
    ms = ms_local
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_local, r.get("exchange_ms") or 0.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        r["exchange_ms"] = float(t[1].item())
    summ, dom, dms, achieved = summarize(r, peak)
    tt = traffic_table().get(f"{args.workload}:{dom}") if world == 1 else None   # table holds single-GPU launches
    work = r["work"]
    line = {
        "metric": metric,
        "value": work / (ms * 1e-3) / 1e9,
        "unit": "GNNZ/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": r["dtype"], "data": "synthetic (seeded power-law CSR, workloads/ recipe)",
        "config": {"workload": wname, "scale": args.scale, "P": r["P"],
                   "l2": "flushed between timed steps (untimed memset of 2x L2)", "parallelism": f"dp{world}",
                   "launch": r.get("launch", "eager"),
                   **({"k": 3, "nnz_per_operand": r["wl"].ops[0].nnz, "nnz_Z": r["nnz_z"]}
                      if args.workload == "c2" and r.get("wl") is not None else {}),
                   **({"sharding": "device cuts = Alg. 1 with P = D; each rank holds and computes only its shard; "
                                   "value = kernel-only time (max over ranks); the output exchange is timed "
                                   "separately as exchange_ms", "exchange": ex.backend,
                       "shard_rank0": r.get("shard"), "setup": r.get("setup")} if world > 1 else {})},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "frac_nominal_8tbs": achieved / NOMINAL_HBM_GBS, "traffic": tt,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": r["kernel_bytes"][dom]},
        "step_roofline_frac": summ["step_hbm_frac"],
        "sections_ms": summ["sections_ms"],
        "two_pass": r.get("two_pass"),
        "single_read_variants_ms": r.get("variants_ms"),
        "exchange_ms": r.get("exchange_ms"),
        "end_to_end_ms": (ms + r["exchange_ms"]) if world > 1 else None,
        "gpu_launches": r["launches"] * args.steps,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_e2e and args.workload == "c2":
        line["e2e"] = e2e_spadd(N, torch, r["wl"], args, r.get("best") == "spadd_staged")
    if rank == 0 and world == 1 and not args.no_cpu:
        if args.workload == "c2":
            line["cpu_baseline"] = cpu_baseline([A.numpy() for A in r["wl"].ops], r["P"])
        else:
            line["cpu_baseline"] = cpu_baseline_spmv(r["wl"].ops[0], r["wl"].x, r["P"])
    if world > 1 and ex is not None:
        ex.close()
    wl_keep = r.pop("wl", None)
    del wl_keep, r
    torch.cuda.empty_cache()
    if not args.quick and world == 1 and args.workload == "c2":
        kern = {}
        for name, fn in [("c5_spmv_csr_f32", lambda: bench_spmv(N, W, torch, "c5", args.scale, 10, 3, timer)),
                         ("c3_spmv_dcsr_f32", lambda: bench_spmv(N, W, torch, "c3", args.scale, 10, 3, timer)),
                         ("c4_spmm_f32_nb64", lambda: bench_spmm(N, W, torch, args.scale, 5, 2, timer)),
                         ("c2_hadamard3_and_inner", lambda: bench_intersection(N, W, torch, args.scale, 10, 3, timer)),
                         ("c3_dcsr_hadamard_recursive", lambda: bench_recursive(N, W, torch, args.scale, 5, 2, timer)),
                         ("c2ops_spgemm_esc", lambda: bench_esc(N, W, torch, args.scale, 5, 2, timer)),
                         ("c2ops_sssmm_esc", lambda: bench_esc(N, W, torch, args.scale, 5, 2, timer, sampled=True)),
                         ("c1_spmv_csr_f64_P8", lambda: bench_spmv(N, W, torch, "c1", 1.0, 20, 3, timer))]:
            try:
                rr = fn()
                s, d, _, ach = summarize(rr, peak)
                if rr.get("gather_bytes"):
                    kern.setdefault(name, {})["gather_bound_frac"] = rr["gather_bytes"] / (
                        statistics.mean(rr["sec"][d]) * 1e-3) / 1e9 / peak
                kern[name] = {**kern.get(name, {}), "gnnz_s": s["gnnz_s"], "ms_per_step": s["ms_per_step"],
                              "step_hbm_frac": s["step_hbm_frac"], "dominant": d,
                              "dominant_hbm_frac": ach / peak, "dominant_frac_nominal_8tbs": ach / NOMINAL_HBM_GBS, "sections_ms": s["sections_ms"], "P": s["P"],
                              "traffic": traffic_table().get(f"{name.split('_')[0]}:{d}")}
                if "n_products" in rr:   # ESC lines: gnnz_s counts products of the expansion
                    kern[name].update(unit="G products/s", products=rr["n_products"], kept=rr["n_kept"],
                                      nnz_out=rr["nnz_out"])
                del rr
            except Exception as e:  # report, never hide
                kern[name] = {"error": repr(e)[:300]}
            torch.cuda.empty_cache()
        line["kernels"] = kern
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
