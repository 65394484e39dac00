#!/usr/bin/env python
"""Benchmark of the B200 divide-and-conquer sampler (arXiv 1610.05141).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--workload headline|cfg1|cfg0|complement|bernoulli|wr|gnm|algb]

One "step" = one pass of the whole hot path over one sample: the split tree,
the leaves and the stores, plus, for N > 1, the NCCL
all-gather of per-GPU counts.  Default workload: rs_sample_wor for
n = 2^32 per GPU from N = 2^48 (the north-star headline at N = 1; weak
scaling "n = p * 2^32" at N > 1), seed 1.  Inputs are three scalars, so they
are "resident" by construction; the 32 GiB output per GPU is far larger than
the 126 MB L2, so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0 (metric/value/unit/..., roofline, cpu_baseline,
e2e, clocks, gpu_launches).  --impl reference times the CPU oracle (the only
reference this tier has) on a bounded sample of the same workload.
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

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted samples/sec and output HBM GB/s vs peak at 1/2/4/8 B200"
RING_ELEMS = 2 * (2 ** 27 + 2 ** 21)     # e2e at N > 1: 2 batch slots (batches <= 2^27 values)
UNIT = "samples/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# per-GPU work fixed as N grows (weak) vs total work fixed (strong)
WEAK_WORKLOADS = ("headline", "weak30")


def _scaling(name):
    return "weak" if name in WEAK_WORKLOADS else "strong"


def _workload(name, world):
    from paper_1610_05141_b200 import workloads as W
    if name == "headline":
        n = world * W.HEADLINE["n"]
        wl = "wor_n2^32_N2^48" if world == 1 else f"weak_wor_n2^32perGPU_N2^48_p{world}"
        return dict(name=wl, mode="wor", N=W.HEADLINE["N"], n=n, seed=1)
    if name == "weak30":
        return dict(name=f"weak_wor_n2^30perGPU_N2^48_p{world}", mode="wor", N=2 ** 48,
                    n=world * 2 ** 30, seed=1)
    if name == "cfg1":
        return dict(W.CFG1)
    if name == "cfg0":
        return dict(W.CFG0)
    if name == "complement":
        return dict(W.CFG3A)
    if name == "bernoulli":
        return dict(W.CFG3B_ROOF)
    if name == "bernoulli32":
        return dict(W.CFG3B)
    if name == "wr":
        return dict(W.CFG4)
    if name == "gnm":
        return dict(W.GNM)
    if name == "algb":
        return dict(W.ALGB)
    raise SystemExit(f"unknown workload {name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu=timestamp,{self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is not None:
            time.sleep(0.12)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        try:
            self.f.seek(0)
            rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                r = [x.strip() for x in r]
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _merge_clocks(per_rank):
    """Rank 0's view of every rank's clock sample: the slowest rank's median,
    the union of throttle reasons, and the per-rank summaries."""
    per_rank = [c for c in per_rank if c]
    if not per_rank:
        return None
    if len(per_rank) == 1:
        return per_rank[0]
    meds = [c["sm_mhz"] for c in per_rank if c.get("sm_mhz") is not None]
    return {"sm_mhz": min(meds) if meds else None,
            "sm_max_mhz": max((c.get("sm_max_mhz") or 0) for c in per_rank) or None,
            "reasons": sorted({r for c in per_rank for r in c.get("reasons", [])}),
            "per_rank": per_rank}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU oracle timings (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------

def oracle_sample(wl, target_s=10.0, leaf_start=0, threads=None):
    """Time the oracle (as it stands) on a bounded sample of the workload:
    a contiguous run of output leaves (found by path replay) or Bernoulli
    chunks, sized for ~target_s seconds on all host cores."""
    import oracle as O
    cores = threads or os.cpu_count() or 1
    if wl["mode"] == "bernoulli":
        N, rho = wl["N"], wl["rho"]
        nch = 1 << O.bern_depth(N, rho)
        t = time.perf_counter(); _, v = O.bern_chunks_digest(N, rho, wl["seed"], 0, 64)
        rate = v / max(time.perf_counter() - t, 1e-6)
        chunks = int(min(nch, max(64, rate * target_s / max(v / 64, 1))))
        t = time.perf_counter(); _, v = O.bern_chunks_digest(N, rho, wl["seed"], 0, chunks)
        dt = time.perf_counter() - t
        return dict(value=v / dt, unit=UNIT, cores=1, kind="oracle",
                    sample=f"first {chunks} of {nch} Bernoulli chunks of {wl['name']} ({v} values, "
                           f"{dt:.1f} s, single-threaded oracle)")
    if wl["mode"] == "algb":          # whole Algorithm B runs at a reduced n
        N, ns = wl["N"], 2 ** 14
        t = time.perf_counter(); O.algb(N, ns, wl["seed"], wl["slack"]); dt = time.perf_counter() - t
        while dt < target_s / 4 and ns < wl["n"]:
            ns *= 4
            t = time.perf_counter(); O.algb(N, ns, wl["seed"], wl["slack"]); dt = time.perf_counter() - t
        return dict(value=ns / dt, unit=UNIT, cores=1, kind="oracle",
                    sample=f"whole Algorithm B at n={ns} of N={N} ({dt:.1f} s, single-threaded oracle)")
    mode = O.MODE_WR if wl["mode"] == "wr" else O.MODE_WOR
    N, n = wl["N"], wl["n"]
    D = O.plan(N, n, mode)[0]
    nl = 1 << D
    probe = min(nl, 256)
    t = time.perf_counter()
    _, v = O.digest_leaves_replay(N, n, wl["seed"], mode, leaf_start, leaf_start + probe, cores)
    dt = time.perf_counter() - t
    leaves = int(min(nl - leaf_start, max(probe, probe * target_s / max(dt, 1e-6))))
    t = time.perf_counter()
    _, v = O.digest_leaves_replay(N, n, wl["seed"], mode, leaf_start, leaf_start + leaves, cores)
    dt = time.perf_counter() - t
    return dict(value=v / dt, unit=UNIT, cores=cores, kind="oracle",
                sample=f"leaves [{leaf_start},{leaf_start + leaves}) of {nl} of {wl['name']} "
                       f"({v} values by path replay, {dt:.1f} s, {cores} threads)")


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    wl = _workload(args.workload, world)
    steps = []
    # each step = a bounded sample of the same workload (distinct leaves)
    per_step_s = max(1.0, min(20.0, 120.0 / max(args.steps + args.warmup, 1)))
    base = None
    for i in range(args.warmup + args.steps):
        r = oracle_sample(wl, target_s=per_step_s)
        if i >= args.warmup:
            steps.append(r["value"])
        base = r
    val = sorted(steps)[len(steps) // 2] if steps else base["value"]
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": _scaling(args.workload),
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": wl["name"], "N": wl["N"], "n": wl.get("n"), "rho": wl.get("rho"),
                   "seed": wl["seed"], "impl_note": "CPU oracle (oracle/rso.c), bounded sample per step"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                         "sample": base["sample"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------
# native (GPU) arm
# ---------------------------------------------------------------------------

def run_native(args):
    import paper_1610_05141_b200 as rs
    world, rank, local = _dist()
    local = local % max(torch.cuda.device_count(), 1)   # (gloo smoke test: ranks may share a GPU)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")   # collective tensors
    wl = _workload(args.workload, world)
    mode = wl["mode"]
    stream = torch.cuda.current_stream()

    # ---- buffers (outside the timed region)
    if mode == "bernoulli":
        N, rho, seed = wl["N"], wl["rho"], wl["seed"]
        cap = rs.bernoulli_capacity(N, rho)
        local_cap = cap if world == 1 else (cap // world + 64 * int(math.sqrt(cap)) + 64)
        out = torch.empty(local_cap, dtype=torch.uint64, device=dev)
        cnt = torch.zeros(1, dtype=torch.uint64, device=dev)
        ws = torch.empty(rs.workspace_bytes(rs.MODE_BERNOULLI, N, 0, rho, world), dtype=torch.uint8,
                         device=dev)
        n_local_expected = None

        def step():
            rs.bernoulli_ws(N, rho, seed, world, rank, out, local_cap, cnt, ws)
            if world > 1:
                allc = torch.empty(world, dtype=torch.int64, device=cdev)
                dist.all_gather_into_tensor(allc, cnt.view(torch.int64).to(cdev))
    elif mode == "algb":
        N, n, seed = wl["N"], wl["n"], wl["seed"]
        if world > 1:
            raise SystemExit("algb: single GPU only (comparison baseline)")
        m, n_local, g_off = rs.MODE_WOR, n, 0
        out = torch.empty(n, dtype=torch.uint64, device=dev)
        ws = torch.empty(rs.algb_workspace_bytes(N, n, wl["slack"]), dtype=torch.uint8, device=dev)

        def step():
            rs.sample_wor_algb(N, n, seed, slack=wl["slack"], out=out, ws=ws)
    else:
        N, n, seed = wl["N"], wl["n"], wl["seed"]
        m = rs.MODE_WR if mode == "wr" else rs.MODE_WOR
        if mode == "gnm" and world > 1:
            raise SystemExit("gnm: single GPU only")
        n_local, g_off = rs.shard_info(N, n, seed, world, rank, m)
        out = torch.empty(max(n_local, 1), dtype=torch.uint64, device=dev)
        ws = torch.empty(rs.workspace_bytes(m, N, n, 0.0, world), dtype=torch.uint8, device=dev)
        cnt = torch.tensor([n_local], dtype=torch.int64, device=cdev)
        fn = rs.sample_wr_ws if m == rs.MODE_WR else rs.sample_wor_ws
        allc = torch.empty(world, dtype=torch.int64, device=cdev)

        def step():
            if mode == "gnm":
                rs.gnm(wl["V"], n, seed, out=out, ws=ws)
            else:
                fn(N, n, seed, world, rank, out, ws)
            if world > 1:
                dist.all_gather_into_tensor(allc, cnt)   # per-GPU counts -> global offsets

    # ---- warm-up (untimed)
    for _ in range(max(args.warmup, 3 if args.warmup >= 3 else args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    rs.timing_enable(True)
    rs.timing_read(reset=True)
    rs.launch_count(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e0.record(stream)
    for i in range(args.steps):
        step()
        ev[i].record(stream)      # per-step split (median / best); the value uses e0..e1
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = rs.launch_count(reset=True)
    rs.timing_enable(False)
    kt = rs.timing_read(reset=True)
    clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    per_step = sorted([e0.elapsed_time(ev[0])] + [ev[i - 1].elapsed_time(ev[i]) for i in range(1, args.steps)])
    ms_max = _max_over_ranks(ms, world, dev)

    # ---- correctness of what was timed (untimed): sizes, order, range
    if mode == "bernoulli":
        c_local = min(int(cnt.item()), local_cap) if args.no_check else int(cnt.item())
        assert c_local <= local_cap, "bernoulli capacity exceeded"
        bad = 0 if args.launch_list else rs.validate(out[:c_local], N, strict=True)
        n_local_done = c_local
    else:
        bad = 0 if args.launch_list else rs.validate(out[:n_local], 2 ** 64 - 1 if mode == "gnm" else N,
                                                     strict=(mode != "wr"))
        n_local_done = n_local
        if world > 1:
            off = int(allc[:rank].sum().item())
            assert off == g_off, "all-gathered offset disagrees with the Algorithm P replay"
    if not args.no_check:
        assert bad == 0, f"validation failed: {bad} bad values"
        assert rs.device_errors(clear=True) == 0, "device capacity flag raised"
    total = torch.tensor([n_local_done], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(total)
    n_total = float(total.item())

    value = n_total / (ms_max / 1e3)
    gbs = 8.0 * n_total / (ms_max / 1e3) / 1e9

    # ---- roofline of the dominant kernel (leaf / Bernoulli), live CUDA events
    peak, peak_src = _peaks()
    if mode == "bernoulli":
        kms, kl = kt["bernoulli"]
        nunits = 1 << (rs.plan(rs.MODE_BERNOULLI, N, 0, rho)[0])
        bytes_per_launch = 8.0 * n_local_done + 8.0 * nunits / world
        kname = "k_bernoulli"
    elif mode == "algb":               # dominant of the Bernoulli pass and the compaction
        rho = min(1.0, (n + wl["slack"] * math.sqrt(n)) / N)
        npr = n + wl["slack"] * math.sqrt(n)                  # E[n'] (the pass count is host-side)
        kb, kc = kt["bernoulli"], kt["other"]
        if kb[0] >= kc[0]:
            kms, kl = kb
            bytes_per_launch = 8.0 * npr + 8.0 * (1 << rs.plan(rs.MODE_BERNOULLI, N, 0, rho)[0])
            kname = "k_bernoulli64d"
        else:
            kms, kl = kc
            bytes_per_launch = 8.0 * npr + 8.0 * n
            kname = "k_algb_compact"
    else:
        kms, kl = kt["leaf"]
        D = rs.plan(m, N, n)[0]
        nleaves = (1 << D) // world
        bytes_per_launch = 8.0 * n_local + 12.0 * nleaves
        comp = bool(rs.plan(m, N, n)[1])
        r_max = (N >> D) + 1
        if mode == "wor" and r_max <= 2 ** 15:
            kname = "k_leaf_bitmap_comp" if comp else "k_leaf_bitmap_wor"
        elif r_max > 0xfffff000 and mode != "gnm":
            kname = "k_leaf_warp_wide_wr" if mode == "wr" else "k_leaf_warp_wide_wor"
        else:
            kname = {"wr": "k_leaf_warp_wr", "gnm": "k_leaf_warp_gnm"}.get(mode, "k_leaf_warp_wor")
            # the top-up kernels: plain WOR at every range, G(n, m) for small ranges
            if mode == "wor" or (mode == "gnm" and r_max <= 2 ** 21):
                kname += "_tu"
            if mode in ("wor", "wr") and (N & (N - 1)) == 0:     # power-of-two N: the _p2 kernels
                kname += "_p2"
                if mode == "wor" and (N >> D) >= 2 ** 24:          # the kernel without the duplicate
                    kname = "k_leaf_warp_wor_sd_p2"                # path (+ its listed-leaf pass)
        # shard trees of depth <= 14 on the warp paths: split + leaves in one
        # launch (rs_fused.cuh); its time is the "leaf" class, split_ms ~ 0
        if mode in ("wor", "wr") and not comp and kname.startswith("k_leaf_warp_") and \
                D - (world - 1).bit_length() <= 14:
            kname = kname.replace("k_leaf_warp_", "k_fused_")
    kms_per = kms / max(kl, 1)
    achieved = bytes_per_launch / (kms_per / 1e3) / 1e9 if kms_per > 0 else None
    traffic, winst = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(wl["name"])
            traffic = float(t["bytes_per_launch"]) if t else None
            winst = float(t["warp_inst_per_launch"]) if t and t.get("warp_inst_per_launch") else None
    except Exception:
        pass
    # write-only ceiling on the same buffer: torch's vectorised fill of the
    # output (untimed by the step; a store-only path's honest denominator)
    fill_gbs = None
    try:
        if args.launch_list:
            raise RuntimeError("skipped")
        view = out.view(torch.int64)
        view.fill_(1)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(3):
            view.fill_(1)
        f1.record(stream)
        torch.cuda.synchronize()
        fill_gbs = 3 * 8.0 * view.numel() / (f0.elapsed_time(f1) / 1e3) / 1e9
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "fill_ceiling": fill_gbs,
                "frac_of_fill": (achieved / fill_gbs) if (achieved and fill_gbs) else None,
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": kname, "kernel_ms": kms_per, "peak_source": peak_src,
                "step_share": kms / max(args.steps, 1) / ms if ms > 0 else None,
                "split_ms": kt["split"][0] / max(args.steps, 1),
                "classes_ms": {k: v[0] / max(args.steps, 1) for k, v in kt.items()}}
    # second ceiling: instruction issue.  Warp instructions per
    # launch from the committed ncu capture (profiles/traffic.json) over the
    # live kernel time, against 4 warp-instructions / SM / cycle (one per
    # SMSP; tools/ubench measures 3.95 for an ALU+FMA mix) at the sampled SM clock
    csum0 = clocks.summary()
    f_sm = (csum0.get("sm_mhz") or 1965.0) * 1e6
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    if winst and kms_per > 0:
        ipc = winst / (kms_per / 1e3) / (nsm * f_sm)
        roofline["issue"] = {"warp_inst_per_launch": winst,
                             "warp_inst_per_sample": winst / max(float(n_local_done), 1.0),
                             "achieved_ipc_per_sm": ipc, "peak_ipc_per_sm": 4.0, "frac": ipc / 4.0,
                             "sm_mhz": f_sm / 1e6, "source": "profiles/traffic.json (ncu smsp__inst_executed.sum)"}

    # ---- end to end through the C ABI with a host buffer (fewer steps)
    e2e = None
    if not args.no_e2e and mode not in ("bernoulli", "gnm", "algb"):
        try:
            # N = 1: the whole sample lands in one pinned host buffer.  N > 1:
            # each rank streams its slice through a bounded two-slot pinned ring
            # (rs_sample_shard_host_stream; 8 ranks x 32 GiB would not fit the host)
            ring = world > 1
            elems = RING_ELEMS if ring else max(n_local, 1)
            try:
                host = torch.empty(elems, dtype=torch.uint64, pin_memory=True)
                pinned = True
            except Exception:
                host = torch.empty(elems, dtype=torch.uint64)
                pinned = False

            def e2e_call():
                if ring:
                    rs.sample_shard_host_stream(m, N, n, seed, world, rank, host)
                else:
                    rs.sample_shard_host(m, N, n, seed, world, rank, host)

            e2e_call()        # warm-up
            reps = args.e2e_steps
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            for _ in range(reps):
                e2e_call()
                if world > 1:
                    dist.all_gather_into_tensor(allc, cnt)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) / reps
            dt = _max_over_ranks(dt, world, dev)
            e2e = {"value": n_total / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": int(8 * n_total), "pinned": pinned, "steps": reps,
                   "host_buffer": (f"two-slot pinned ring of {RING_ELEMS} values per rank" if ring
                                   else "pinned, the whole sample"),
                   "note": "rs_sample_shard_host(_stream): device generation + D2H of every value"}
            del host
        except Exception as ex:  # report, never fake
            e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = oracle_sample(wl, target_s=args.cpu_seconds)
            if wl["mode"] not in ("bernoulli", "algb"):     # (those legs are single-threaded already)
                one = oracle_sample(wl, target_s=min(args.cpu_seconds, 5.0), threads=1)
                cpu["value_1thread"] = one["value"]
                cpu["sample_1thread"] = one["sample"]
        except Exception as ex:
            cpu = {"value": None, "error": str(ex)[:200]}

    csum = clocks.summary()
    clocks_all = [csum]
    if world > 1:
        clocks_all = [None] * world
        dist.all_gather_object(clocks_all, csum)
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "step_ms": {"mean": ms, "median": per_step[len(per_step) // 2], "best": per_step[0],
                        "rank": 0},
            "higher_is_better": True, "scaling": _scaling(args.workload), "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": wl["name"], "N": wl["N"], "n": wl.get("n"), "rho": wl.get("rho"),
                       "seed": wl["seed"], "parallelism": f"shard{world}",
                       "l2": "output >> 126 MB L2 (no flush needed)" if n_total * 8 > 1e9
                       else "output smaller than L2 (cache-warm)"},
            "output_gbs": gbs, "output_frac_of_peak": gbs / peak,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": _merge_clocks(clocks_all), "gpu_launches": launches,
        }
        print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _relaunch(n):
    """python bench.py --gpus N (N > 1, no WORLD_SIZE): one process per GPU
    under torch.distributed.run (127.0.0.1 rendezvous), same arguments; rank 0
    prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of one node; > 1 without WORLD_SIZE re-launches under torch.distributed.run")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="headline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-check", action="store_true", help="dev: skip the output validation asserts")
    ap.add_argument("--launch-list", action="store_true",
                    help="only the step's kernels (no validation / fill-ceiling kernels): for the ncu launch list")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: smoke-test the N > 1 path with ranks sharing one GPU")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus is not None and args.gpus > 1 and env_world is None:
        return _relaunch(args.gpus)
    if args.gpus is not None and env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={env_world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
