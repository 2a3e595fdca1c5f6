#!/usr/bin/env python
"""Benchmark of the Neptune attention hot path on B200 (driver contract).

Headline (BASELINE.json metric): attention forward TFLOP/s and % of BF16
peak on the MHA prefill config (B=8, H=16, S=4096, D=128, non-causal, bf16)
through the tcgen05 Rolling Update kernel; a secondary ``decode`` object
reports split-KV decode HBM GB/s on config 5 (Hq=32, Hkv=8, KV 128K, D=128).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...    (one process per GPU)

Multi-GPU: prefill shards independent (b, h) units (weak scaling: every rank
runs its own B=8 shard of a global batch of 8N, no collective); decode shards
the KV sequence (strong scaling) and combines the per-rank (m, l, O) triples
after one NCCL all-gather (paper_2510_08726_b200.dist).

Timing: W warm-up steps, then exactly K steps between barrier +
synchronize, CUDA events on the launching stream, max over ranks.  Inputs
are larger than L2 (126 MB) for every timed workload, so no flush is needed.
nvidia-smi clocks are sampled during the timed region.
``--impl reference`` times the fp64 CPU oracle (the reference arm of this
tier) on a bounded sample of the same workload."""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attn fwd TFLOP/s & % BF16 peak (seq 4096, d128); decode HBM GB/s; 1/2/4/8 GPU"

WORKLOADS = {
    # name: (config id, B, Hq, Hkv, S, D, variant)
    "mha": (2, 8, 16, 16, 4096, 128, dict()),
    "mha_causal": (2, 8, 16, 16, 4096, 128, dict(causal=True)),
    "gqa_window": (3, 4, 32, 8, 8192, 128, dict(causal=True, window=(4095, 0))),
    "var_scaled_dot": (4, 8, 16, 16, 2048, 64, dict()),
    "var_alibi_causal": (4, 8, 16, 16, 2048, 64, dict(causal=True, alibi=True)),
    "var_softcap_causal": (4, 8, 16, 16, 2048, 64, dict(causal=True, softcap=50.0)),
    # the config-4 family's other combinations (secondary lines; not in the default run)
    "var_causal": (4, 8, 16, 16, 2048, 64, dict(causal=True)),
    "var_alibi": (4, 8, 16, 16, 2048, 64, dict(alibi=True)),
    "var_softcap": (4, 8, 16, 16, 2048, 64, dict(softcap=50.0)),
    # ALiBi at D = 128 on the config-2 shape (the paper's MPT-7B ALiBi operator has D = 128)
    "mha_alibi": (2, 8, 16, 16, 4096, 128, dict(alibi=True)),
    "mha_alibi_causal": (2, 8, 16, 16, 4096, 128, dict(causal=True, alibi=True)),
}


def allowed_pairs(S: int, variant: dict) -> int:
    """Number of (query, key) pairs the mask allows for one (b, h), Sq = Skv = S."""
    causal = variant.get("causal", False)
    wl, wr = variant.get("window", (-1, -1))
    total = 0
    for i in range(S) if (wl >= 0 or wr >= 0) else ():
        lo = max(0, i - wl) if wl >= 0 else 0
        hi = min(S - 1, i + wr) if wr >= 0 else S - 1
        if causal:
            hi = min(hi, i)
        total += max(0, hi - lo + 1)
    if wl >= 0 or wr >= 0:
        return total
    return S * (S + 1) // 2 if causal else S * S


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), tf=float(d["bf16_tflops"]),
                    tf_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), src="measured")
    except Exception:
        return dict(hbm=6650.0, tf=1590.0, tf_sustained=1400.0, src="fallback")


class ClockSampler:
    """SM clock (every ~1 ms) and clock-event (throttle) reasons sampled during the
    timed region, through NVML (nvidia-smi's library)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_uuid: str):
        self.uuid, self.samples, self.reasons, self.max_mhz, self.err = gpu_uuid, [], set(), None, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByUUID(self.uuid.encode() if isinstance(self.uuid, str) else self.uuid)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = f"{type(e).__name__}: {e}"
            self.t = None
        return self

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        i = 0
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                if i % 4 == 0:   # the reasons query is the slow one
                    r = get_r(self.h)
                    for bit, name in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
            i += 1
            self._stop.wait(0.001)

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "error": self.err}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(self.samples), "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- reference arm / cpu baseline
def oracle_sample_rate(name: str, budget_s: float = 15.0, max_heads: int = 64):
    """fp64 oracle (as it stands) on whole (b, h) heads of the workload: TFLOP/s."""
    import numpy as np

    import datagen
    import oracle
    cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
    seed = datagen.config_seed(cid)
    p = oracle.Problem(B, Hq, Hkv, S, S, D, scale=1.0 / math.sqrt(D), causal=var.get("causal", False),
                       window_left=var.get("window", (-1, -1))[0], window_right=var.get("window", (-1, -1))[1],
                       softcap=var.get("softcap", 0.0),
                       alibi_slopes=datagen.alibi_slopes(Hq) if var.get("alibi") else None)
    rng = np.random.default_rng(0)
    flops_head = 4.0 * D * allowed_pairs(S, var)
    done, t_total = 0, 0.0
    while done < max_heads and (done == 0 or t_total < budget_s):
        b, hq = int(rng.integers(B)), int(rng.integers(Hq))
        g = oracle.head_group(p, hq)
        qs = datagen.as_f64(datagen.slab(seed, 1, (B, Hq, S, D), b, hq), "bf16")
        ks = datagen.as_f64(datagen.slab(seed, 2, (B, Hkv, S, D), b, g), "bf16")
        vs = datagen.as_f64(datagen.slab(seed, 3, (B, Hkv, S, D), b, g), "bf16")
        t0 = time.perf_counter()
        oracle.attention_bh(p, qs, ks, vs, hq)
        t_total += time.perf_counter() - t0
        done += 1
    return flops_head * done / t_total / 1e12, done, t_total


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.workload
    cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
    for _ in range(args.warmup):
        oracle_sample_rate(name, budget_s=0.0, max_heads=1)
    rates, times = [], []
    for _ in range(args.steps):
        r, n, t = oracle_sample_rate(name, budget_s=0.0, max_heads=1)
        rates.append(r)
        times.append(t)
    value = 4.0 * D * allowed_pairs(S, var) * len(times) / sum(times) / 1e12
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(name, args.gpus),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": f"1 whole (b, h) head of {name} per step ({S}x{S}, D={D}), fp64 numpy oracle"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(name, n):
    cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
    v = {k: (list(x) if isinstance(x, tuple) else x) for k, x in var.items()}
    return {"workload": f"{name} (BASELINE config {cid})", "batch_per_gpu": B, "global_batch": B * n,
            "heads_q": Hq, "heads_kv": Hkv, "seq_len": S, "head_dim": D, "variant": v,
            "parallelism": f"(b,h)-shard x{n}" if n > 1 else "single GPU",
            "l2": "inputs larger than L2 (no flush needed)"}


# ----------------------------------------------------------------------------- GPU arm
def main_gpu(args):
    import torch
    import torch.distributed as dist

    import datagen
    import paper_2510_08726_b200 as pb
    from datagen import device as dgd
    from paper_2510_08726_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo lets the N > 1 code path run with several ranks sharing one GPU
    # (a functional check on a 1-GPU box; its timings are meaningless).  Default: NCCL, one GPU per rank.
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    peaks = load_peaks()
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    gpu_id = uuid if uuid.startswith("GPU-") else f"GPU-{uuid}"  # NVML form

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup, sampler=True):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs = ClockSampler(gpu_id)
        with (cs if sampler else _Null()):
            s0.record()
            for _ in range(steps):
                fn()
            s1.record()
            torch.cuda.synchronize()
        barrier()
        ms = s0.elapsed_time(s1) / steps
        return max_over_ranks(ms), (cs.summary() if sampler else None)

    # ------------------------------------------------------------- prefill (headline)
    name = args.workload
    cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
    seed = datagen.config_seed(cid)
    q = torch.empty(B, Hq, S, D, dtype=torch.bfloat16, device=dev)
    k = torch.empty(B, Hkv, S, D, dtype=torch.bfloat16, device=dev)
    v = torch.empty(B, Hkv, S, D, dtype=torch.bfloat16, device=dev)
    # rank r owns batch rows [rB, (r+1)B) of a global [B*W, ...] tensor (weak scaling)
    dgd.fill_(q, seed, 1, start=rank * q.numel())
    dgd.fill_(k, seed, 2, start=rank * k.numel())
    dgd.fill_(v, seed, 3, start=rank * v.numel())
    o = torch.empty_like(q)
    kw = dict(causal=var.get("causal", False), window=var.get("window", (-1, -1)), softcap=var.get("softcap", 0.0))
    if var.get("alibi"):
        kw["alibi_slopes"] = torch.tensor(datagen.alibi_slopes(Hq), device=dev)
    step = lambda: pb.fused_fwd(q, k, v, out=o, **kw)  # noqa: E731
    step()
    torch.cuda.synchronize()
    launches_per_step = pb.last_launch_count()
    ms, clocks = timed(step, args.steps, args.warmup)
    flops = 4.0 * D * allowed_pairs(S, var) * B * Hq
    value = world * flops / (ms * 1e-3) / 1e12
    achieved = flops / (ms * 1e-3) / 1e12
    traffic, traffic_decode, traffic_smr = None, None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            traffic = tr.get(f"fwd_{name}")
            traffic_decode = tr.get(f"decode_b{args.decode_batch}") if world == 1 else None
            traffic_smr = tr.get("softmax_rows")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded datagen, N(0,1)-like, bf16)",
        "config": config_dict(name, world), "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["tf"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["tf"], "traffic": traffic,
                     "peak_src": f"{peaks['src']} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                     "kernel": "fwd_tc_kernel (tcgen05 Rolling Update)",
                     "algorithmic_flops_per_launch": flops},
    }
    # The exponentials (and softcap's tanh) run on the SFU (MUFU): 16 results/clk/SM (measured,
    # profiles/r1_microbench.md).  At D = 128 a 128x128 tile's exponentials take exactly as long
    # as its two MMAs; at D = 64 twice as long, so the D = 64 lines are bound by MUFU ("alu"),
    # not by the tensor core.  MUFU work = one ex2 per allowed (q, k) pair (+ one tanh with softcap).
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = float((clocks or {}).get("sm_max_mhz") or 1965.0)
    mufu_ops = allowed_pairs(S, var) * B * Hq * (2 if var.get("softcap") else 1)
    mufu_peak = 16.0 * sm_count * sm_mhz * 1e6 / 1e9                      # Gop/s
    mufu_ach = mufu_ops / (ms * 1e-3) / 1e9
    mufu = {"bound": "alu", "achieved": mufu_ach, "peak": mufu_peak, "unit": "Gop/s (MUFU ex2/tanh)",
            "frac": mufu_ach / mufu_peak, "ops_per_launch": mufu_ops,
            "peak_src": f"16 MUFU results/clk/SM x {sm_count} SMs x {sm_mhz:.0f} MHz"}
    if D == 64:
        tensor = line["roofline"]
        line["roofline"] = dict(mufu, traffic=traffic, kernel=tensor["kernel"],
                                tensor={k: tensor[k] for k in ("achieved", "peak", "unit", "frac")})
    else:
        line["roofline"]["mufu"] = mufu

    # ------------------------------------------------------------- e2e through the public API, host buffers
    if not args.no_e2e:
        hq_, hk_, hv_ = (t.cpu().pin_memory() for t in (q, k, v))
        ho_ = torch.empty(o.shape, dtype=o.dtype).pin_memory()
        e2e_steps = max(1, min(args.steps, 5))

        def e2e_step():
            return pb.fused_fwd(hq_, hk_, hv_, out=ho_, **kw)
        ms_e2e, _ = timed(e2e_step, e2e_steps, 1, sampler=False)
        line["e2e"] = {"value": world * flops / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 3 * q.numel() * 2, "d2h_bytes_per_step": o.numel() * 2,
                       "ms_per_step": ms_e2e, "steps": e2e_steps}
        del hq_, hk_, hv_, ho_

    del q, k, v, o
    torch.cuda.empty_cache()

    # ------------------------------------------------------------- decode (secondary metric)
    if not args.no_decode:
        Hqd, Hkvd, L, Dd = 32, 8, 131072, 128
        seed5 = datagen.config_seed(5)
        lo, hi = pdist.shard_range(L, rank, world)

        def run_decode(Bd, steps, warmup):
            qd = torch.empty(Bd, Hqd, 1, Dd, dtype=torch.bfloat16, device=dev)
            dgd.fill_(qd, seed5, 1)
            kd = torch.empty(Bd, Hkvd, hi - lo, Dd, dtype=torch.bfloat16, device=dev)
            vd = torch.empty_like(kd)
            for b in range(Bd):
                for h in range(Hkvd):
                    start = ((b * Hkvd + h) * L + lo) * Dd
                    dgd.fill_(kd[b, h], seed5, 2, start=start)
                    dgd.fill_(vd[b, h], seed5, 3, start=start)
            od = torch.empty_like(qd)
            ws = torch.zeros(pb.workspace_bytes(qd, kd), dtype=torch.uint8, device=dev)  # ticket block must start at 0
            if world == 1:
                dstep = lambda: pb.splitkv_decode(qd, kd, vd, causal=True, out=od, workspace=ws)  # noqa: E731
            else:
                dstep = lambda: pdist.decode_kv_sharded(qd, kd, vd, kv_pos_offset=lo,  # noqa: E731
                                                        seqlen_kv_total=L, causal=True)
            dstep()
            torch.cuda.synchronize()
            nl = pb.last_launch_count()
            if world == 1 and not args.no_graph:
                # A decode step is ~0.1 ms of GPU work at B = 1, less than the Python binding's
                # per-call host time: capture the step in a CUDA graph (the ABI is capture-safe:
                # no host sync, tensor maps are kernel parameters) and replay it.
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    dstep()
                torch.cuda.current_stream().wait_stream(side)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    dstep()
                dstep = graph.replay
            dms, dclk = timed(dstep, steps, warmup)
            breakdown = None
            if world > 1:   # local decode, local combine, all-gather, final combine
                var5 = dict(causal=True)
                parts = pdist._local_kernels(qd, kd, vd, kv_pos_offset=lo, seqlen_kv_total=L, num_splits=0,
                                             variant=var5)
                send = torch.empty(1, Bd, Hqd, Dd + 2, dtype=torch.float32, device=dev)
                recv = torch.empty(world, Bd, Hqd, Dd + 2, dtype=torch.float32, device=dev)
                pieces = {
                    "local_decode": lambda: pdist._local_kernels(qd, kd, vd, kv_pos_offset=lo, seqlen_kv_total=L,
                                                                 num_splits=0, variant=var5),
                    "local_combine": lambda: pdist._merge_kernels(parts, pb.Parts.packed(send)),
                    "all_gather": lambda: dist.all_gather_into_tensor(recv, send),
                    "final_combine": lambda: pdist._final_kernels(pb.Parts.packed(recv), torch.bfloat16, False),
                }
                breakdown = {key: round(timed(fn, steps, 2, sampler=False)[0], 5) for key, fn in pieces.items()}
                nl = 0   # kernels of one sharded step: local decode + local combine + final combine
                for key in ("local_decode", "local_combine", "final_combine"):
                    pieces[key]()
                    nl += pb.last_launch_count()
                del parts, send, recv
            del qd, kd, vd, od, ws
            torch.cuda.empty_cache()
            kv_bytes = 2.0 * Bd * Hkvd * L * Dd * 2
            return kv_bytes, dms, dclk, nl, breakdown

        def run_decode_bh(Bd, steps, warmup):
            """Communication-free alternative for large B: each rank decodes
            B/W whole sequences (all L keys), no collective."""
            Bl = Bd // world
            qd = torch.empty(Bl, Hqd, 1, Dd, dtype=torch.bfloat16, device=dev)
            kd = torch.empty(Bl, Hkvd, L, Dd, dtype=torch.bfloat16, device=dev)
            vd = torch.empty_like(kd)
            dgd.fill_(qd, seed5, 1, start=rank * qd.numel())
            dgd.fill_(kd, seed5, 2, start=rank * kd.numel())
            dgd.fill_(vd, seed5, 3, start=rank * vd.numel())
            od = torch.empty_like(qd)
            ws = torch.zeros(pb.workspace_bytes(qd, kd), dtype=torch.uint8, device=dev)
            fn = lambda: pb.splitkv_decode(qd, kd, vd, causal=True, out=od, workspace=ws)  # noqa: E731
            fn()
            ms, _ = timed(fn, steps, warmup, sampler=False)
            del qd, kd, vd, od, ws
            torch.cuda.empty_cache()
            return 2.0 * Bd * Hkvd * L * Dd * 2 / (ms * 1e-3) / 1e9, ms

        sweep, breakdowns = {}, {}
        for Bd in sorted(set([1, 4, args.decode_batch])):
            kv_bytes, dms, dclk, dl, bd = run_decode(Bd, max(args.steps, 20), args.warmup)
            sweep[Bd] = {"GB/s": kv_bytes / (dms * 1e-3) / 1e9, "ms_per_step": dms,
                         "frac_of_hbm_peak": kv_bytes / world / (dms * 1e-3) / 1e9 / peaks["hbm"]}
            if bd is not None:
                breakdowns[str(Bd)] = bd
        Bd = args.decode_batch
        gbs, dms = sweep[Bd]["GB/s"], sweep[Bd]["ms_per_step"]
        per_rank = gbs / world
        line["decode"] = {
            "metric": "split-KV decode HBM GB/s (K+V bytes read once / time)", "value": gbs, "unit": "GB/s",
            "ms_per_step": dms, "scaling": "strong" if world > 1 else None, "clocks": dclk,
            "config": {"workload": "decode (BASELINE config 5)", "batch": Bd, "heads_q": Hqd, "heads_kv": Hkvd,
                       "kv_len": L, "head_dim": Dd, "causal": True,
                       "parallelism": f"KV-sequence shard x{world} + NCCL all-gather of (m,l,O)" if world > 1
                       else "single GPU split-KV", "l2": "KV larger than L2",
                       "launch": "CUDA graph replay" if world == 1 and not args.no_graph else "eager"},
            "batch_sweep": {str(b): {k: round(v, 4) for k, v in d.items()} for b, d in sweep.items()},
            "gpu_launches_per_step": dl,
            "breakdown_ms": breakdowns or None,
            "roofline": {"bound": "hbm", "achieved": per_rank, "peak": peaks["hbm"], "unit": "GB/s",
                         "frac": per_rank / peaks["hbm"], "traffic": traffic_decode,
                         "peak_src": f"{peaks['src']} hbm_gbs (copy)", "kernel": "decode_split_kernel (fused Eq. 8 combine)",
                         "algorithmic_bytes_per_launch": 2.0 * Bd * Hkvd * L * Dd * 2 / world},
        }

        if world > 1 and args.decode_batch % world == 0:
            gbs_bh, ms_bh = run_decode_bh(args.decode_batch, max(args.steps, 20), args.warmup)
            line["decode"]["bh_sharded"] = {
                "GB/s": gbs_bh, "ms_per_step": ms_bh, "scaling": "strong",
                "parallelism": f"(b, hkv) sharding: {args.decode_batch // world} sequences per rank, no collective"}

    # ------------------------------------------------------------- NEXT-4: Fig. 2 reduction chain (softmax rows)
    if not args.no_softmax:
        rows, cols = 65536, 4096
        xs = torch.empty(rows, cols, dtype=torch.bfloat16, device=dev)
        dgd.fill_(xs, datagen.config_seed(6), 1, start=rank * xs.numel())
        ys = torch.empty_like(xs)
        sstep = lambda: pb.softmax_rows(xs, out=ys)  # noqa: E731
        sstep()
        torch.cuda.synchronize()
        sms, sclk = timed(sstep, max(args.steps, 20), args.warmup)
        sbytes = 2.0 * rows * cols * 2          # read x once + write y once
        sgbs = sbytes / (sms * 1e-3) / 1e9
        line["softmax_rows"] = {
            "metric": "Fig. 2 chain (row max, row sum, softmax) HBM GB/s (x read + y write)", "value": world * sgbs,
            "unit": "GB/s", "ms_per_step": sms, "scaling": "weak" if world > 1 else None,
            "config": {"workload": "softmax rows (NEXT-4)", "rows": rows, "cols": cols, "dtype": "bf16"},
            "roofline": {"bound": "hbm", "achieved": sgbs, "peak": peaks["hbm"], "unit": "GB/s",
                         "frac": sgbs / peaks["hbm"], "traffic": traffic_smr, "kernel": "softmax_rows16_kernel",
                         "algorithmic_bytes_per_launch": sbytes},
        }
        del xs, ys

    # ------------------------------------------------------------- CPU baseline (oracle), rank 0, N = 1
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, heads, secs = oracle_sample_rate(name, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": rate, "unit": "TFLOP/s", "cores": blas_threads(), "kind": "oracle",
                                "sample": f"{heads} whole (b,h) heads of {name} ({S}x{S}, D={D}) in {secs:.1f} s, "
                                          "fp64 numpy oracle (oracle.attention_bh)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="mha")
    ap.add_argument("--decode-batch", type=int, default=16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-softmax", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="decode: eager launches instead of a CUDA graph")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        main_gpu(args)


if __name__ == "__main__":
    main()
