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
synchronize, CUDA events on the launching stream, max over ranks.  A workload
whose inputs are smaller than 2 x L2 (the D = 64 configs; a rank's decode KV
shard at large N) has the L2 flushed between steps (a 252 MB write outside the
timed events, per-step events); the others are larger than L2.  NVML clocks
are sampled during every timed region.

At N = 1 the line also carries the other §8(d) configs (C2b ``mha_causal``, C3
``gqa_window``, C4 ``var_*``), each with clocks and tensor + MUFU rooflines; at
N > 1 a ``strong_scaling`` object (the fixed C2a problem's (b, h) units
sharded over the ranks).
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
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "cpu_model": cpu_model(),
                         "nproc": os.cpu_count(), "kind": "oracle",
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
L2_BYTES = 126 << 20            # B200 L2 (B200_PROFILING.md)
# The §8(d) configs reported next to the headline in the N = 1 line (each with its own
# clocks, tensor + MUFU roofline and ncu traffic): C2b, C3 and the C4 variant family.
EXTRA_WORKLOADS = ("mha_causal", "gqa_window", "var_scaled_dot", "var_alibi_causal", "var_softcap_causal")


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_decode_rate(budget_s: float = 10.0, n_distinct: int = 2, max_groups: int = 4096):
    """fp64 oracle (as it stands) on whole (b, hkv) groups of config 5 (KV 128K, D = 128, 4 q heads
    per group): algorithmic K+V GB/s of the groups it finished.  n_distinct groups are generated
    (the generator is not timed) and cycled until the time budget is spent."""
    import numpy as np

    import datagen
    import oracle
    B, Hq, Hkv, L, D = 16, 32, 8, 131072, 128
    seed = datagen.config_seed(5)
    p = oracle.Problem(B, Hq, Hkv, 1, L, D, scale=1.0 / math.sqrt(D), causal=True)
    rng = np.random.default_rng(5)
    groups = []
    for _ in range(n_distinct):
        b, g = int(rng.integers(B)), int(rng.integers(Hkv))
        ks = datagen.as_f64(datagen.slab(seed, 2, (B, Hkv, L, D), b, g), "bf16")
        vs = datagen.as_f64(datagen.slab(seed, 3, (B, Hkv, L, D), b, g), "bf16")
        qs = [datagen.as_f64(datagen.slab(seed, 1, (B, Hq, 1, D), b, hq), "bf16") for hq in range(g * 4, g * 4 + 4)]
        groups.append((g, qs, ks, vs))
    done, t_total = 0, 0.0
    while done < max_groups and (done == 0 or t_total < budget_s):
        g, qs, ks, vs = groups[done % n_distinct]
        t0 = time.perf_counter()
        for i, hq in enumerate(range(g * 4, g * 4 + 4)):
            oracle.attention_bh(p, qs[i], ks, vs, hq)
        t_total += time.perf_counter() - t0
        done += 1
    return 2.0 * L * D * 2 * done / t_total / 1e9, done, t_total


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
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)   # L2 flush: a write > L2

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup, sampler=True, flush=False):
        """ms per step on the device (CUDA events on the launching stream), max over ranks.
        flush: the L2 is flushed (a 2 x L2 write) between steps, outside the timed events."""
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        cs = ClockSampler(gpu_id)
        with (cs if sampler else _Null()):
            if flush:
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(steps)]
                for e0, e1 in evs:
                    flush_buf.zero_()
                    e0.record()
                    fn()
                    e1.record()
                torch.cuda.synchronize()
                ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
            else:
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                for _ in range(steps):
                    fn()
                s1.record()
                torch.cuda.synchronize()
                ms = s0.elapsed_time(s1) / steps
        barrier()
        return max_over_ranks(ms), (cs.summary() if sampler else None)

    traffic_tab = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic_tab = json.load(open(tpath))
        except Exception:
            traffic_tab = {}

    # ------------------------------------------------------------- prefill
    def prefill(name, batch_lo=None, batch_hi=None, steps=None):
        """One prefill workload: rank r runs its own B-batch shard of a global batch B*W (weak
        scaling), or batches [batch_lo, batch_hi) of the fixed config (strong scaling)."""
        cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
        seed = datagen.config_seed(cid)
        if batch_lo is None:
            b0, nb = rank * B, B
        else:
            b0, nb = batch_lo, batch_hi - batch_lo
        q = torch.empty(nb, Hq, S, D, dtype=torch.bfloat16, device=dev)
        k = torch.empty(nb, Hkv, S, D, dtype=torch.bfloat16, device=dev)
        v = torch.empty(nb, Hkv, S, D, dtype=torch.bfloat16, device=dev)
        dgd.fill_(q, seed, 1, start=b0 * Hq * S * D)
        dgd.fill_(k, seed, 2, start=b0 * Hkv * S * D)
        dgd.fill_(v, seed, 3, start=b0 * Hkv * S * D)
        o = torch.empty_like(q)
        kw = dict(causal=var.get("causal", False), window=var.get("window", (-1, -1)), softcap=var.get("softcap", 0.0))
        if var.get("alibi"):
            kw["alibi_slopes"] = torch.tensor(datagen.alibi_slopes(Hq), device=dev)
        step = lambda: pb.fused_fwd(q, k, v, out=o, **kw)  # noqa: E731
        step()
        torch.cuda.synchronize()
        launches = pb.last_launch_count()
        in_bytes = 2 * (q.numel() + k.numel() + v.numel() + o.numel())
        flush = in_bytes < 2 * L2_BYTES
        ms, clocks = timed(step, steps or args.steps, args.warmup, flush=flush)
        flops = 4.0 * D * allowed_pairs(S, var) * nb * Hq
        achieved = flops / (ms * 1e-3) / 1e12
        sm_mhz = float((clocks or {}).get("sm_max_mhz") or 1965.0)
        mufu_ops = allowed_pairs(S, var) * nb * Hq * (2 if var.get("softcap") else 1)
        mufu_peak = 16.0 * sm_count * sm_mhz * 1e6 / 1e9                      # Gop/s
        mufu_ach = mufu_ops / (ms * 1e-3) / 1e9
        tensor = {"bound": "tensor", "achieved": achieved, "peak": peaks["tf"], "unit": "TFLOP/s",
                  "frac": achieved / peaks["tf"], "traffic": traffic_tab.get(f"fwd_{name}"),
                  "peak_src": f"{peaks['src']} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                  "kernel": "fwd_tc_persist_kernel" if (D == 128 and var.get("causal") and "window" not in var
                                                        and not var.get("alibi")) else "fwd_tc_kernel",
                  "algorithmic_flops_per_launch": flops}
        # The exponentials (and softcap's tanh) run on the SFU (MUFU): 16 results/clk/SM (measured,
        # profiles/r1_microbench.md).  At D = 128 a 128x128 tile's exponentials take exactly as long
        # as its two MMAs; at D = 64 twice as long, so the D = 64 lines are bound by MUFU ("alu").
        sm_now = float((clocks or {}).get("sm_mhz") or sm_mhz)
        mufu = {"bound": "alu", "achieved": mufu_ach, "peak": mufu_peak, "unit": "Gop/s (MUFU ex2/tanh)",
                "frac": mufu_ach / mufu_peak, "ops_per_launch": mufu_ops,
                "peak_src": f"16 MUFU results/clk/SM x {sm_count} SMs x {sm_mhz:.0f} MHz (max SM clock)",
                # the same bound at the SM clock sampled during this run (the SFU rate scales with it)
                "frac_at_sampled_clock": mufu_ach / (16.0 * sm_count * sm_now * 1e6 / 1e9)}
        if D == 64:
            roof = dict(mufu, traffic=tensor["traffic"], kernel=tensor["kernel"],
                        tensor={kk: tensor[kk] for kk in ("achieved", "peak", "unit", "frac")})
        else:
            roof = dict(tensor, mufu=mufu)
        res = {"value": world * flops / (ms * 1e-3) / 1e12 if batch_lo is None else None, "unit": "TFLOP/s",
               "ms_per_step": ms, "clocks": clocks, "roofline": roof, "gpu_launches_per_step": launches,
               "config": config_dict(name, world), "flops_per_rank": flops,
               "l2": "flushed between steps (2 x L2 write, outside the timed events)" if flush
                     else "inputs larger than L2 (no flush)"}
        res["config"]["l2"] = res["l2"]
        return res, (q, k, v, o, kw, flops)

    name = args.workload
    head, (q, k, v, o, kw, flops) = prefill(name)
    line = {
        "metric": METRIC, "value": head["value"], "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded datagen, N(0,1)-like, bf16)",
        "config": head["config"], "clocks": head["clocks"],
        "gpu_launches": head["gpu_launches_per_step"] * args.steps,
        "roofline": head["roofline"],
    }

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
                       "ms_per_step": ms_e2e, "steps": e2e_steps,
                       "path": "pb.fused_fwd on pinned host tensors (H2D of q, k, v and D2H of o inside the timed "
                               "region, chunked over two streams)"}
        del hq_, hk_, hv_, ho_
    del q, k, v, o
    torch.cuda.empty_cache()

    # ------------------------------------------------------------- the other §8(d) configs (N = 1)
    if world == 1 and not args.no_workloads:
        for w in EXTRA_WORKLOADS:
            if w == name:
                continue
            # the board settles below its boost clock after seconds of full-power compute (no NVML
            # reason); an idle pause before each config keeps them comparable
            time.sleep(args.cooldown)
            res, tensors = prefill(w)
            del tensors
            torch.cuda.empty_cache()
            line[w] = res

    # ------------------------------------------------------------- strong scaling of C2a (§8(e))
    if world > 1:
        cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
        if B % world == 0:
            lo, hi = pdist.shard_range(B, rank, world)
            res, tensors = prefill(name, lo, hi)
            del tensors
            torch.cuda.empty_cache()
            total = 4.0 * D * allowed_pairs(S, var) * B * Hq
            line["strong_scaling"] = {
                "value": total / (res["ms_per_step"] * 1e-3) / 1e12, "unit": "TFLOP/s",
                "ms_per_step": res["ms_per_step"], "scaling": "strong",
                "parallelism": f"the fixed {name} problem's {B * Hq} (b, h) units sharded {B // world} batches "
                               f"x {Hq} heads per rank (shard_range), no collective",
                "flops_total": total, "clocks": res["clocks"]}

    # ------------------------------------------------------------- decode (secondary metric)
    if not args.no_decode:
        time.sleep(args.cooldown)
        Hqd, Hkvd, L, Dd = 32, 8, 131072, 128
        seed5 = datagen.config_seed(5)
        lo, hi = pdist.shard_range(L, rank, world)
        use_cabi = world > 1 and backend == "nccl"
        comm = pdist.NcclComm(rank, world) if use_cabi else None

        def make_decode_inputs(Bd):
            qd = torch.empty(Bd, Hqd, 1, Dd, dtype=torch.bfloat16, device=dev)
            dgd.fill_(qd, seed5, 1)
            kd = torch.empty(Bd, Hkvd, hi - lo, Dd, dtype=torch.bfloat16, device=dev)
            vd = torch.empty_like(kd)
            for b in range(Bd):
                for h in range(Hkvd):
                    start = ((b * Hkvd + h) * L + lo) * Dd
                    dgd.fill_(kd[b, h], seed5, 2, start=start)
                    dgd.fill_(vd[b, h], seed5, 3, start=start)
            return qd, kd, vd

        def run_decode(Bd, steps, warmup):
            qd, kd, vd = make_decode_inputs(Bd)
            od = torch.empty_like(qd)
            shard_bytes = 2 * kd.numel() * 2
            flush = shard_bytes < 2 * L2_BYTES
            if world == 1:
                ws = torch.zeros(pb.workspace_bytes(qd, kd), dtype=torch.uint8, device=dev)  # tickets start at 0
                dstep = lambda: pb.splitkv_decode(qd, kd, vd, causal=True, out=od, workspace=ws)  # noqa: E731
            elif use_cabi:   # the C ABI's one-call path: fused local merge, NCCL all-gather, Eq. 8
                dstep = lambda: comm.decode_kv_sharded(qd, kd, vd, kv_pos_offset=lo, seqlen_kv_total=L,  # noqa: E731
                                                       out=od, causal=True)
            else:
                dstep = lambda: pdist.decode_kv_sharded(qd, kd, vd, kv_pos_offset=lo,  # noqa: E731
                                                        seqlen_kv_total=L, causal=True)
            dstep()
            torch.cuda.synchronize()
            nl = pb.last_launch_count()
            graphed = (world == 1 or use_cabi) and not args.no_graph
            if graphed:
                # A decode step is ~0.1 ms of GPU work at B = 1, less than the Python binding's
                # per-call host time: capture the step (NCCL included at N > 1) in a CUDA graph.
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    dstep()
                torch.cuda.current_stream().wait_stream(side)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    dstep()
                dstep = graph.replay
            dms, dclk = timed(dstep, steps, warmup, flush=flush)
            breakdown = None
            if world > 1:   # local decode (+ fused local merge), all-gather, final combine
                send = torch.empty(Bd, Hqd, Dd + 2, dtype=torch.float32, device=dev)
                recv = torch.empty(world, Bd, Hqd, Dd + 2, dtype=torch.float32, device=dev)
                wsl = torch.zeros(pb.workspace_bytes(qd, kd), dtype=torch.uint8, device=dev)
                pieces = {
                    "local_decode_and_merge": lambda: pb.splitkv_decode(qd, kd, vd, packed=send, workspace=wsl,
                                                                        kv_pos_offset=lo, seqlen_kv_total=L,
                                                                        causal=True),
                    "all_gather": lambda: dist.all_gather_into_tensor(recv.view(world * Bd, Hqd, Dd + 2), send),
                    "final_combine": lambda: pdist._final_kernels(pb.Parts.packed(recv), torch.bfloat16, False),
                }
                breakdown = {key: round(timed(fn, steps, 2, sampler=False, flush=flush)[0], 5)
                             for key, fn in pieces.items()}
                del send, recv, wsl
            del qd, kd, vd, od
            torch.cuda.empty_cache()
            kv_bytes = 2.0 * Bd * Hkvd * L * Dd * 2
            return kv_bytes, dms, dclk, nl, breakdown, graphed, flush

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
        dl, graphed, dflush, dclk_head = 1, False, False, None
        for Bd in sorted(set([1, 4, args.decode_batch])):
            kv_bytes, dms, dclk, nl, bd, graphed_b, flush_b = run_decode(Bd, max(args.steps, 20), args.warmup)
            sweep[Bd] = {"GB/s": kv_bytes / (dms * 1e-3) / 1e9, "ms_per_step": dms,
                         "frac_of_hbm_peak": kv_bytes / world / (dms * 1e-3) / 1e9 / peaks["hbm"]}
            if bd is not None:
                breakdowns[str(Bd)] = bd
            if Bd == args.decode_batch:
                dl, graphed, dflush, dclk_head = nl, graphed_b, flush_b, dclk
        Bd = args.decode_batch
        gbs, dms = sweep[Bd]["GB/s"], sweep[Bd]["ms_per_step"]
        per_rank = gbs / world
        line["decode"] = {
            "metric": "split-KV decode HBM GB/s (K+V bytes read once / time)", "value": gbs, "unit": "GB/s",
            "ms_per_step": dms, "scaling": "strong" if world > 1 else None, "clocks": dclk_head,
            "config": {"workload": "decode (BASELINE config 5)", "batch": Bd, "heads_q": Hqd, "heads_kv": Hkvd,
                       "kv_len": L, "head_dim": Dd, "causal": True,
                       "parallelism": (f"KV-sequence shard x{world}: fused local merge + NCCL all-gather of (m,l,O) + "
                                       "Eq. 8 (attn_decode_kv_sharded, one C-ABI call)" if use_cabi else
                                       f"KV-sequence shard x{world} (torch.distributed all-gather)") if world > 1
                       else "single GPU split-KV",
                       "l2": ("flushed between steps (a rank's K/V shard fits in L2)" if dflush
                              else "KV larger than L2 (no flush)"),
                       "launch": "CUDA graph replay" if graphed else "eager"},
            "batch_sweep": {str(b): {kk: round(vv, 4) for kk, vv in d.items()} for b, d in sweep.items()},
            "gpu_launches_per_step": dl,
            "breakdown_ms": breakdowns or None,
            "roofline": {"bound": "hbm", "achieved": per_rank, "peak": peaks["hbm"], "unit": "GB/s",
                         "frac": per_rank / peaks["hbm"],
                         "traffic": traffic_tab.get(f"decode_b{Bd}") if world == 1 else None,
                         "peak_src": f"{peaks['src']} hbm_gbs (copy)", "kernel": "decode_split_kernel (fused Eq. 8 combine)",
                         "algorithmic_bytes_per_launch": 2.0 * Bd * Hkvd * L * Dd * 2 / world},
        }
        # e2e: host q in, host O out through the public API (KV cache resident in HBM, as in serving)
        if world == 1 and not args.no_e2e:
            qd, kd, vd = make_decode_inputs(Bd)
            qh = qd.cpu().pin_memory()
            fn = lambda: pb.splitkv_decode(qh, kd, vd, causal=True)  # noqa: E731
            ms_e2e, _ = timed(fn, 10, 3, sampler=False)
            line["decode"]["e2e"] = {
                "value": 2.0 * Bd * Hkvd * L * Dd * 2 / (ms_e2e * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": qd.numel() * 2, "d2h_bytes_per_step": qd.numel() * 2,
                "path": "pb.splitkv_decode(q on pinned host, K/V cache resident on the device) -> O on the host"}
            del qd, kd, vd, qh
            torch.cuda.empty_cache()
        if rank == 0 and world == 1 and not args.no_cpu:
            rate, groups, secs = oracle_decode_rate(budget_s=args.cpu_budget * 2 / 3)
            line["decode"]["cpu_baseline"] = {
                "value": rate, "unit": "GB/s", "cores": blas_threads(), "cpu_model": cpu_model(),
                "nproc": os.cpu_count(), "kind": "oracle",
                "sample": f"{groups} (b, hkv) group decodes of config 5 (4 q heads x 131072 keys, D=128; 2 distinct "
                          f"groups cycled) in {secs:.1f} s, fp64 numpy oracle (oracle.attention_bh); GB/s = their "
                          "K+V bf16 bytes / time"}
        if world > 1 and args.decode_batch % world == 0:
            gbs_bh, ms_bh = run_decode_bh(args.decode_batch, max(args.steps, 20), args.warmup)
            line["decode"]["bh_sharded"] = {
                "GB/s": gbs_bh, "ms_per_step": ms_bh, "scaling": "strong",
                "parallelism": f"(b, hkv) sharding: {args.decode_batch // world} sequences per rank, no collective"}
        if comm is not None:
            comm.close()

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
            "unit": "GB/s", "ms_per_step": sms, "scaling": "weak" if world > 1 else None, "clocks": sclk,
            "config": {"workload": "softmax rows (NEXT-4)", "rows": rows, "cols": cols, "dtype": "bf16",
                       "l2": "inputs larger than L2 (no flush)"},
            "roofline": {"bound": "hbm", "achieved": sgbs, "peak": peaks["hbm"], "unit": "GB/s",
                         "frac": sgbs / peaks["hbm"], "traffic": traffic_tab.get("softmax_rows"),
                         "kernel": "softmax_rows16_kernel", "algorithmic_bytes_per_launch": sbytes},
        }
        del xs, ys

    # ------------------------------------------------------------- CPU baseline (oracle), rank 0, N = 1
    if rank == 0 and world == 1 and not args.no_cpu:
        cid, B, Hq, Hkv, S, D, var = WORKLOADS[name]
        rate, heads, secs = oracle_sample_rate(name, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": rate, "unit": "TFLOP/s", "cores": blas_threads(), "cpu_model": cpu_model(),
                                "nproc": os.cpu_count(), "kind": "oracle",
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
    ap.add_argument("--no-workloads", action="store_true", help="skip the other §8(d) prefill configs (N = 1)")
    ap.add_argument("--no-graph", action="store_true", help="decode: eager launches instead of a CUDA graph")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cooldown", type=float, default=2.0, help="idle seconds before each secondary config")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        main_gpu(args)


if __name__ == "__main__":
    main()
