#!/usr/bin/env python
"""Benchmark of the any4 hot path on B200 (contract: see DESIGN.md §Measurement).

Headline (BASELINE.json metric "any4 GEMM µs and % HBM peak at M=1–16 (Llama-3
shapes); k-means rows/s", config[1] "Llama-3-8B layer shapes ... M=1..16"):

  step   = the seven Llama-3-8B decoder-layer GEMMs (q,k,v,o,gate,up,down) at
           M=1 on any4 g128 weights, y = x W^T, bf16 x/y, with the decoder's
           data dependencies (o reads y_q, gate/up read y_o, down reads y_up),
           as ONE k_lutgemv chain launch per layer. Weights rotate over LAYERS
           layers (> L2), so every step streams its weights from HBM. CUDA
           graphs remove host launch overhead.
  value  = algorithmic bytes streamed per step / device time per step (GB/s),
           whole job over all ranks.
  e2e    = same metric through the public API with HOST buffers: the layer
           input is copied H2D from pinned memory and all seven outputs D2H
           inside the timed region, every step (one GPU: on two copy streams,
           pipelined with the neighbouring steps' launches and captured with
           them as one graph of the K steps, as a serving loop would run them).
  extras = per-shape µs and % of HBM peak, the M=1..16 sweep, k-means rows/s
           (config 1), roofline of the dominant kernel, CPU baseline.

`--impl reference` times the reference's own CPU GEMM (oracle/_ref, the
unmodified reference built in place) on the host cores with the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Llama-3-8B linear layers (N x K) — SURVEY.md §8(d) config 2.
LAYER = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
         ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
GROUP = 128
MODEL = "8b"
METRIC = "any4 GEMM µs and % HBM peak at M=1–16 (Llama-3 shapes); k-means rows/s"
UNIT = "GB/s"
LAYER_70B = [("q", 8192, 8192), ("k", 1024, 8192), ("v", 1024, 8192), ("o", 8192, 8192),
             ("gate", 28672, 8192), ("up", 28672, 8192), ("down", 8192, 28672)]


def algo_bytes(n, k, m, bits=4, group=GROUP):
    """Algorithmic bytes of one GEMM: codes + fp16 alpha/beta
    + fp16 LUT + bf16 x + bf16 y."""
    codes = n * ((k * bits + 7) // 8)
    scales = n * ((k + group - 1) // group) * 2 * 2
    lut = n * (1 << bits) * 2
    return codes + scales + lut + m * k * 2 + m * n * 2


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def hbm_peak_tflops():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 1590.0


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi equivalent through NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, dev_index=0, period=0.0002):
        self.samples, self.reasons, self.timed = [], set(), []
        self.t_start, self.t_end = None, None
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.timed.append((time.perf_counter(), mhz, r))
            except Exception:
                pass
            time.sleep(self.period)

    def wait_running(self, n=3, timeout=2.0):
        """Block until the sampler has taken n samples (its first NVML calls are slow)."""
        t_end = time.time() + timeout
        while self.nv is not None and len(self.timed) < n and time.time() < t_end:
            time.sleep(0.001)

    def mark(self, which):
        setattr(self, "t_" + which, time.perf_counter())

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        # the samples taken while the timed region ran (host marks around it)
        lo = self.t_start if self.t_start is not None else -1e30
        hi = self.t_end if self.t_end is not None else 1e30
        for t, mhz, r in self.timed:
            if lo <= t <= hi:
                self.samples.append(mhz)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# synthetic any4 weights
# ---------------------------------------------------------------------------
def synthetic_qtensor(n, k, seed, fmt="any4"):
    """Random-code tensor of a format: any4 / any3 (learned LUTs, sorted in the
    scaled domain) or int4 / nf4 (the reference's fixed tables, asymmetric)."""
    from paper_2507_04610_b200 import _abi
    from paper_2507_04610_b200.qtensor import QuantizedTensor

    rng = np.random.default_rng(seed)
    cb = {"any4": _abi.CB_ANY, "any3": _abi.CB_ANY, "int4": 0, "nf4": 2}[fmt]
    bits = 3 if fmt == "any3" else 4
    cfg = _abi.default_config(codebook=cb, group_size=GROUP)
    cfg.bits = bits
    qt = QuantizedTensor.empty(n, k, cfg)
    if bits == 4:  # int4 / nf4 / any4: all 16 codes are valid
        qt.codes[:] = rng.integers(0, 256, qt.codes.size, dtype=np.uint8)
    else:  # any3: 3-bit packed codes
        from paper_2507_04610_b200 import anyq

        qt.codes[:] = anyq.pack_codes(rng.integers(0, 8, (n, k), dtype=np.uint8), bits).ravel()
    if qt.luts is not None:
        # learned LUTs live in the scaled domain [0, 15], sorted (pack.hpp invariants)
        lut = np.sort(rng.random((n, 1 << bits), dtype=np.float32) * 15.0, axis=1)
        qt.luts[:] = lut.ravel()
    qt.alphas[:] = (0.01 + 0.04 * rng.random(qt.alphas.size, dtype=np.float32))
    qt.betas[:] = -0.3 * rng.random(qt.betas.size, dtype=np.float32)
    return qt


def make_layers(nlayers, shard=(0, 1)):
    """Device tensors for `nlayers` layers; with shard=(r, P) each tensor holds
    rows [r*N/P, (r+1)*N/P) of every weight (column-sharded TP)."""
    from paper_2507_04610_b200 import anyq

    r, P = shard
    layers = []
    for l in range(nlayers):
        mats = []
        for i, (name, n, k) in enumerate(LAYER):
            ns = n // P
            qt = synthetic_qtensor(ns, k, seed=1000 * l + 10 * i + r)
            mats.append((name, ns, k, anyq.DeviceTensor(qt)))
        layers.append(mats)
    return layers


# ---------------------------------------------------------------------------
# reference arm (CPU)
# ---------------------------------------------------------------------------
def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle.refpy import REF_SO, have_ref, oracle, ref

    lib = ref() if have_ref() else oracle()
    kind = "reference" if have_ref() else "port"
    threads = os.cpu_count() or 1
    # one full decoder layer at M=1, rows split over the host threads
    # (gemm_fused is single-threaded by design, qgemm.cpp:113-126; the split
    # over output rows is harness parallelism, labelled as such)
    m = 1
    work = []
    for i, (name, n, k) in enumerate(LAYER):
        qt = synthetic_qtensor(n, k, seed=10 * i)
        x = np.random.default_rng(i).standard_normal((m, k)).astype(np.float32)
        parts = []
        step = (n + threads - 1) // threads
        for r0 in range(0, n, step):
            r1 = min(n, r0 + step)
            sub = qt.clone()
            sub.rows = r1 - r0
            bpr = (k * 4 + 7) // 8
            gpr = (k + GROUP - 1) // GROUP
            sub.codes = qt.codes[r0 * bpr:r1 * bpr].copy()
            sub.luts = qt.luts[r0 * 16:r1 * 16].copy()
            sub.alphas = qt.alphas[r0 * gpr:r1 * gpr].copy()
            sub.betas = qt.betas[r0 * gpr:r1 * gpr].copy()
            parts.append(sub)
        work.append((n, k, x, parts))
    step_bytes = sum(algo_bytes(n, k, m) for (_, n, k) in LAYER)

    def one_step(pool):
        futs = [pool.submit(lib.gemm_fused, x, sub) for (n, k, x, parts) in work for sub in parts]
        for f in futs:
            f.result()

    with ThreadPoolExecutor(max_workers=threads) as pool:
        for _ in range(args.warmup):
            one_step(pool)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(pool)
        dt = (time.perf_counter() - t0) / args.steps
    value = step_bytes / dt / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dt * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"llama3-{MODEL}-layer-gemms", "M": m, "group_size": GROUP,
                   "shapes": [[n, k] for (_, n, k) in LAYER]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"one Llama-3-{MODEL} layer (7 GEMMs) at M=1, reference gemm_fused "
                                   f"(qgemm.cpp:71) over {threads} row slices (harness-parallel)",
                         "library": os.path.relpath(REF_SO, ROOT) if kind == "reference" else
                         "oracle/_build/liboracle.so"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kmeans_cpu_baseline(layer):
    """Reference quantize_any on the host cores, stratified one-layer sample."""
    from oracle.refpy import _abi, have_ref, oracle, ref

    lib = ref() if have_ref() else oracle()
    kind = "reference" if have_ref() else "port"
    threads = os.cpu_count() or 1
    cfg = _abi.default_config(codebook=_abi.CB_ANY)
    rates = {}
    for k, rows in ((4096, 2048), (14336, 512)):
        w = lib.gaussian(rows, k, 1)
        exj = lib.synthetic_stats(k, 10007)
        secs = lib.time_quantize(w, cfg, exj, threads)
        rates[k] = rows / secs
    lrows = sum(n for (_, n, _) in layer)
    layer_s = sum(n / rates[k] for (_, n, k) in layer)
    return {"value": round(lrows / layer_s, 1), "unit": "rows/s", "cores": threads, "kind": kind,
            "rows_per_s_by_K": {str(k): round(v, 1) for k, v in rates.items()},
            "sample": "reference quantize_any (learner.cpp:392-448), any4 g128 with synthetic stats, "
                      f"{threads} threads: 2048 rows x 4096 and 512 rows x 14336, one 8B layer "
                      "(38912 rows at K=4096, 4096 at K=14336) extrapolated from the two rates"}


def kmeans_roofline():
    """The k-means kernel's bound from its committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_kmeans.json")
    try:
        m = json.load(open(path))["metrics"]
        fp64 = float(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]["value"]) / 100
        issue = float(m["sm__issue_active.avg.pct_of_peak_sustained_elapsed"]["value"]) / 100
    except (OSError, KeyError, ValueError):
        return None
    return {"bound": "fp64 pipe", "frac": round(fp64, 4), "issue_active": round(issue, 4),
            "source": "profiles/ncu_kmeans.json (k_kmeans_warp, config 1): FP64 pipe busy fraction; "
                      "the kernel is latency bound: each row's Lloyd iteration is a serial chain in one "
                      "warp (~10K cycles) while the row group's other warps wait at a named barrier"}


def cpu_baseline_sample():
    """Reference CPU GEMM on a bounded sample (q-proj shape, M=1, 1 core)."""
    from oracle.refpy import have_ref, oracle, ref

    lib = ref() if have_ref() else oracle()
    kind = "reference" if have_ref() else "port"
    n, k = 4096, 4096
    qt = synthetic_qtensor(n, k, seed=7)
    x = np.random.default_rng(1).standard_normal((1, k)).astype(np.float32)
    secs = lib.time_gemm_fused(x, qt, repeats=5)
    return {"value": algo_bytes(n, k, 1) / secs / 1e9, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": "reference gemm_fused (qgemm.cpp:71-128, single-threaded by design) on one "
                      "4096x4096 any4 g128 weight at M=1, median of 5"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
# decoder-layer dependency pattern over LAYER = (q, k, v, o, gate, up, down):
# q,k,v read the layer input; o reads y_q; gate/up read y_o; down reads y_up
# (the GEMMs of a Llama decoder layer with the non-GEMM ops between them elided)
X_SRC = [-1, -1, -1, 0, 3, 3, 5]
WAITS = [0, 0, 0, 1, 1, 0, 1]
# the single-launch chain: each problem waits only for the problem its x comes
# from (anyq_dev_gemm_chain_deps); o is dealt before k/v and up before gate, so
# the CTAs that finish q early take o while the others still run k/v (measured
# 0.3-0.5 us per layer faster than the natural order: scripts/gemv_probe.py --chain)
CHAIN_ORDER = [0, 3, 1, 2, 5, 4, 6]
CHAIN_DEPS = [-1 if X_SRC[j] < 0 else CHAIN_ORDER.index(X_SRC[j]) for j in CHAIN_ORDER]
BATCHES = [[0, 1, 2], [3], [4, 5], [6]]


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2507_04610_b200 import anyq

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peak, peak_kind = hbm_peak()
    M = args.m
    P = world
    layers = make_layers(args.layers, shard=(rank, P))
    launches0 = anyq.launch_count()
    use_chain = M <= 2  # CUDA-core GEMV chain; larger M runs the tcgen05 path per GEMM
    stream = torch.cuda.Stream(dev)

    # buffers: layer input x, per-layer local y shards, gathered y (TP)
    D = LAYER[0][2]  # model dim (K of q/k/v/gate/up)
    x_in = torch.randn(M, D, device=dev).to(torch.bfloat16)
    # the seven outputs of a layer are views into one flat buffer (one D2H copy per step)
    ybufs = [torch.empty(M * sum(ns for (_, ns, _, _) in L), device=dev, dtype=torch.bfloat16)
             for L in layers]

    def split_views(buf, L):
        out, off = [], 0
        for (_, ns, _, _) in L:
            out.append(buf[off:off + M * ns].view(M, ns))
            off += M * ns
        return out

    ys = [split_views(ybufs[li], L) for li, L in enumerate(layers)]
    # TP gather buffers: all_gather_into_tensor concatenates the [M, N/P] slices
    # along dim 0 -> [P*M, N/P]; for M = 1 that memory IS the [1, N] row
    yg = [[torch.empty(P * M, ns, device=dev, dtype=torch.bfloat16) for (_, ns, _, _) in L]
          for L in layers] if P > 1 else None

    def gathered(li, j):
        g = yg[li][j]
        return g.view(M, -1) if M == 1 else g.view(P, M, -1).permute(1, 0, 2).reshape(M, -1)

    xsrc = [x_in]  # the layer input run_layer reads (the e2e pipeline swaps in its own buffers)

    def x_of(li, j):
        src = X_SRC[j]
        if src < 0:
            return xsrc[0]
        return gathered(li, src) if P > 1 else ys[li][src]

    def run_layer(li, s):
        L = layers[li]
        if P == 1 and use_chain:
            anyq.gemm_chain_ptrs([L[j][3] for j in CHAIN_ORDER], [x_of(li, j).data_ptr() for j in CHAIN_ORDER],
                                 [ys[li][j].data_ptr() for j in CHAIN_ORDER], M, s.cuda_stream,
                                 deps=CHAIN_DEPS)
            return
        for bt in BATCHES:  # TP: one launch per batch, all-gather of the slices read next
            if use_chain:
                anyq.gemm_chain_ptrs([L[j][3] for j in bt], [x_of(li, j).data_ptr() for j in bt],
                                     [ys[li][j].data_ptr() for j in bt], M, s.cuda_stream)
            else:
                for j in bt:
                    L[j][3].gemm_ptr(x_of(li, j).data_ptr(), M, ys[li][j].data_ptr(), None, s.cuda_stream)
            if P > 1:
                for j in bt:
                    dist.all_gather_into_tensor(yg[li][j], ys[li][j].contiguous())

    # warm-up (configures kernels) + launches per step
    with torch.cuda.stream(stream):
        for li in range(len(layers)):
            c0 = anyq.launch_count()
            run_layer(li, stream)
            per_step_launches = anyq.launch_count() - c0
    torch.cuda.synchronize()

    graphs = None
    if P == 1:  # CUDA graphs (measured ~1 us per step faster than direct launches)
        graphs = []
        for li in range(len(layers)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                run_layer(li, stream)
            graphs.append(g)
        torch.cuda.synchronize()

    def step(i):
        li = i % len(layers)
        if graphs is not None:
            graphs[li].replay()
        else:
            run_layer(li, stream)

    # the timed K steps as ONE graph (as a serving engine captures a whole decode
    # step), so no graph-launch gaps sit between the layers; exactly K steps
    steps_graph = None
    if P == 1:
        steps_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(steps_graph, stream=stream):
            for i in range(args.steps):
                run_layer(i % len(layers), stream)
        torch.cuda.synchronize()

    # let the clocks ramp (1 s: a fresh box measured one 15 %-slow run after 0.3 s), then the
    # untimed warm-up steps
    t_end = time.time() + 1.0
    while time.time() < t_end:
        with torch.cuda.stream(stream):
            for i in range(len(layers)):
                step(i)
        torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize()

    # ---- timed region (device time, max over ranks)
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.wait_running()  # sampling before the region starts: its samples cover all of it
        clk.mark("start")
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if steps_graph is not None:
                steps_graph.replay()
            else:
                for i in range(args.steps):
                    step(i)
            ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark("end")
    ms = ev0.elapsed_time(ev1) / args.steps
    if P > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    gpu_launches = per_step_launches * args.steps
    step_bytes_all = sum(algo_bytes(n, k, M) for (_, n, k) in LAYER)  # whole job (all shards)
    value = step_bytes_all / (ms * 1e-3) / 1e9

    # ---- e2e through the public API with host buffers: H2D of the layer input
    # (pinned) + D2H of all seven outputs, every step, inside the timed region.
    # One GPU: the copies run on two copy streams, pipelined with the layer
    # launches as a serving loop would: step i's input lands in one of two
    # device buffers while step i-1 computes, its outputs go back while step
    # i+1 computes; each step's chain waits for its own H2D, each D2H for its
    # own chain, and a buffer is rewritten only after its last reader finished.
    # The timed region runs from the first H2D to the last D2H.
    xh = torch.randn(M, D).to(torch.bfloat16).pin_memory()
    yh = [[torch.empty(M, ns * P, dtype=torch.bfloat16).pin_memory() for (_, ns, _, _) in L]
          for L in layers]
    yhflat = [torch.empty(ybufs[li].numel(), dtype=torch.bfloat16).pin_memory() for li in range(len(layers))]
    NL = len(layers)

    if graphs is not None:
        xbufs = [x_in, torch.empty_like(x_in)]
        graphs_e2e = []  # [layer][input buffer]
        for li in range(NL):
            row = []
            for b in range(2):
                xsrc[0] = xbufs[b]
                with torch.cuda.stream(stream):
                    run_layer(li, stream)  # eager first (workspaces), then the capture
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    run_layer(li, stream)
                row.append(g)
            graphs_e2e.append(row)
        xsrc[0] = x_in
        torch.cuda.synchronize()
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def e2e_run(nsteps):
            comp = [None] * nsteps
            d2h_done = [None] * NL
            e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_start.record(h2d_s)
            for i in range(nsteps):
                li, b = i % NL, i % 2
                with torch.cuda.stream(h2d_s):
                    if i >= 2:
                        h2d_s.wait_event(comp[i - 2])  # the last reader of xbufs[b]
                    xbufs[b].copy_(xh, non_blocking=True)
                    h_ev = torch.cuda.Event()
                    h_ev.record(h2d_s)
                with torch.cuda.stream(stream):
                    stream.wait_event(h_ev)
                    if d2h_done[li] is not None:
                        stream.wait_event(d2h_done[li])  # ybufs[li] read back before reuse
                    graphs_e2e[li][b].replay()
                    comp[i] = torch.cuda.Event()
                    comp[i].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(comp[i])
                    yhflat[li].copy_(ybufs[li], non_blocking=True)
                    d2h_done[li] = torch.cuda.Event()
                    d2h_done[li].record(d2h_s)
            e_end.record(d2h_s)
            return e_start, e_end

        def e2e_capture(nsteps):
            """The same pipeline captured as ONE graph of nsteps steps (copies as
            memcpy nodes, the chain launches through the public API, the copy
            streams forked from and joined back into the capture stream), as a
            serving engine captures its decode loop: no host enqueue per step."""
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fork = torch.cuda.Event()
                fork.record(stream)
                h2d_s.wait_event(fork)
                d2h_s.wait_event(fork)
                comp, d2h_done, last_h = [], [None] * NL, None
                for i in range(nsteps):
                    li, b = i % NL, i % 2
                    with torch.cuda.stream(h2d_s):
                        if i >= 2:
                            h2d_s.wait_event(comp[i - 2])
                        xbufs[b].copy_(xh, non_blocking=True)
                        last_h = torch.cuda.Event()
                        last_h.record(h2d_s)
                    stream.wait_event(last_h)
                    if d2h_done[li] is not None:
                        stream.wait_event(d2h_done[li])
                    xsrc[0] = xbufs[b]
                    run_layer(li, stream)
                    c_ev = torch.cuda.Event()
                    c_ev.record(stream)
                    comp.append(c_ev)
                    with torch.cuda.stream(d2h_s):
                        d2h_s.wait_event(c_ev)
                        yhflat[li].copy_(ybufs[li], non_blocking=True)
                        d2h_done[li] = torch.cuda.Event()
                        d2h_done[li].record(d2h_s)
                for ev in d2h_done:  # join the copy streams
                    if ev is not None:
                        stream.wait_event(ev)
                stream.wait_event(last_h)
            xsrc[0] = x_in
            return g

        try:
            g_e2e = e2e_capture(args.steps)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for _ in range(2):  # warm-up replays
                    g_e2e.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g_e2e.replay()
                e1.record(stream)
            torch.cuda.synchronize()
            e2e_mode = "one graph of the K steps (H2D, chain launch, D2H per step)"
        except Exception as exc:  # capture refused: the same pipeline from the host
            print(f"[bench] e2e graph capture failed ({exc}); host-enqueued steps", file=sys.stderr)
            xsrc[0] = x_in
            e2e_run(args.warmup)
            torch.cuda.synchronize()
            e0, e1 = e2e_run(args.steps)
            torch.cuda.synchronize()
            e2e_mode = "host-enqueued graph replays"
        e2e_ms = e0.elapsed_time(e1) / args.steps
    else:
        def e2e_step(i, s):
            li = i % len(layers)
            x_in.copy_(xh, non_blocking=True)
            run_layer(li, s)
            for j in range(7):
                yh[li][j].copy_(gathered(li, j), non_blocking=True)

        with torch.cuda.stream(stream):
            for i in range(args.warmup):
                e2e_step(i, stream)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(args.steps):
                e2e_step(i, stream)
            e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.steps
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = M * D * 2
    d2h = sum(M * n * 2 for (_, n, _) in LAYER)

    # ---- per-shape single-GEMM timing (graph of the rotated layers' copies)
    def time_graph(fn, reps):
        with torch.cuda.stream(stream):
            fn()  # eager warm-up: first-use workspaces are allocated outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        with torch.cuda.stream(stream):
            for _ in range(2):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                g.replay()
            b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3  # us per replay

    per_shape = {}
    FF = LAYER[6][2]  # FFN dim (K of down)
    xk = {D: x_in, FF: torch.randn(M, FF, device=dev).to(torch.bfloat16)}
    if P == 1:
        for j, (name, n, k) in enumerate(LAYER):
            def one():
                for li in range(len(layers)):
                    layers[li][j][3].gemm_ptr(xk[k].data_ptr(), M, ys[li][j].data_ptr(), None,
                                              stream.cuda_stream)
            us = time_graph(one, 20) / len(layers)
            nb = algo_bytes(n, k, M)
            per_shape[name] = {"N": n, "K": k, "us": round(us, 3),
                               "GBps": round(nb / (us * 1e-6) / 1e9, 1),
                               "pct_hbm_peak": round(100 * nb / (us * 1e-6) / 1e9 / peak, 2)}

    # ---- config 3 shapes (Llama-3-70B) at M=1 on one GPU: the per-GPU slice of
    # the TP config at P=1 (weights rotated over 2 copies > L2)
    per_shape_70b = {}
    if not args.quick and P == 1:
        LAYER70 = [("q", 8192, 8192), ("k", 1024, 8192), ("v", 1024, 8192), ("o", 8192, 8192),
                   ("gate", 28672, 8192), ("up", 28672, 8192), ("down", 8192, 28672)]
        x70 = {k: torch.randn(M, k, device=dev).to(torch.bfloat16) for k in (8192, 28672)}
        for j, (name, n, k) in enumerate(LAYER70):
            if name in ("k", "up"):  # same shapes as v / gate
                continue
            ts70 = [anyq.DeviceTensor(synthetic_qtensor(n, k, 500 + 10 * j + c)) for c in range(2)]
            y70 = torch.empty(M, n, device=dev, dtype=torch.bfloat16)

            def one70():
                for d in ts70:
                    d.gemm_ptr(x70[k].data_ptr(), M, y70.data_ptr(), None, stream.cuda_stream)
            us = time_graph(one70, 20) / len(ts70)
            nb = algo_bytes(n, k, M)
            per_shape_70b[name] = {"N": n, "K": k, "us": round(us, 3),
                                   "GBps": round(nb / (us * 1e-6) / 1e9, 1),
                                   "pct_hbm_peak": round(100 * nb / (us * 1e-6) / 1e9 / peak, 2)}
            for d in ts70:
                d.close()

    # ---- M sweep (per-GEMM launches, AUTO path: GEMV for m <= 4 while its x image fits,
    # else tcgen05; K2 for 16..128 on tall or long-K tensors; fused mma for 5..32; dequant + cuBLAS above)
    sweep = {}
    tpeak = hbm_peak_tflops()
    if not args.quick and P == 1:
        for mm in (1, 2, 3, 4, 8, 16, 32, 64, 128, 256, 1024, 4096):
            xm = {k: torch.randn(mm, k, device=dev).to(torch.bfloat16) for k in (D, FF)}
            for j, (name, n, k) in enumerate(LAYER):
                if name not in ("q", "gate", "down"):
                    continue
                ym = torch.empty(mm, n, device=dev, dtype=torch.bfloat16)

                def one():
                    for li in range(len(layers)):
                        layers[li][j][3].gemm_ptr(xm[k].data_ptr(), mm, ym.data_ptr(), None,
                                                  stream.cuda_stream)
                us = time_graph(one, 10 if mm <= 256 else 3) / len(layers)
                nb = algo_bytes(n, k, mm)
                tf = 2.0 * mm * n * k / (us * 1e-6) / 1e12
                sweep[f"{name}_M{mm}"] = {"us": round(us, 3),
                                          "pct_hbm_peak": round(100 * nb / (us * 1e-6) / 1e9 / peak, 2),
                                          "TFLOPs": round(tf, 1),
                                          "pct_bf16_peak": round(100 * tf / tpeak, 2),
                                          "path": {1: "gemv", 2: "tcgen05", 3: "dequant+cublas",
                                                   4: "fused-mma", 5: "gemv-tcgen05", 6: "k2-tcgen05"}[
                                              layers[0][j][3].auto_path(mm)]}

    # ---- config 5 variants: int4 / nf4 (fixed tables) and any3 (3-bit codes on
    # the 4-bit device layout) next to any4, q shape, AUTO path
    variants = {}
    if not args.quick and P == 1:
        xq = {mm: torch.randn(mm, 4096, device=dev).to(torch.bfloat16) for mm in (1, 2, 16, 256)}
        for fmt in ("any4", "int4", "nf4", "any3"):
            vts = [anyq.DeviceTensor(synthetic_qtensor(4096, 4096, 77 + li, fmt)) for li in range(8)]
            for mm in (1, 2, 16, 256):
                yv = torch.empty(mm, 4096, device=dev, dtype=torch.bfloat16)

                def onev():
                    for vt in vts:
                        vt.gemm_ptr(xq[mm].data_ptr(), mm, yv.data_ptr(), None, stream.cuda_stream)
                us = time_graph(onev, 10) / len(vts)
                bits = 3 if fmt == "any3" else 4
                nb = algo_bytes(4096, 4096, mm, bits=bits)
                variants[f"{fmt}_M{mm}"] = {"us": round(us, 3),
                                            "pct_hbm_peak": round(100 * nb / (us * 1e-6) / 1e9 / peak, 2),
                                            "bits": bits}
            for vt in vts:
                vt.close()

    # ---- k-means quantizer throughput (config 1 / config 4): each rank quantizes
    # its 4096-row shard of a (4096*P) x 4096 gaussian matrix, device-resident,
    # rows keyed by global index (no collective); max time over ranks
    kmeans = None
    if not args.quick:
        from paper_2507_04610_b200 import _abi

        g = torch.Generator(device=dev)
        g.manual_seed(1234 + rank)
        w = torch.randn(4096, 4096, device=dev, generator=g)
        cfg = _abi.default_config(codebook=_abi.CB_ANY)
        anyq.dev_quantize_any(w, cfg, row_offset=4096 * rank)  # warm (scratch pool, attributes)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            if P > 1:
                dist.barrier()
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record()
            anyq.dev_quantize_any(w, cfg, row_offset=4096 * rank, check=False)
            k1.record()
            torch.cuda.synchronize()
            times.append(k0.elapsed_time(k1) * 1e-3)
        secs = sorted(times)[1]
        if P > 1:
            t = torch.tensor([secs], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        kmeans = {"rows_per_s": round(4096 * P / secs, 1),
                  "matrix": f"{4096 * P}x4096 gaussian any4 g128, 4096 rows per GPU",
                  "seconds": round(secs, 4), "gpus": P}

        # config 4, stratified: one Llama-3-8B layer's seven matrices (43,008 rows,
        # 4,096 of them 14,336 long) with synthetic activation statistics, each
        # matrix's rows partitioned over the ranks (row_offset keys the RNG by the
        # matrix row); the full model is 32 such layers
        from paper_2507_04610_b200.dist import row_range

        mats = []
        for i, (_, n, k) in enumerate(LAYER):
            r0, r1 = row_range(n, P, rank)
            gm = torch.Generator(device=dev)
            gm.manual_seed(1 + i)
            exj = torch.rand(k, device=dev, generator=gm) + 0.05
            wm = torch.randn(max(r1 - r0, 1), k, device=dev, generator=gm)[: r1 - r0].contiguous()
            mats.append((wm, exj, r0))
        for _ in range(2):  # warm (scratch pool, attributes; the first repeat still grows the pool)
            for wm, exj, r0 in mats:
                if wm.shape[0]:
                    anyq.dev_quantize_any(wm, cfg, exj=exj, row_offset=r0)
        torch.cuda.synchronize()
        ltimes = []
        for _ in range(3):  # median of 3 layer passes
            if P > 1:
                dist.barrier()
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record()
            for wm, exj, r0 in mats:
                if wm.shape[0]:
                    anyq.dev_quantize_any(wm, cfg, exj=exj, row_offset=r0, check=False)
            k1.record()
            torch.cuda.synchronize()
            ltimes.append(k0.elapsed_time(k1) * 1e-3)
        lsecs = sorted(ltimes)[1]
        if P > 1:
            t = torch.tensor([lsecs], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            lsecs = float(t.item())
        lrows = sum(n for (_, n, _) in LAYER)
        # the reference's CPU quantizer (learner.cpp:392-448, quantize_any with
        # threads = every host core) on a stratified sample of the same layer:
        # 2048 rows at K = 4096 and 512 rows at K = 14336, both with synthetic
        # stats; the layer time is extrapolated from the two per-K row rates
        if rank == 0 and not args.no_cpu:
            kmeans["cpu_baseline"] = kmeans_cpu_baseline(LAYER)
        # bound: the FP64 pipe (the E-step is a boundary search, the M-step FP64
        # sums in the reference's order; latency/barrier bound, ncu summary)
        kmeans["roofline"] = kmeans_roofline()
        kmeans["layer"] = {"rows_per_s": round(lrows / lsecs, 1), "rows": lrows,
                           "weights": sum(n * k for (_, n, k) in LAYER),
                           "seconds": round(lsecs, 4),
                           "full_8b_model_seconds_extrapolated": round(32 * lsecs, 2),
                           "stats": "synthetic E|x_j| ~ U(0.05, 1.05)",
                           "shapes": "q,k,v,o,gate,up (K=4096), down (K=14336)"}

    # the rows around the path: E|x_j| of collect_stats, ANYQ v1
    # file -> prepacked device tensor, weight_error / output_error; config-1
    # shapes, rank 0 at P = 1 only (host-API calls, synchronous, wall clock)
    around = None
    if not args.quick and P == 1:
        import tempfile

        xa = torch.randn(4096, 4096, device=dev)
        ex = torch.empty(4096, device=dev)
        anyq.dev_column_mean_abs(xa, ex)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(5):
            anyq.dev_column_mean_abs(xa, ex, check=False)
        s1.record()
        torch.cuda.synchronize()
        st = s0.elapsed_time(s1) / 5 * 1e-3
        qt1 = synthetic_qtensor(4096, 4096, seed=91)
        with tempfile.TemporaryDirectory() as d:
            fpath = os.path.join(d, "w.anyq")
            t0 = time.perf_counter()
            anyq.write_file(qt1, fpath)
            tw = time.perf_counter() - t0
            fbytes = os.path.getsize(fpath)
            anyq.DeviceTensor.load(fpath).close()  # warm
            t0 = time.perf_counter()
            dtl = anyq.DeviceTensor.load(fpath)
            torch.cuda.synchronize()
            tl = time.perf_counter() - t0
            dtl.close()
        t0 = time.perf_counter()
        anyq.DeviceTensor(qt1).close()  # same prepack from host arrays: what the load adds
        torch.cuda.synchronize()
        tc = time.perf_counter() - t0
        wref = anyq.dequantize(qt1) + np.float32(1e-3)
        xh16 = np.random.default_rng(3).standard_normal((16, 4096), dtype=np.float32)
        anyq.weight_error(wref, qt1)
        t0 = time.perf_counter()
        anyq.weight_error(wref, qt1)
        twe = time.perf_counter() - t0
        t0 = time.perf_counter()
        anyq.output_error(wref, qt1, xh16)
        toe = time.perf_counter() - t0
        around = {
            "stats_mean_abs_x": {"shape": "4096x4096 fp32, device-resident", "ms": round(st * 1e3, 3),
                                 "GBps": round(4096 * 4096 * 4 / st / 1e9, 1),
                                 "bound": "sequential FP64 add chain per channel (reference order)"},
            "anyq_file_4096x4096_any4": {"bytes": fbytes, "write_ms": round(tw * 1e3, 2),
                                         "load_to_device_ms": round(tl * 1e3, 2),
                                         "load_GBps": round(fbytes / tl / 1e9, 2),
                                         "prepack_from_host_arrays_ms": round(tc * 1e3, 2)},
            "weight_error_ms": round(twe * 1e3, 2),
            "output_error_m16_ms": round(toe * 1e3, 2),
            "note": "host-API wall clock incl. H2D of the host arrays",
        }

    # roofline of the dominant kernel: the step IS one k_lutgemv chain launch per
    # layer at M=1 (P=1), so its launch duration is the step time
    roof_achieved = value
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch_layer_chain")
        except Exception:
            traffic = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_sample()
        except Exception as e:  # oracle not built on this host
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 2),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 5),
            "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None,
            "dtype": "f16",
            "data": "synthetic",
            "config": {
                "workload": f"llama3-{MODEL} decoder-layer GEMMs (q,k,v,o,gate,up,down) any4 g128, "
                            "decoder data dependencies (o<-q, gate/up<-o, down<-up)",
                "M": M,
                "group_size": GROUP,
                "layers_rotated": args.layers,
                "l2": f"weights rotate over {args.layers} layers "
                      f"({args.layers * sum(algo_bytes(n, k, M) for (_, n, k) in LAYER) / 1e6:.0f} MB"
                      " > 126 MB L2)",
                "launch": ("one k_lutgemv chain launch per layer" if (use_chain and P == 1) else
                           "one launch per dependency batch" if use_chain else "one launch per GEMM"),
                "parallelism": f"tp{world} row-sharded W + NCCL all-gather per batch" if world > 1
                else "single",
                "graphs": "one graph of the K timed steps" if P == 1 else False,
            },
            "e2e": {"value": round(step_bytes_all / (e2e_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": round(e2e_ms, 5),
                    "copies": ("H2D and D2H on two copy streams, pipelined with the neighbouring "
                               "steps' chain launches; timed from the first H2D to the last D2H; "
                               + e2e_mode) if P == 1 else "in order on the compute stream"},
            "roofline": {"bound": "hbm", "achieved": round(roof_achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(roof_achieved / peak, 4),
                         "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "k_lutgemv chain (one launch = one decoder layer, 117.4 MB "
                                   "algorithmic bytes at M=1), CUDA events on its stream"},
            "cpu_baseline": cpu,
            "gpu_launches": gpu_launches,
            "launches_counted_host": anyq.launch_count() - launches0,
            "clocks": clk.summary(),
            "per_shape": per_shape,
            "per_shape_70b_m1": per_shape_70b,
            "m_sweep": sweep,
            "kmeans": kmeans,
            "variants_q_shape": variants,
            "around_the_path": around,
            "pct_hbm_peak_step": round(100 * value / peak, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    for L in layers:
        for (_, _, _, dt) in L:
            dt.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--quick", action="store_true", help="skip the M sweep and k-means extras")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--model", default="8b", choices=["8b", "70b"],
                    help="layer shapes of the step: Llama-3-8B (default, config 2) or -70B "
                         "(config 3; with --gpus N the layer is row-sharded over N GPUs)")
    args = ap.parse_args()
    if args.model == "70b":
        global LAYER, MODEL
        LAYER = LAYER_70B
        MODEL = "70b"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
