"""Bench: single-stream time steps/s of blocked SRU/QRNN inference vs T_b.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--block 32] [--mode f32]

One "step" = one pass of the hot path (a whole-sequence blocked forward,
``rnnb_forward``) over the workload's synthetic input; the metric is time
steps of the sequence per second, summed over GPUs.  Default workload is
BASELINE.json configs[1] (cfg2: QRNN w=2, D=H=1024, L=2048, fp32), which the
metric is quoted on; the headline T_b is --block and every T_b of the
config's sweep is reported under "sweep".

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events
on the launching stream; L2 (126 MB) is flushed by writing a 256 MB buffer
before every timed step (outside the events), so weights and inputs start
cold in HBM each step.  Barrier + synchronize around the timed region, max
over ranks.  nvidia-smi clocks are sampled during the timed region.  cfg2
does not shard (single layer, single stream): N>1 runs N independent
replicas (weak scaling).

--impl reference times the reference algorithm on the host CPU cores (the
C port of rnnblock's fast path under oracle/, all host threads) on a
bounded prefix of the same workload; rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1803_11389_b200 import workloads  # noqa: E402

METRIC = "single-stream time steps/sec vs block size T_b"
UNIT = "steps/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampling during the timed region


class ClockSampler:
    """SM clock + throttle reasons sampled every ~2 ms during the timed
    region through NVML (nvidia_ml_py), nvidia-smi as a fallback."""

    # NVML clocks-event-reason bits (nvml.h)
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], None, set()
        self._stop = threading.Event()
        self.thread = None
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, n in self.REASONS.items():
                            if bits & k:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            time.sleep(0.01)
        except Exception:
            self.nvml = None

    def stop(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        time.sleep(0.004)
        self._stop.set()
        self.thread.join(timeout=1)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 2 ms"}


# ---------------------------------------------------------------------------
# our arm


def roofline_for(w, T_b, mode, ms_per_launch, launches_per_step, pk, traffic, tc=None):
    """Dominant kernel = the fused layer kernel (one launch per layer).  The
    pipe follows the kernel that actually ran (`tc`: the tcgen05 kernel ran
    every layer); tensor-core modes that fell back to the FFMA kernel are
    rated against the CUDA-core peak."""
    if tc is None:
        tc = mode in ("bf16", "tf32", "f32x3")
    L = w.seq_len
    flops = workloads.flops_per_step(w) * L / launches_per_step
    s_w = {"f32": 4, "tf32": 4, "bf16": 2, "f64": 8, "f32x3": 8}[mode]
    s_a = 8 if mode == "f64" else 4
    params = workloads.param_count(w)
    nblocks = -(-L // T_b)
    # cold-cache traffic model (rnnblock traffic.py:26-27,64-68) + input/output once
    bytes_model = (params * s_w * nblocks + (w.X.shape[1] + w.layers[-1].d_h) * s_a * L) / launches_per_step
    sec = ms_per_launch / 1e3
    mhz = pk.get("sm_max_mhz", 1965.0)
    if not tc:
        # CUDA-core pipe: MEASURED_PEAKS.json has no CUDA-core figure, so use the
        # FFMA throughput measured on this pool by tools/ffma_peak.cu
        fp = os.path.join(REPO, "profiles", "ffma_peak.json")
        if os.path.exists(fp):
            with open(fp) as f:
                peak = json.load(f)["fma_peak_tflops"]
            src = ("measured: tools/ffma_peak2.cu packed FFMA2, 32 independent chains, profiles/ffma_peak.json "
                   "(0.96 of nominal)")
        else:
            peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
            src = f"nominal: 148 SMs x 128 lanes x 2 FLOP x {mhz:.0f} MHz"
        if mode == "f64":
            peak *= 0.5
            src += " x 0.5 (fp64 rate)"
        pipe = "fp64 dfma (CUDA cores)" if mode == "f64" else "fp32 ffma (CUDA cores)"
    else:
        peak = pk["bf16_tflops"] * (0.5 if mode in ("tf32", "f32x3") else 1.0)
        pipe = "tcgen05 " + mode
        src = "MEASURED_PEAKS.json bf16_tflops" + (" x 0.5 (tf32 rate)" if mode in ("tf32", "f32x3") else "")
        if mode == "f32x3":
            src += "; algorithmic FLOPs only (3 tf32 products per fp32 product executed)"
    achieved = flops / sec / 1e12
    hbm = pk["hbm_gbs"]
    # weight-stream roofline: the tensor-core kernel fetches every weight tile
    # from L2 once per block (the same bytes as the cold-cache model); rated
    # against the L2 read throughput measured by tools/l2_peak.cu
    l2 = None
    lp = os.path.join(REPO, "profiles", "l2_peak.json")
    if os.path.exists(lp):
        with open(lp) as f:
            l2 = json.load(f)["l2_read_gbs"]
    return {
        "bound": "tensor" if tc else "compute",
        "pipe": pipe,
        "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
        "frac": round(achieved / peak, 4), "peak_source": src,
        "traffic": traffic,
        "flops_per_launch": flops, "ms_per_launch": round(ms_per_launch, 5),
        "hbm_model": {
            "note": "reference cold-cache byte model (weights re-fetched every block); "
                    "the kernel keeps the weight slice SMEM/L2-resident, so this exceeds real DRAM traffic",
            "bytes_per_launch": bytes_model, "achieved_gbs": round(bytes_model / sec / 1e9, 1),
            "peak_gbs": hbm, "frac": round(bytes_model / sec / 1e9 / hbm, 4)},
        "l2_model": None if l2 is None else {
            "note": "same bytes against the measured L2 read throughput (profiles/l2_peak.json): the bound of "
                    "the tensor-core kernel, which streams each weight tile from L2 once per block",
            "achieved_gbs": round(bytes_model / sec / 1e9, 1), "peak_gbs": l2,
            "frac": round(bytes_model / sec / 1e9 / l2, 4)},
    }


def load_traffic(workload, T_b, mode):
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{workload}/{mode}/T{T_b}")
    return None if e is None else e["dram_bytes_per_launch"]


def time_sweep(st, X, out, blocks, args, rank, world, local_rank, flush, clocks_for=None):
    """Per T_b: W warm-up forwards, then K forwards each bracketed by CUDA
    events on the launching stream with an L2 flush in between (outside the
    events); max over ranks."""
    import torch
    stream = torch.cuda.current_stream()
    dev = X.device
    dist = world > 1
    results = {}
    for T_b in blocks:
        for _ in range(args.warmup):
            st.forward(X, T_b, out=out)
        torch.cuda.synchronize()
        launches = st.last_launches
        tc = [bool(st.query(9, li)) for li in range(st.n_layers)]
        ws = [bool(st.query(6, li)) for li in range(st.n_layers)]
        rg = [bool(st.query(10, li)) for li in range(st.n_layers)]
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        sampler = None
        if clocks_for == T_b and rank == 0:
            sampler = ClockSampler(local_rank)
            sampler.start()
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush, outside the events
            ev[i][0].record(stream)
            st.forward(X, T_b, out=out)
            ev[i][1].record(stream)
        if sampler is not None:
            # poll (GIL released between polls) so the sampler thread runs while the GPU works
            while not ev[-1][1].query():
                time.sleep(0.0005)
        torch.cuda.synchronize()
        if dist:
            torch.distributed.barrier()
        clocks = sampler.stop() if sampler is not None else None
        ms = [e0.elapsed_time(e1) for e0, e1 in ev]
        ms_step = sum(ms) / len(ms)
        if dist:
            t = torch.tensor([ms_step], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms_step = float(t.item())
        results[T_b] = {"ms_per_step": ms_step, "ms_min": min(ms), "launches": launches, "clocks": clocks,
                        "tcgen05": tc, "ffma_ws": ws, "ffma_reg": rg}
    return results


def kernel_name(r):
    if all(r.get("ffma_reg", [False])):
        return "ffma_reg (weights in registers, FFMA2, epilogue warp)"
    if all(r["tcgen05"]):
        return "tc_layer (tcgen05 + TMEM + TMA, look-back carry)"
    if all(r["ffma_ws"]):
        return "ffma_ws (TMA producer + mbarrier ring + epilogue warps)"
    return "ffma_layer"


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1803_11389_b200 as P

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workloads.make(args.workload)
    if w.bidirectional or w.proj is not None:
        raise SystemExit(f"bench workload {args.workload} is not a plain stack yet")
    st = P.DeviceStack(w.kind, w.layers, mode=args.mode, device=local_rank)
    dt = st.dtype
    X = torch.from_numpy(w.X.astype(st.np_dtype)).to(dev)
    L = w.seq_len
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    blocks = list(w.block_sizes) if args.sweep else []
    if args.block not in blocks:
        blocks.append(args.block)
    blocks = sorted(set(blocks))
    out = torch.empty((L, st.d_h[-1]), dtype=dt, device=dev)
    results = time_sweep(st, X, out, blocks, args, rank, world, local_rank, flush, clocks_for=args.block)

    # the same workload in the tensor-core numerics modes (reported beside, not the headline)
    extra = {}
    for m in [m for m in args.extra_modes.split(",") if m and m != args.mode]:
        sm = P.DeviceStack(w.kind, w.layers, mode=m, device=local_rank)
        outm = torch.empty((L, sm.d_h[-1]), dtype=sm.dtype, device=dev)
        Xm = X if sm.dtype == dt else X.to(sm.dtype)
        extra[m] = time_sweep(sm, Xm, outm, blocks, args, rank, world, local_rank, flush)
        sm.close()

    # end-to-end through the public C-ABI host entry point (pinned host buffers)
    dist = world > 1
    Xh = torch.from_numpy(w.X.astype(st.np_dtype)).pin_memory()
    Hh = torch.empty((L, st.d_h[-1]), dtype=dt).pin_memory()
    Xn, Hn = Xh.numpy(), Hh.numpy()
    for _ in range(max(1, args.warmup)):
        st.forward_host(Xn, args.block, out=Hn)
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e_steps = max(3, min(args.steps, 50))
    e_ts = []
    for _ in range(e_steps):
        t0 = time.perf_counter()
        st.forward_host(Xn, args.block, out=Hn)  # synchronises before returning
        e_ts.append((time.perf_counter() - t0) * 1e3)
    # median per call: host scheduling hiccups (a few % of calls) do not move it
    e2e_ms = statistics.median(e_ts)
    e2e_mean_ms = sum(e_ts) / len(e_ts)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    itemsize = np.dtype(st.np_dtype).itemsize
    e2e = {"value": round(L * world / (e2e_ms / 1e3), 1), "unit": UNIT,
           "h2d_bytes_per_step": int(L * w.X.shape[1] * itemsize),
           "d2h_bytes_per_step": int(L * st.d_h[-1] * itemsize),
           "ms_per_step": round(e2e_ms, 4), "ms_per_step_mean": round(e2e_mean_ms, 4),
           "timing": f"wall clock per call, median of {e_steps}",
           "api": "rnnb_forward_host (C ABI, pinned host X/H)"}

    if rank != 0:
        st.close()
        return None
    pk, pk_src = peaks()

    def sweep_of(res, mode):
        out_ = {}
        for T_b, r in res.items():
            rf = roofline_for(w, T_b, mode, r["ms_per_step"] / (r["launches"] or 1), r["launches"] or 1,
                              pk, None, tc=all(r["tcgen05"]))
            out_[str(T_b)] = {"steps_per_s": round(L * world / (r["ms_per_step"] / 1e3), 1),
                              "ms_per_step": round(r["ms_per_step"], 5), "frac": rf["frac"],
                              "tflops": rf["achieved"], "pipe": rf["pipe"], "kernel": kernel_name(r),
                              "hbm_model_frac": rf["hbm_model"]["frac"],
                              "l2_model_frac": rf["l2_model"]["frac"] if rf["l2_model"] else None}
        return out_

    head = results[args.block]
    roof = roofline_for(w, args.block, args.mode, head["ms_per_step"] / (head["launches"] or 1),
                        head["launches"] or 1, pk, load_traffic(args.workload, args.block, args.mode),
                        tc=all(head["tcgen05"]))
    roof["peaks_file"] = pk_src
    resident = [bool(st.query(3, li)) for li in range(st.n_layers)]
    line = {
        "metric": METRIC, "value": round(L * world / (head["ms_per_step"] / 1e3), 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(head["ms_per_step"], 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.mode,
        "data": "synthetic (seeded PCG64, BASELINE.json distributions)",
        "config": {"workload": args.workload, "cell": w.kind.value, "d_in": int(w.X.shape[1]),
                   "d_h": int(w.layers[-1].d_h), "n_layers": len(w.layers), "seq_len": L,
                   "block_size": args.block, "mode": args.mode,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "flushed before every timed step (256 MB write)",
                   "weights_smem_resident": resident,
                   "units_per_cta": [st.query(2, li) for li in range(st.n_layers)],
                   "grid": [st.query(4, li) for li in range(st.n_layers)],
                   "kernel": kernel_name(head)},
        "e2e": e2e,
        "gpu_launches": int(head["launches"] * args.steps),
        "roofline": roof,
        "sweep": sweep_of(results, args.mode),
        "modes": {m: sweep_of(r, m) for m, r in extra.items()},
        "clocks": head["clocks"],
    }
    if args.cpu_baseline and world == 1:  # the CPU baseline is a rank-0, N=1 measurement
        line["cpu_baseline"] = cpu_baseline(args, w, sample_steps=args.cpu_sample)
    st.close()
    return line


# ---------------------------------------------------------------------------
# partitioned configs across ranks: the fused peer-memory partitions (p2p.py)


def run_partitioned(args, rank, world, local_rank):
    """BASELINE cfg4 (--partition pipeline: layer pipeline of time chunks) or
    cfg5 (--partition hidden: hidden-dimension sharding with the all-gather
    in the epilogue) over the ranks, one GPU each (CUDA IPC between the rank
    processes; BENCH_SHARE_GPU=1 puts every rank on cuda:0 to exercise the
    path).  Strong scaling: the whole sequence per step, time = max over
    ranks of the device time per step."""
    import torch
    import torch.distributed as dist
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import p2p
    from paper_1803_11389_b200.partition import layer_ranges

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workloads.make(args.workload)
    L = w.seq_len
    last = rank == world - 1
    if args.partition == "pipeline":
        if w.bidirectional or w.proj is not None:
            raise SystemExit("--partition pipeline needs a plain stack (cfg4)")
        lo, hi = layer_ranges(len(w.layers), world)[rank]
        st = P.DeviceStack(w.kind, w.layers[lo:hi], mode=args.mode, device=local_rank)
        obj = p2p.P2PPipelineStage(st, rank, world, args.chunk, args.block, slots=2)
        X = torch.from_numpy(w.X).to(dev) if rank == 0 else None
        out = torch.empty((L, st.d_h[-1]), dtype=torch.float32, device=dev) if last else None
        d_in, d_out = int(w.X.shape[1]), int(w.layers[-1].d_h)

        def step():
            obj.enqueue(L, X, out)
            obj.advance(L)
            obj.finish()
        par = f"pipeline{world} (layers {lo}..{hi - 1} on rank {rank}, chunk {args.chunk})"
    else:
        if not w.bidirectional:
            raise SystemExit("--partition hidden needs the bidirectional stack (cfg5)")
        obj = p2p.P2PBidirSRU(w.layers, w.layers_bwd, rank, world, args.block, args.mode, L, device=local_rank)
        X = torch.from_numpy(w.X).to(dev)
        out = torch.empty((L, 2 * obj.H), dtype=torch.float32, device=dev)
        d_in, d_out = int(w.X.shape[1]), 2 * obj.H

        def step():
            obj.enqueue(X, out)
            obj.close_call()
            torch.cuda.current_stream(dev).wait_stream(obj.stream)
        par = f"hidden{world} (units {obj.u0}..{obj.u1 - 1} of each direction on rank {rank})"
    if world > 1:
        obj.connect_ipc()
    else:
        obj.connect_local([obj])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.start()
    for i in range(args.steps):
        flush.fill_(float(i))
        ev[i][0].record()
        step()
        ev[i][1].record()
    while not ev[-1][1].query():
        time.sleep(0.0005)
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    # end to end: rank 0 copies the sequence in from pinned host memory, the
    # ranks holding the output copy it out; wall clock, max over ranks
    Xh = torch.from_numpy(w.X).pin_memory() if X is not None else None
    Oh = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory() if out is not None else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        if Xh is not None:
            X.copy_(Xh, non_blocking=True)
        step()
        if Oh is not None and (last if args.partition == "pipeline" else rank == 0):
            Oh.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
    if world > 1:
        t = torch.tensor([ms, e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), float(t[1])
    # this rank's kernel launches per step (layer kernels + operand copies + flag signals)
    if args.partition == "pipeline":
        n_chunks = -(-L // args.chunk)
        launches = n_chunks * (obj.stack.last_launches + (rank < world - 1) + (rank > 0))
    else:
        per_dir = [st_.last_launches for st_ in obj.stages[-1]]
        launches = len(obj.stages) * (sum(per_dir) + 1 + world) + 1
    obj.close()
    if rank != 0:
        return None
    pk, pk_src = peaks()
    flops = workloads.flops_per_step(w) * L
    tc = args.mode in ("bf16", "tf32")
    peak = (pk["bf16_tflops"] * (0.5 if args.mode == "tf32" else 1.0)) if tc else 71.29
    achieved = flops / (ms / 1e3) / 1e12
    itemsize = 4
    return {
        "metric": METRIC, "value": round(L / (ms / 1e3), 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.mode,
        "data": "synthetic (seeded PCG64, BASELINE.json distributions)",
        "config": {"workload": args.workload, "seq_len": L, "block_size": args.block, "mode": args.mode,
                   "parallelism": par, "transport": "fused epilogue stores to CUDA-IPC-mapped peer buffers + "
                   "stream-ordered flags" if world > 1 else "single rank (no peers)",
                   "l2": "flushed before every timed step (256 MB write)"},
        "e2e": {"value": round(L / (e2e_ms / 1e3), 1), "unit": UNIT,
                "h2d_bytes_per_step": int(L * d_in * itemsize),
                "d2h_bytes_per_step": int(L * d_out * itemsize),
                "ms_per_step": round(e2e_ms, 4), "api": "p2p partition objects, pinned host X / output"},
        "gpu_launches": int(launches * args.steps),
        "roofline": {"bound": "tensor" if tc else "compute", "achieved": round(achieved, 2),
                     "peak": round(peak * world, 1), "unit": "TFLOP/s", "frac": round(achieved / (peak * world), 4),
                     "peak_source": ("MEASURED_PEAKS.json" if tc else "profiles/ffma_peak.json") + f" x {world} GPUs",
                     "traffic": None},
        "clocks": clocks,
    }


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle port of rnnblock's fast path


def _oracle():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    O.lib()
    return O


def cpu_baseline(args, w, sample_steps):
    O = _oracle()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    L = min(sample_steps, w.seq_len)
    X = np.ascontiguousarray(w.X[:L])
    layers = [lay.mats() for lay in w.layers]
    O.run_blocked(w.kind.value, layers, X, args.block)  # warm-up
    times = []
    t_end = time.perf_counter() + args.cpu_seconds
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        O.run_blocked(w.kind.value, layers, X, args.block)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": round(L / med, 1), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{args.workload} first {L} of {w.seq_len} steps, T_b={args.block}, "
                      f"median of {len(times)} runs, oracle/ C port of rnnblock fast kernel, "
                      f"OpenMP {cores} threads"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    w = workloads.make(args.workload)
    O = _oracle()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    L = min(args.cpu_sample, w.seq_len)
    X = np.ascontiguousarray(w.X[:L])
    layers = [lay.mats() for lay in w.layers]
    for _ in range(args.warmup):
        O.run_blocked(w.kind.value, layers, X, args.block)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.run_blocked(w.kind.value, layers, X, args.block)
        ts.append(time.perf_counter() - t0)
    ms = sum(ts) / len(ts) * 1e3
    v = round(L / (ms / 1e3), 1)
    sample = (f"{args.workload} first {L} of {w.seq_len} steps per step, T_b={args.block}; "
              f"oracle/ C port of rnnblock's fast path (numba prange -> OpenMP), {cores} threads")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded PCG64, BASELINE.json distributions)",
            "config": {"workload": args.workload, "block_size": args.block, "mode": "f32",
                       "seq_len_sample": L},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--block", type=int, default=32)
    ap.add_argument("--mode", default="f32", choices=("f32", "f64", "bf16", "tf32"))
    ap.add_argument("--no-sweep", dest="sweep", action="store_false")
    ap.add_argument("--extra-modes", default="bf16,tf32,f32x3",
                    help="tensor-core numerics modes timed beside the headline mode")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-sample", type=int, default=512, help="time steps in the CPU sample")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--partition", choices=("replicas", "pipeline", "hidden"), default="replicas",
                    help="replicas: N independent copies of the workload (cfg1/cfg2 do not shard); "
                         "pipeline: cfg4 layer pipeline across ranks; hidden: cfg5 hidden sharding")
    ap.add_argument("--chunk", type=int, default=4096, help="pipeline chunk (steps, a multiple of --block)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: W < 3 warm-up steps violates the timing rules; using 3")
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo + BENCH_SHARE_GPU=1: exercise the N>1 code path
    # with independent replicas sharing one GPU (host-logic check only; the
    # driver's scaling runs use nccl, one GPU per rank)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if os.environ.get("BENCH_SHARE_GPU") == "1":
        local_rank = 0
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            else:
                dist.init_process_group(backend)
        if args.partition == "replicas":
            line = run_ours(args, rank, world, local_rank)
        else:
            line = run_partitioned(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
