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


def _json(name):
    p = os.path.join(REPO, "profiles", name)
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def ffma_peak():
    d = _json("ffma_peak.json")
    if d:
        return d["fma_peak_tflops"], ("measured: tools/ffma_peak2.cu packed FFMA2, 32 independent chains, "
                                      "profiles/ffma_peak.json (0.96 of nominal)")
    return 148 * 128 * 2 * 1965e6 / 1e12, "nominal: 148 SMs x 128 lanes x 2 FLOP x 1965 MHz"


def mma_floor_cycles(kind="f16"):
    """Cycles per tcgen05.mma (M=128, one K-step, both operands in shared
    memory) measured by tools/mma_rate.cu (profiles/mma_rate_r2.json): a
    floor of ~51 cycles for any N <= 64, N/2 cycles above (math-bound)."""
    d = _json("mma_rate_r2.json")
    if d:
        cg = 10 if kind == "tf32" else 1
        rows = [r for r in d["rows"] if r["cta_group"] == cg and r["M"] == 128 and r["N"] <= 64]
        if rows:
            return max(r["cycles_per_mma"] for r in rows), "measured: tools/mma_rate.cu, profiles/mma_rate_r2.json"
    return 51.3, "tools/mma_rate.cu round-2 measurement (51.3 cycles)"


def tc_pick_n(T):
    return 16 if T <= 16 else 32 if T <= 32 else 64 if T <= 64 else 128


def roofline_for(w, T_b, mode, ms_per_launch, launches_per_step, pk, traffic, tc=None, sm_mhz=None, nt=None,
                 reg=False):
    """Roofline of the dominant kernel, per regime:

    * tcgen05 path (bf16 / tf32 / fp32-accurate 3xTF32): the weights are
      streamed into the tensor pipe once per block, so the applicable bound
      is the slower of (a) the MMA instruction floor -- every 128 x N x K-step
      MMA takes max(51 cycles, N/2) (tools/mma_rate.cu): below N = 128 the
      pipe runs at N/102 of its peak -- and (b) the L2 -> shared-memory feed
      of the weight and x tiles (measured 23.9 TB/s, tools/l2_tma_peak.cu).
      `peak` is the algorithmic TFLOP/s that bound allows at this T_b;
      the nominal tensor peak (MEASURED_PEAKS.json bf16) is reported beside.
    * FFMA path (fp32 / f64 on CUDA cores): the FMA pipe (measured FFMA2 peak).
    The reference's cold-cache byte model (traffic.py:26-27) is reported as
    bytes only -- it describes the CPU, not these kernels."""
    if tc is None:
        tc = mode in ("bf16", "tf32", "f32x3")
    L = w.seq_len
    flops = workloads.flops_per_step(w) * L / launches_per_step
    sec = ms_per_launch / 1e3
    mhz = sm_mhz or pk.get("sm_max_mhz", 1965.0)
    achieved = flops / sec / 1e12
    s_w = {"f32": 4, "tf32": 4, "bf16": 2, "f64": 8, "f32x3": 8, "f32_ffma": 4}[mode]
    s_a = 8 if mode == "f64" else 4
    params = workloads.param_count(w)
    cold = (params * s_w * -(-L // T_b) + (w.X.shape[1] + w.layers[-1].d_h) * s_a * L) / launches_per_step
    out = {"traffic": traffic, "flops_per_launch": flops, "ms_per_launch": round(ms_per_launch, 5),
           "reference_cold_cache_bytes_per_launch": cold}
    if tc:
        x3 = mode in ("f32", "f32x3")
        T_eff = min(T_b, 32) if x3 else T_b  # 3xTF32 runs blocks of at most 32 steps
        N = tc_pick_n(T_eff)
        KT, es, kstep = (64, 2, 16) if mode == "bf16" else (32, 4, 8)
        planes = 2 if x3 else 1
        floor_cyc, floor_src = mma_floor_cycles("f16" if mode == "bf16" else "tf32")
        cyc = max(floor_cyc, (2 * N if x3 else N) / 2)
        n_instr = 0.0
        l2_bytes = 0.0
        taps = 2 if w.kind.value == "qrnn" else 1
        for lay in w.layers + (w.layers_bwd if w.bidirectional else []):
            nU = -(-lay.d_h // 128)
            nK = taps * -(-lay.d_in // KT)
            nB = -(-L // T_eff)
            # 3xTF32 issues 2 MMAs per gate and K-step: W_hi.[x_hi | x_lo] (N' = 2N) + W_lo.x_hi
            n_instr += nU * nB * nK * 3 * (KT // kstep) * (2 if x3 else 1)
            l2_bytes += nU * nB * nK * planes * (3 * 128 + N) * KT * es
        n_instr /= launches_per_step
        l2_bytes /= launches_per_step
        t_mma = n_instr * cyc / 148 / (mhz * 1e6)
        l2j = _json("l2_peak.json") or {}
        l2 = max(l2j.get("l2_read_gbs", 23887.0), l2j.get("l2_tma_tile_gbs_in_kernel", 0.0))
        t_l2 = l2_bytes / (l2 * 1e9)
        t_bound = max(t_mma, t_l2)
        nominal = pk["bf16_tflops"] * (1.0 if mode == "bf16" else 0.5)
        out.update({
            "bound": "tensor", "pipe": "tcgen05 " + ("3xTF32 (fp32-accurate)" if x3 else mode),
            "achieved": round(achieved, 3), "peak": round(flops / t_bound / 1e12, 2), "unit": "TFLOP/s",
            "frac": round(t_bound / sec, 4),
            "peak_source": (f"tcgen05 weight stream at N={N}: max(MMA issue floor {cyc:.1f} cycles x "
                            f"{n_instr:.3g} MMAs / 148 SMs at {mhz:.0f} MHz = {t_mma * 1e6:.1f} us, "
                            f"L2->SMEM tiles {l2_bytes / 1e9:.3g} GB / {l2:.0f} GB/s = {t_l2 * 1e6:.1f} us); "
                            + floor_src),
            "tensor_issue": {"mma_instructions": n_instr, "cycles_per_mma": cyc, "floor_us": round(t_mma * 1e6, 2),
                             "frac": round(t_mma / sec, 4)},
            "l2_feed": {"bytes": l2_bytes, "peak_gbs": l2, "achieved_gbs": round(l2_bytes / sec / 1e9, 1),
                        "frac": round(t_l2 / sec, 4)},
            "tensor_nominal": {"peak_tflops": nominal, "frac": round(achieved * (3 if x3 else 1) / nominal, 4),
                               "note": "issued MMA work (3 products per fp32 product for 3xTF32) vs MEASURED_PEAKS "
                                       "bf16 (x0.5 for tf32): reachable only with N >= 128, i.e. T_b >= 128"},
        })
        return out
    peak, src = ffma_peak()
    if mode == "f64":
        peak *= 0.5
        src += " x 0.5 (fp64 rate)"
    # FFMA kernels keep a layer's weights in shared memory and read each weight
    # once per pass of min(T_b, 32) time steps: at small T_b the applicable
    # bound is that SHARED-MEMORY weight stream (north_star's "weight bandwidth
    # for small T_b"), not the FMA pipe.  Peak: tools/lds_bench.cu, 16-byte
    # loads at 1.067 cycles per warp and scheduler = 120 B/clk/SM.
    lds = _json("lds_bench_r1.json")
    lds_bpc = 120.0
    if lds:
        best = min(r["clk_per_warp_lds"] for r in lds["rows"] if r["bytes"] == 16)
        lds_bpc = 512.0 / (4.0 * best)
    smem_gbs = 148 * lds_bpc * mhz * 1e6 / 1e9
    t_pass = min(T_b, 32)
    smem_bytes = params * s_w * -(-L // t_pass) / launches_per_step
    t_smem = 0.0 if reg else smem_bytes / (smem_gbs * 1e9)  # ffma_reg: the weights live in registers
    t_fma = flops / (peak * 1e12)
    t_bound = max(t_smem, t_fma)
    smem_bound = t_smem > t_fma
    out.update({"bound": "smem" if smem_bound else "compute",
                "pipe": ("shared-memory weight stream (weights resident in SMEM, read once per block)" if smem_bound
                         else "fp64 dfma (CUDA cores)" if mode == "f64" else "fp32 ffma (CUDA cores)"),
                "achieved": round(achieved, 3), "peak": round(flops / t_bound / 1e12, 2), "unit": "TFLOP/s",
                "frac": round(t_bound / sec, 4),
                "peak_source": (f"max(FMA pipe {peak:.1f} TFLOP/s [{src}] = {t_fma * 1e6:.1f} us, shared-memory weight "
                                f"stream {smem_bytes / 1e9:.3g} GB / {smem_gbs:.0f} GB/s [tools/lds_bench.cu: "
                                f"{lds_bpc:.0f} B/clk/SM] = {t_smem * 1e6:.1f} us)"),
                "fma_pipe": {"peak_tflops": round(peak, 2), "frac": round(achieved / peak, 4)},
                "smem_weight_stream": {"bytes": smem_bytes, "peak_gbs": round(smem_gbs, 1),
                                       "achieved_gbs": round(smem_bytes / sec / 1e9, 1),
                                       "frac": round(t_smem / sec, 4)}})
    sw = _json("ncu_sweep_r1.json")
    if sw and w.name == "cfg2" and mode in ("f32", "f32_ffma"):
        for r in sw["rows"]:
            if r["mode"] == "f32" and r["T_b"] == T_b:
                cycles = r["us"] * 1e-6 * mhz * 1e6 * 148
                out["smem_pipe"] = {
                    "frac": round(r["smem_wavefronts_M"] * 1e6 / cycles, 4),
                    "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared / SM cycles, profiles/ncu_sweep_r1.json "
                              "(cfg2 f32, same kernel): the shared-memory pipe that feeds the resident weights"}
    return out


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
    if any(r["tcgen05"]):
        return "mixed (tc_layer / ffma)"
    if all(r["ffma_ws"]):
        return "ffma_ws (TMA producer + mbarrier ring + epilogue warps)"
    return "ffma_layer"


CONFIG_LINES = (("cfg1", "f32", (1, 4, 16)), ("cfg3", "f32", (1, 8, 32)), ("cfg3", "bf16", (1, 8, 32)),
                ("cfg3", "tf32", (8, 32)), ("cfg4", "f32", (32,)), ("cfg4", "bf16", (32,)),
                ("cfg5", "bf16", (16, 64)))


def time_configs(args, local_rank, pk, mhz):
    """Every other BASELINE config on this GPU (whole-model forwards: cfg3 =
    projection + 6 SRU + logits, cfg5 = the fused sharded bidirectional
    stack at G = 1), L2 flushed before every timed step; kernel recorded."""
    import torch
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import p2p
    from paper_1803_11389_b200.acoustic import AcousticSRU
    dev = torch.device("cuda", local_rank)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    steps = max(3, min(args.steps, 10))
    out = {}
    cache = {}
    for name, mode, blocks in CONFIG_LINES:
        if name not in cache:
            cache.clear()
            cache[name] = workloads.make(name)
        w = cache[name]
        L = w.seq_len
        X = torch.from_numpy(w.X).to(dev)
        if name == "cfg3":
            obj = AcousticSRU(w.proj, w.layers, w.logits, mode=mode, device=local_rank)
            run = lambda T: obj.forward(X, T)  # noqa: E731
            stack = obj.stack
        elif name == "cfg5":
            obj = p2p.P2PBidirSRU(w.layers, w.layers_bwd, 0, 1, blocks[0], mode, L, device=local_rank)
            obj.connect_local([obj])

            def run(T, obj=obj):
                obj.block_size = T
                return obj.forward(X)
            stack = obj.stages[0][0]
        else:
            obj = P.DeviceStack(w.kind, w.layers, mode=mode, device=local_rank)
            run = lambda T: obj.forward(X, T)  # noqa: E731
            stack = obj
        rows = {}
        for T in blocks:
            for _ in range(3):
                run(T)
            torch.cuda.synchronize()
            tc = [bool(stack.query(9, li)) for li in range(stack.n_layers)]
            reg = [bool(stack.query(10, li)) for li in range(stack.n_layers)]
            wsk = [bool(stack.query(6, li)) for li in range(stack.n_layers)]
            wst = [bool(stack.query(11, li)) for li in range(stack.n_layers)]
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for i in range(steps):
                flush.fill_(float(i))
                ev[i][0].record()
                run(T)
                ev[i][1].record()
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev) / steps
            rf = roofline_for(w, T, mode, ms, 1, pk, None, tc=all(tc), sm_mhz=mhz, reg=all(reg))
            kern = ("tc_layer (tcgen05)" if all(tc) else "ffma_reg (register-resident)" if all(reg)
                    else "ffma_ws weight-streaming" if all(wst) else "ffma_ws (SMEM-resident)" if all(wsk)
                    else "ffma_layer")
            rows[str(T)] = {"steps_per_s": round(L / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
                            "tflops": rf["achieved"], "frac": rf["frac"], "bound": rf["bound"],
                            "peak_tflops": rf["peak"], "kernel": kern}
        out[f"{name}/{mode}"] = {"seq_len": L, "blocks": rows}
        obj.close()
        del obj, X
        torch.cuda.empty_cache()
    return out


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

    # the same workload in the other numerics modes (reported beside, not the
    # headline); "f32_ffma" = fp32 mode held on the FFMA kernels at every T_b
    extra = {}
    for m in [m for m in args.extra_modes.split(",") if m and m != args.mode]:
        real = "f32" if m == "f32_ffma" else m
        if m == "f32_ffma":
            os.environ["RNNB_F32_TC"] = "0"
        sm = P.DeviceStack(w.kind, w.layers, mode=real, device=local_rank)
        outm = torch.empty((L, sm.d_h[-1]), dtype=sm.dtype, device=dev)
        Xm = X if sm.dtype == dt else X.to(sm.dtype)
        extra[m] = time_sweep(sm, Xm, outm, blocks, args, rank, world, local_rank, flush)
        sm.close()
        os.environ.pop("RNNB_F32_TC", None)

    # end-to-end through the public C-ABI host entry point (pinned host buffers)
    dist = world > 1
    Xh = torch.from_numpy(w.X.astype(st.np_dtype)).pin_memory()
    Hh = torch.empty((L, st.d_h[-1]), dtype=dt).pin_memory()
    Xn, Hn = Xh.numpy(), Hh.numpy()
    # (the leg follows the sweeps' stack teardowns and the pinned allocations:
    # a longer warm-up lets the driver settle before the timed calls)
    for _ in range(max(20, args.warmup) if args.e2e else 0):
        st.forward_host(Xn, args.block, out=Hn)
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e_steps = max(3, min(args.steps, 100))
    e_ts = [float("nan")] if not args.e2e else []
    for _ in range(e_steps if args.e2e else 0):
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
    e2e = None if not args.e2e else {
           "value": round(L * world / (e2e_ms / 1e3), 1), "unit": UNIT,
           "h2d_bytes_per_step": int(L * w.X.shape[1] * itemsize),
           "d2h_bytes_per_step": int(L * st.d_h[-1] * itemsize),
           "ms_per_step": round(e2e_ms, 4), "ms_per_step_mean": round(e2e_mean_ms, 4),
           "timing": f"wall clock per call, median of {e_steps}",
           "api": "rnnb_forward_host (C ABI, pinned host X/H)"}

    # the partitioned BASELINE configs across all ranks (cfg4 layer pipeline,
    # cfg5 hidden sharding): strong scaling; at N = 1 these are the anchors
    partitioned = {}
    if args.partitioned:
        for part, wl in (("pipeline", "cfg4"), ("hidden", "cfg5")):
            blk = 32 if part == "pipeline" else 64
            partitioned[part] = run_partitioned(args, rank, world, local_rank, workload=wl, partition=part,
                                                mode="bf16", block=blk, chunk=args.chunk)
    # the reference-facing drop-in call (run_blocked, blocked.py:221-268):
    # host arrays in and out, and -- as the reference re-stacks its weights
    # on every call -- a full weight upload/repack per call
    dropin = None
    if rank == 0 and args.dropin:
        cfg_ = P.RnnConfig(w.kind, int(w.X.shape[1]), int(w.layers[-1].d_h), n_layers=len(w.layers),
                           precision="f32")
        ws_ = P.WeightSet(w.kind, "f32", w.layers)
        Xf = np.ascontiguousarray(w.X, np.float32)
        P.run_blocked(cfg_, ws_, Xf, args.block)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            P.run_blocked(cfg_, ws_, Xf, args.block)
            ts.append((time.perf_counter() - t0) * 1e3)
        dms = statistics.median(ts)
        dropin = {"value": round(L / (dms / 1e3), 1), "unit": UNIT, "ms_per_call": round(dms, 3),
                  "api": "paper_1803_11389_b200.run_blocked (reference signature; weights uploaded and "
                         "repacked on every call, as the reference re-stacks them)"}
    if rank != 0:
        st.close()
        return None
    pk, pk_src = peaks()

    head = results[args.block]
    mhz = (head["clocks"] or {}).get("sm_mhz")

    def sweep_of(res, mode):
        out_ = {}
        for T_b, r in res.items():
            rf = roofline_for(w, T_b, mode, r["ms_per_step"] / (r["launches"] or 1), r["launches"] or 1,
                              pk, None, tc=all(r["tcgen05"]), sm_mhz=mhz, reg=all(r.get("ffma_reg", [False])))
            row = {"steps_per_s": round(L * world / (r["ms_per_step"] / 1e3), 1),
                   "ms_per_step": round(r["ms_per_step"], 5), "frac": rf["frac"], "bound": rf["bound"],
                   "tflops": rf["achieved"], "peak_tflops": rf["peak"], "pipe": rf["pipe"],
                   "kernel": kernel_name(r)}
            if "smem_pipe" in rf:
                row["smem_pipe_frac"] = rf["smem_pipe"]["frac"]
            if rf["bound"] == "tensor":
                row["tensor_issue_frac"] = rf["tensor_issue"]["frac"]
                row["l2_feed_frac"] = rf["l2_feed"]["frac"]
            out_[str(T_b)] = row
        return out_

    roof = roofline_for(w, args.block, args.mode, head["ms_per_step"] / (head["launches"] or 1),
                        head["launches"] or 1, pk, load_traffic(args.workload, args.block, args.mode),
                        tc=all(head["tcgen05"]), sm_mhz=mhz, reg=all(head.get("ffma_reg", [False])))
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
    if dropin:
        line["dropin"] = dropin
    if partitioned:
        line["partitioned"] = partitioned
    if args.configs and world == 1:
        line["configs"] = time_configs(args, local_rank, pk, mhz)
    if args.cpu_baseline and world == 1:  # the CPU baseline is a rank-0, N=1 measurement
        line["cpu_baseline"] = cpu_baseline(args, w, sample_steps=args.cpu_sample)
    st.close()
    return line


# ---------------------------------------------------------------------------
# partitioned configs across ranks: the fused peer-memory partitions (p2p.py)


def run_partitioned(args, rank, world, local_rank, workload=None, partition=None, mode=None, block=None,
                    chunk=None):
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

    import copy
    args = copy.copy(args)
    for k, v in (("workload", workload), ("partition", partition), ("mode", mode), ("block", block),
                 ("chunk", chunk)):
        if v is not None:
            setattr(args, k, v)
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
    # the bound that applies at this T_b (tcgen05 weight stream, see roofline_for), split over the ranks
    rfa = roofline_for(w, args.block, args.mode, ms * world, 1, pk, None, tc=tc) if tc else None
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
                     "peak_source": ("MEASURED_PEAKS.json" if tc else "profiles/ffma_peak.json") + f" x {world} GPUs"
                                    + " (nominal tensor peak: reachable only with N >= 128)" * bool(tc),
                     "applicable": None if rfa is None else {
                         "what": "tcgen05 weight stream at this T_b (MMA issue floor / L2 feed), per-GPU bound / N GPUs",
                         "peak": round(rfa["peak"] * world, 1), "frac": rfa["frac"]},
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _time_oracle(O, w, X, T_b, seconds):
    layers = [lay.mats() for lay in w.layers]
    O.run_blocked(w.kind.value, layers, X, T_b)  # warm-up
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        O.run_blocked(w.kind.value, layers, X, T_b)
        times.append(time.perf_counter() - t0)
    return statistics.median(times), len(times)


def cpu_baseline(args, w, sample_steps):
    """The oracle's C port of rnnblock's fast path on this box's host cores
    (all threads, plus a 1-thread row and the CPU
    model), on a bounded prefix of the same workload."""
    O = _oracle()
    cores = os.cpu_count() or 1
    L = min(sample_steps, w.seq_len)
    X = np.ascontiguousarray(w.X[:L])
    O.set_threads(cores)
    med, n = _time_oracle(O, w, X, args.block, args.cpu_seconds)
    L1 = max(args.block, L // 8)  # the 1-thread row on a shorter prefix (same per-step work)
    O.set_threads(1)
    med1, n1 = _time_oracle(O, w, np.ascontiguousarray(w.X[:L1]), args.block, min(args.cpu_seconds, 8.0))
    O.set_threads(cores)
    return {"value": round(L / med, 1), "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{args.workload} first {L} of {w.seq_len} steps, T_b={args.block}, "
                      f"median of {n} runs, oracle/ C port of rnnblock fast kernel, "
                      f"OpenMP {cores} threads",
            "single_thread": {"value": round(L1 / med1, 1), "unit": UNIT, "cores": 1,
                              "sample": f"{args.workload} first {L1} steps, T_b={args.block}, median of {n1} runs"}}


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
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
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
    ap.add_argument("--extra-modes", default="f32_ffma,bf16,tf32",
                    help="numerics modes timed beside the headline mode (f32_ffma: fp32 on the FFMA kernels)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false",
                    help="skip the host-buffer (e2e) leg: for the ncu launch list, where the profiler serialises "
                         "the kernels the streaming host path runs side by side")
    ap.add_argument("--cpu-sample", type=int, default=512, help="time steps in the CPU sample")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--partition", choices=("replicas", "pipeline", "hidden"), default="replicas",
                    help="replicas: N independent copies of the workload (cfg1/cfg2 do not shard); "
                         "pipeline: cfg4 layer pipeline across ranks; hidden: cfg5 hidden sharding")
    ap.add_argument("--chunk", type=int, default=2048,
                    help="pipeline chunk (steps, a multiple of --block); 2048 balances the per-chunk launch cost "
                         "against the (G-1)/n bubble: profiles/pipeline_chunks_r2.json")
    ap.add_argument("--no-dropin", dest="dropin", action="store_false",
                    help="skip timing the reference-signature run_blocked call")
    ap.add_argument("--no-partitioned", dest="partitioned", action="store_false",
                    help="skip the cfg4 pipeline / cfg5 hidden-sharding sub-object")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the other BASELINE configs (single-GPU lines)")
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
