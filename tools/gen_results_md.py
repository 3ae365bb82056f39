"""Regenerate DESIGN.md section 5 and the README results block from
profiles/bench_r2.json (the bench line this round's numbers are quoted from)."""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(REPO, "profiles", "bench_r2.json")))
sw, m, cfgs, cpu, pp = d["sweep"], d["modes"], d["configs"], d["cpu_baseline"], d["partitioned"]
TS = ("1", "2", "4", "8", "16", "32", "64")


def row(res):
    return " | ".join(f"{res[t]['steps_per_s'] / 1e6:.3g} ({res[t]['frac']:.2f})" for t in TS)


def cfgrow(k):
    return ", ".join(f"{t} → {r['steps_per_s'] / 1e6:.3g} ({r['frac']:.2f}, {r['kernel'].split(' ')[0]})"
                     for t, r in cfgs[k]["blocks"].items())


sec5 = f'''## 5. Measurement (round 2, one B200; `profiles/bench_r2.json`)

Default bench = BASELINE configs[1] (cfg2: QRNN w=2, D=H=1024, L=2048,
fp32), headline T_b = 32; L2 flushed (256 MB write) before every timed step;
CUDA events on the launching stream; NVML clocks sampled during the timed
region ({d['clocks']['sm_mhz']} MHz, throttle reasons {d['clocks']['reasons'] or 'none'}).  Fractions are of the bound that
applies (§4.0): tcgen05 weight stream for the tensor-core kernels,
max(shared-memory weight stream, FMA pipe) for the FFMA kernels.

| cfg2, M steps/s (frac of the applicable bound) | T_b=1 | 2 | 4 | 8 | 16 | 32 | 64 |
|---|---|---|---|---|---|---|---|
| **fp32** (FFMA below 8, 3xTF32 tcgen05 from 8) | {row(sw)} |
| fp32 on the FFMA kernels only (`f32_ffma`) | {row(m['f32_ffma'])} |
| bf16 (tcgen05) | {row(m['bf16'])} |
| tf32 (tcgen05; FFMA at T_b=1) | {row(m['tf32'])} |
| reference arm (oracle port, {cpu['cores']} host threads / 1 thread) | | | | | | {cpu['value'] / 1e6:.4f} / {cpu['single_thread']['value'] / 1e6:.4f} | |

* **Headline** fp32 T_b = 32: **{d['value'] / 1e6:.2f} M steps/s** ({d['roofline']['achieved']:.0f} TFLOP/s
  algorithmic; {d['roofline']['frac']:.2f} of the tcgen05 weight-stream bound — MMA issue floor
  69.4 µs per launch vs L2 feed 62.8 µs —, {d['roofline']['tensor_nominal']['frac']:.2f} of the nominal tf32 tensor
  peak in issued products; round 1: 2.96 M on the FFMA kernel); **e2e
  {d['e2e']['value'] / 1e6:.2f} M steps/s** through `rnnb_forward_host` ({d['e2e']['ms_per_step']:.3f} ms per call;
  round 1: 2.68 M); reference arm {cpu['value'] / 1e3:.1f} k steps/s on {cpu['cores']} host
  threads ("{cpu.get('cpu_model', '')}"), {cpu['single_thread']['value'] / 1e3:.1f} k on one; the
  reference-signature drop-in `run_blocked` (weights re-uploaded and repacked
  on the GPU per call): {d['dropin']['ms_per_call']:.1f} ms per call = {d['dropin']['value'] / 1e3:.0f} k steps/s (83 ms before
  the GPU repack).
* Box to box (same final binary, five bench runs this round): device 9.47-9.66 M
  steps/s, e2e 5.2-5.5 M on four boxes and 2.5-3.8 M on the slow-host box of
  §4.5.
* ncu launch list of the bench command (`profiles/ncu_launches_r2.csv`,
  summary beside it): the 3xTF32 `tc_layer_kernel` 88 % of GPU time (219 µs
  per cold launch), the L2 flush fill 6 %, the one-time weight repack 4 %,
  the operand conversion 2 %.  Full captures:
  `profiles/r2_tc_f32x3_cfg2_T32_summary.txt` (tensor pipe 36 % active — the
  51-cycle floor at N = 32/64 allows ~47 % —, 254 registers, no spills, DRAM
  91 MB against 75.5 MB algorithmic: weights hi+lo, x hi+lo once, h once),
  and the bf16 T_b = 64 kernel; per-T_b counters `profiles/ncu_sweep_r2.json`.
* Other BASELINE configs (bench `configs`, one GPU, L2 flushed; T_b → M steps/s
  (frac, kernel)):

  | config | mode: T_b → M steps/s (frac, kernel) |
  |---|---|
  | cfg1 SRU 512, L 256 | f32: {cfgrow('cfg1/f32')} — a 256-step sequence is launch/latency bound |
  | cfg3 proj + 6 SRU + logits, L 4096 | f32: {cfgrow('cfg3/f32')}; bf16: {cfgrow('cfg3/bf16')}; tf32: {cfgrow('cfg3/tf32')} |
  | cfg4 8 × QRNN 2048, L 65536 | f32 (3xTF32): {cfgrow('cfg4/f32')}; bf16: {cfgrow('cfg4/bf16')} (power-capped, §4.0) |
  | cfg5 bidir SRU 4096, L 8192 (fused sharded stack, G = 1) | bf16: {cfgrow('cfg5/bf16')} (power-capped) |

* Partitioned (bench `partitioned`, strong scaling, every N): cfg4 bf16 layer
  pipeline and cfg5 bf16 hidden sharding; at N = 1 (the anchors):
  {pp['pipeline']['value'] / 1e6:.2f} M (2048-step chunks; {pp['pipeline']['roofline']['applicable']['frac']:.2f} of the applicable weight-stream bound, {pp['pipeline']['roofline']['frac']:.2f} of
  the nominal tensor peak) and {pp['hidden']['value'] / 1e6:.3f} M steps/s ({pp['hidden']['roofline']['applicable']['frac']:.2f} / {pp['hidden']['roofline']['frac']:.2f}).

'''
p = os.path.join(REPO, "DESIGN.md")
s = open(p).read()
a, b = s.index("## 5. Measurement (round 2"), s.index("### 5.1 Switches")
open(p, "w").write(s[:a] + sec5 + s[b:])

c3 = cfgs
readme = f'''## Results (round 2, one B200; details and evidence in DESIGN.md §4-5 and `profiles/`)

* Headline (BASELINE cfg2: QRNN 1024, L = 2048, fp32, T_b = 32): **{d['value'] / 1e6:.2f} M
  steps/s** on the device (fp32-accurate 3xTF32 on tcgen05: {d['roofline']['achieved']:.0f} TFLOP/s, {d['roofline']['frac']:.2f}
  of the measured tcgen05 weight-stream bound; round 1: 2.96 M), **{d['e2e']['value'] / 1e6:.2f} M
  steps/s end to end** from pinned host buffers ({d['e2e']['ms_per_step']:.2f} ms per call: copy engines
  in, a persistent conversion kernel, h stored straight into pinned memory;
  round 1: 2.68 M); the reference algorithm on the box's {cpu['cores']} host threads:
  {cpu['value'] / 1e3:.0f} k steps/s ({cpu['single_thread']['value'] / 1e3:.1f} k on one).
* T_b sweep (fp32): {sw['1']['steps_per_s'] / 1e6:.2f} / {sw['2']['steps_per_s'] / 1e6:.2f} / {sw['4']['steps_per_s'] / 1e6:.2f} M steps/s at T_b = 1 / 2 / 4 on the
  FFMA kernels ({sw['1']['frac']:.2f} / {sw['2']['frac']:.2f} / {sw['4']['frac']:.2f} of max(shared-memory weight stream, FMA
  pipe)), {sw['8']['steps_per_s'] / 1e6:.2f} / {sw['16']['steps_per_s'] / 1e6:.2f} / {sw['32']['steps_per_s'] / 1e6:.2f} / {sw['64']['steps_per_s'] / 1e6:.2f} M at 8 / 16 / 32 / 64 on tcgen05; bf16
  {m['bf16']['1']['steps_per_s'] / 1e6:.1f} → {m['bf16']['64']['steps_per_s'] / 1e6:.1f} M, tf32 {m['tf32']['1']['steps_per_s'] / 1e6:.2f} → {m['tf32']['64']['steps_per_s'] / 1e6:.1f} M steps/s.
* Every BASELINE config measured on one GPU (cfg1–cfg5) and parity-tested at
  its real shape against the CPU oracle (`tests/test_gpu_full_shapes.py`:
  cfg4's 8 × 2048 stack over all 65536 steps, cfg5's 4096-wide
  bidirectional layers, cfg3's projection + logits on own kernels — fp32
  dense layers on the 3xTF32 path too); cfg3 (acoustic model, L = 4096) at
  T_b = 32: {c3['cfg3/f32']['blocks']['32']['steps_per_s'] / 1e6:.2f} M steps/s in fp32, {c3['cfg3/bf16']['blocks']['32']['steps_per_s'] / 1e6:.2f} M in bf16.
* Measured hardware limits the design leans on: the tcgen05 issue floor
  (`tools/mma_rate.cu`: 51 cycles per 128×N×K-step MMA for N ≤ 64), the
  per-SM L2 → shared-memory fill rate and the fact that cluster multicast
  does not raise it (`tools/l2_mc_peak.cu`), the 1000 W power cap the long
  bf16 launches run into (`tools/clock_probe.py`: cfg4 at 1770 / 1537 MHz for
  T_b = 32 / 64), PCIe duplex behaviour of copy engines vs SM loads/stores of
  pinned memory (`tools/zc_probe.cu`).
* Look-back carry "where the value is the flag": one 8-byte store publishes a
  block's carry map, consumers poll the values themselves (no status words,
  barriers or fences): cfg2 bf16 T_b = 16 110 → 85 µs; with it, two epilogue
  warp groups on alternate items where the epilogue bounds an item: cfg3 bf16
  T_b = 32 0.62 → 0.38 ms.
* The reference-signature `run_blocked` (weights re-uploaded per call, repacked
  by a GPU kernel): {d['dropin']['ms_per_call']:.1f} ms per cfg2 call = {d['dropin']['value'] / 1e3:.0f} k steps/s (83 ms before).
* LSTM partial precompute: 568k / 191k / 175k steps/s at d = 350 / 700 /
  1024.
* Tests: 369 GPU (`-m gpu`), 175 CPU.
'''
p = os.path.join(REPO, "README.md")
r = open(p).read()
open(p, "w").write(r[:r.index("## Results (round 2")] + readme)
print("DESIGN.md section 5 and README results regenerated from profiles/bench_r2.json")
