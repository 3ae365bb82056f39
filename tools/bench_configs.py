"""Time every BASELINE.json config on one GPU (beside bench.py's headline).

    python tools/bench_configs.py [--reps 3] [--out profiles/configs_r1.json]

Per config, mode and T_b: W=3 warm-up forwards, then `reps` forwards, each
bracketed by CUDA events with a 256 MB L2 flush before it; steps/s = L /
mean time.  cfg1-cfg4 run the blocked stack (DeviceStack; cfg3 adds the
120->1024 projection and 1024->2000 logits), cfg5 runs the bidirectional
wide SRU through the fused sharded stack p2p.P2PBidirSRU at G = 1 (all
units on this GPU).  Outputs are not re-verified here (tests/ do that).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402
from paper_1803_11389_b200.acoustic import AcousticSRU  # noqa: E402

PLAN = {
    "cfg1": [("f32", (1, 4, 16))],
    "cfg2": [("f32", (1, 2, 4, 8, 16, 32, 64)), ("bf16", (16, 32, 64)), ("tf32", (16, 32, 64)),
             ("f32x3", (16, 32))],
    "cfg3": [("f32", (1, 8, 32)), ("bf16", (1, 8, 32)), ("tf32", (8, 32))],
    "cfg4": [("bf16", (32,)), ("f32x3", (32,)), ("f32", (32,))],
    "cfg5": [("bf16", (16, 64))],
}


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sum(ts) / len(ts)


def p2p_runs(reps, flush):
    """The fused peer-memory partitions (p2p.py) on ONE GPU: G ranks emulated
    as rank objects with their own streams sharing the device, so the
    numbers show the protocol's overhead (flags, chunking, epilogue stores to
    several destinations) against the unpartitioned run -- not multi-GPU
    scaling, which needs G GPUs."""
    from paper_1803_11389_b200 import p2p
    from paper_1803_11389_b200.partition import layer_ranges
    out = []
    w = workloads.make("cfg4")
    X = torch.from_numpy(w.X).cuda()
    L = w.seq_len
    fl = workloads.flops_per_step(w)
    for mode in ("bf16",):
        whole = P.DeviceStack(w.kind, w.layers, mode=mode)
        ms = timed(lambda: whole.forward(X, 32), reps, flush)
        out.append({"config": "cfg4", "mode": mode, "T_b": 32, "path": "unpartitioned DeviceStack", "G": 1,
                    "ms": round(ms, 3), "steps_per_s": round(L / ms * 1e3, 1)})
        print(out[-1], flush=True)
        whole.close()
        for G in (2, 4):
            stages = []
            for g, (lo, hi) in enumerate(layer_ranges(len(w.layers), G)):
                st = P.DeviceStack(w.kind, w.layers[lo:hi], mode=mode)
                stages.append(p2p.P2PPipelineStage(st, g, G, 4096, 32, slots=2))
            for s_ in stages:
                s_.connect_local(stages)
            ms = timed(lambda: p2p.run_local_pipeline(stages, X, L), reps, flush)
            out.append({"config": "cfg4", "mode": mode, "T_b": 32, "G": G, "chunk": 4096, "slots": 2,
                        "path": "P2P layer pipeline, ranks emulated on one GPU", "ms": round(ms, 3),
                        "steps_per_s": round(L / ms * 1e3, 1), "tflops": round(fl * L / ms / 1e9, 2)})
            print(out[-1], flush=True)
            for s_ in stages:
                s_.stack.close()
    del X
    torch.cuda.empty_cache()
    w = workloads.make("cfg5")
    X = torch.from_numpy(w.X).cuda()
    L = w.seq_len
    for G in (1, 2):
        ranks = [p2p.P2PBidirSRU(w.layers, w.layers_bwd, g, G, 64, "bf16", L) for g in range(G)]
        for r in ranks:
            r.connect_local(ranks)
        ms = timed(lambda: p2p.run_local_bidir(ranks, X), reps, flush)
        out.append({"config": "cfg5", "mode": "bf16", "T_b": 64, "G": G,
                    "path": "P2P hidden sharding, all-gather in the epilogue, ranks emulated on one GPU",
                    "ms": round(ms, 3), "steps_per_s": round(L / ms * 1e3, 1)})
        print(out[-1], flush=True)
        del ranks
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "configs.json"))
    ap.add_argument("--p2p", action="store_true",
                    help="also time the fused peer-memory partitions with G ranks emulated on this one GPU")
    a = ap.parse_args()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    res = {}
    for name in a.configs.split(","):
        t0 = time.time()
        w = workloads.make(name)
        X = torch.from_numpy(w.X).cuda()
        L = w.seq_len
        fl = workloads.flops_per_step(w)
        res[name] = {"seq_len": L, "flops_per_step": fl, "params": workloads.param_count(w), "runs": []}
        for mode, blocks in PLAN[name]:
            if name == "cfg3":
                model = AcousticSRU(w.proj, w.layers, w.logits, mode=mode)
                run = lambda T: model.forward(X, T)
            elif name == "cfg5":
                # the fused sharded stack (p2p.py) at G = 1: all units on this GPU,
                # backward direction stored with a negative row stride (no flips)
                from paper_1803_11389_b200 import p2p
                models = {}

                def run(T, mode=mode):
                    if T not in models:
                        models.clear()
                        torch.cuda.empty_cache()
                        r = p2p.P2PBidirSRU(w.layers, w.layers_bwd, 0, 1, T, mode, L)
                        r.connect_local([r])
                        models[T] = r
                    return models[T].forward(X)
            else:
                st = P.DeviceStack(w.kind, w.layers, mode=mode)
                run = lambda T, st=st: st.forward(X, T)
            for T in blocks:
                ms = timed(lambda: run(T), a.reps, flush)
                entry = {"mode": mode, "T_b": T, "ms": round(ms, 4), "steps_per_s": round(L / ms * 1e3, 1),
                         "tflops": round(fl * L / ms / 1e9, 2)}
                res[name]["runs"].append(entry)
                print(name, entry, flush=True)
            if name == "cfg3":
                model.close()
            elif name not in ("cfg5",):
                st.close()
        res[name]["wall_s"] = round(time.time() - t0, 1)
        del X
        torch.cuda.empty_cache()
    if a.p2p:
        res["p2p_emulated"] = p2p_runs(a.reps, flush)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
