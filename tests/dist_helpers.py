"""Worker functions for the world_size-2 gloo tests of partition.py (CPU,
oracle compute).  Spawned processes import this module by name."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


class OracleStage:
    """Layer range on the CPU oracle with (c, x_carry) carried across chunks."""

    def __init__(self, kind, layers, block_size):
        import oracle as O
        self.O, self.kind, self.layers, self.T = O, kind, layers, block_size
        self.d_in = layers[0][0].shape[1]
        self.c = [np.zeros(l[0].shape[0], np.float32) for l in layers]
        self.xc = [np.zeros(l[0].shape[1], np.float32) for l in layers]

    def __call__(self, x):
        y = x.numpy()
        for i, lay in enumerate(self.layers):
            y, self.c[i], self.xc[i] = self.O.layer_blocked(self.kind, lay, np.ascontiguousarray(y), self.T,
                                                          c=self.c[i], xc=self.xc[i])
        return torch.from_numpy(np.ascontiguousarray(y))


def pipeline_worker(rank, world, port, result_path):
    from paper_1803_11389_b200 import partition
    import oracle as O
    init(rank, world, port)
    layers = O.generate_layers("qrnn", 32, 32, 4, 5, np.float32)
    X = torch.from_numpy(np.random.default_rng(1).standard_normal((256, 32)).astype(np.float32))
    lo, hi = partition.layer_ranges(4, world)[rank]
    stage = OracleStage("qrnn", layers[lo:hi], 16)
    out = partition.pipeline_forward(stage, X if rank == 0 else None, 256, 32, 64, 16, rank, world,
                                     torch.float32, torch.device("cpu"))
    if rank == world - 1:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def sru_wide_numpy(mats, x, hw_off):
    """Reference wide SRU layer (f64 loop): highway reads x[:, hw_off + unit]."""
    W, Wf, Wr, bf, br = [np.asarray(m, np.float64) for m in mats]
    x = np.asarray(x, np.float64)
    sig = lambda z: 0.5 * (1.0 + np.tanh(0.5 * z))
    c = np.zeros(W.shape[0])
    H = np.empty((x.shape[0], W.shape[0]))
    xh = x[:, hw_off:hw_off + W.shape[0]]
    for t in range(x.shape[0]):
        f = sig(Wf @ x[t] + bf)
        r = sig(Wr @ x[t] + br)
        c = f * c + (1.0 - f) * (W @ x[t])
        H[t] = r * np.tanh(c) + (1.0 - r) * xh[t]
    return H


def bidir_reference(layers_f, layers_b, X):
    x = np.asarray(X, np.float64)
    Hd = layers_f[0].mats()[0].shape[0]
    for lf, lb in zip(layers_f, layers_b):
        d_in = lf.mats()[0].shape[1]
        yf = sru_wide_numpy(lf.mats(), x, 0 if d_in == Hd else 0)
        yb = sru_wide_numpy(lb.mats(), x[::-1], 0 if d_in == Hd else Hd)[::-1]
        x = np.concatenate([yf, yb], axis=1)
    return x


def make_bidir(H=16, d0=16, n_layers=2, seed=3):
    from paper_1803_11389_b200.workloads import WideSruWeights
    rng = np.random.default_rng(seed)

    def lay(d_in):
        u = lambda: rng.uniform(-0.3, 0.3, (H, d_in))
        return WideSruWeights(u(), u(), u(), rng.uniform(-0.1, 0.1, H), rng.uniform(-0.1, 0.1, H))
    fw, bw = [], []
    for li in range(n_layers):
        d_in = d0 if li == 0 else 2 * H
        fw.append(lay(d_in))
        bw.append(lay(d_in))
    X = rng.standard_normal((40, d0))
    return fw, bw, X


def sharding_worker(rank, world, port, result_path):
    from paper_1803_11389_b200 import partition
    init(rank, world, port)
    fw, bw, X = make_bidir()

    def make_stage(mats, hw_off):
        return lambda x: torch.from_numpy(sru_wide_numpy(mats, x.numpy(), hw_off))
    model = partition.ShardedBidirSRU(fw, bw, rank, world, make_stage)
    out = model.forward(torch.from_numpy(X))
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()
