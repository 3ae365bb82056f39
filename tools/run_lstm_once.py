"""One LSTM forward (d=1024, L=2048) with no timing: the command ncu captures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402

d = int(os.environ.get("LSTM_D", "1024"))
L = int(os.environ.get("LSTM_L", "2048"))
rng = np.random.default_rng(d)
s = 1.0 / np.sqrt(d)
mats = [rng.uniform(-s, s, (d, d)).astype(np.float32) for _ in range(8)] + [np.zeros(d, np.float32)] * 4
X = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).cuda()
dev = P.DeviceLstm(mats)
H = dev.forward(X, 32)
torch.cuda.synchronize()
print("ok", float(H.abs().sum()))
