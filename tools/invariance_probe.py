"""Where do fp32 scores of a program differ between a 1-program-per-CTA
launch (n <= #SMs) and a multi-program-tile launch?  Compares the last-layer
LSTM outputs (tt_tuner_lstm_outputs_f32) and the scores."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import random_seqs  # noqa: E402

from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms  # noqa: E402

rng = np.random.default_rng(12)
seqs = random_seqs(rng, rng.integers(1, 13, size=9))
m = RecurrentAttentionTuner(epochs=0, seed=5).fit(seqs, rng.uniform(0.2, 0.8, size=9))
m.precision = "fp32"
dims = m._dims()
flat = m._dev_params(dims)


def lstm_out(ss):
    prog = DevicePrograms.from_sequences(ss, "fp32", 6, 35)
    out = m._frozen_outputs(dims, flat, prog)
    return out.cpu().numpy().reshape(-1, 64), m._predict_programs(prog, dims, flat).cpu().numpy()


s1, y1 = lstm_out(seqs)
sb, yb = lstm_out(seqs * 40)
rows = s1.shape[0]
print("S equal:", np.array_equal(s1, sb[:rows]), "max|d|", np.abs(s1 - sb[:rows]).max())
print("y equal:", np.array_equal(y1, yb[:9]), np.abs(y1 - yb[:9]))
