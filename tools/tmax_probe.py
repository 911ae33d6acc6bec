import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from conftest import random_seqs
from paper_2304_05430_b200 import RecurrentAttentionTuner, _lib
for T in (10, 12, 13, 14, 15, 16, 20, 24, 32):
    rng = np.random.default_rng(T)
    lens = rng.integers(1, T + 1, size=32); lens[0] = T
    seqs = random_seqs(rng, lens); y = rng.uniform(0.1, 0.9, size=32)
    m = RecurrentAttentionTuner(epochs=0, seed=1, loss="ranking"); m.precision = "fp32"; m.fit(seqs, y)
    _lib.call("tt_tuner_train_set_path", 2)
    try:
        m.loss_and_gradients(seqs[:16], y[:16]); print(T, "fast ok")
    except Exception as e:
        print(T, "fast NOT eligible:", str(e)[:80])
    _lib.call("tt_tuner_train_set_path", 0)
