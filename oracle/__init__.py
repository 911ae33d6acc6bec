"""CPU oracle for the tensortune hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in float64 numpy, the reference algorithms that the
B200 kernels replace (paths relative to /root/reference/pkg/src/tensortune):

* ``tuner``   -- estimators/tuner.py (biLSTM + iterative attention + head,
                 hand-written backprop, the minibatch Adam training loop)
* ``mlp``     -- estimators/mlp.py (CostMLP forward/backward/fit)
* ``losses``  -- estimators/mlp.py:25-35 ranking_grad, tuner.py:372-375 MSE
* ``adam``    -- estimators/optim.py:8-46
* ``metrics`` -- metrics.py:46-94 (PCA, top-k, rmse, ranking_loss) and the
                 grouped PCA of tuner.py:486-496
* ``sampling``-- sampling.py:37-85 + data.py:440-446 (quantile cut,
                 survivor counts, raw task weights) and numpy's linear
                 quantile (numpy/lib/_function_base_impl.py, numpy 2.3.5)

Pinning: every function here is checked against golden vectors produced by
running the reference itself (tests/golden/make_golden.py, committed with
its outputs) -- see tests/test_oracle_golden.py.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import this package, and
only as the checker or as the timed CPU reference.  The product path
(``paper_2304_05430_b200``) never imports it.
"""
