"""pytest plugin: run the reference's OWN test suite on the B200 kernels.

    PYTHONPATH=<repo>:<repo>/tests python -m pytest -p refsuite_plugin \\
        baseline/_ref/tests/test_tuner.py ...

Loaded before collection, it puts the staged, unmodified reference
(``baseline/_ref/tensortune``, see tools/stage_reference.py) on sys.path,
imports it and calls ``paper_2304_05430_b200.install.install()``, so every
``from tensortune.estimators import RecurrentAttentionTuner`` /
``from tensortune.metrics import pairwise_comparison_accuracy`` in the
reference's tests binds to the GPU classes and kernels.  At session end it
writes the per-entry-point C-ABI call counts (``_lib.CALLS``) to
$TT_REFSUITE_CALLS, the evidence that the suite really ran on the kernels.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    import tensortune  # noqa: F401
    import tensortune.estimators.mlp  # noqa: F401
    import tensortune.estimators.tuner  # noqa: F401
    import tensortune.features  # noqa: F401
    import tensortune.metrics  # noqa: F401
    import tensortune.models  # noqa: F401
    import tensortune.sampling  # noqa: F401
    import tensortune.search  # noqa: F401
    import tensortune.transfer  # noqa: F401

    assert os.path.dirname(tensortune.__file__).startswith(REF), tensortune.__file__
    from paper_2304_05430_b200 import install

    install.install()
    import paper_2304_05430_b200 as pkg

    assert tensortune.estimators.RecurrentAttentionTuner is pkg.RecurrentAttentionTuner
    assert tensortune.estimators.tuner.RecurrentAttentionTuner is pkg.RecurrentAttentionTuner
    assert tensortune.metrics.pairwise_comparison_accuracy is pkg.pairwise_comparison_accuracy


def pytest_report_header(config):
    from paper_2304_05430_b200 import config as gcfg

    return [f"refsuite: tensortune from {REF}, installed on the B200 kernels, "
            f"precision={gcfg.PRECISION}"]


def pytest_sessionfinish(session, exitstatus):
    from paper_2304_05430_b200 import _lib

    out = os.environ.get("TT_REFSUITE_CALLS")
    if out:
        with open(out, "w") as fh:
            json.dump(dict(sorted(_lib.CALLS.items())), fh, indent=1)
