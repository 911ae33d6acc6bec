"""CPU-side checks of the drop-in boundary: the C-ABI library builds for
sm_100a, loads without a GPU, and exports every symbol include/tt_b200.h
declares (no compute calls here)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tt_b200.h")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_exports_every_declared_symbol():
    from paper_2304_05430_b200 import _lib
    from paper_2304_05430_b200.build import build

    path = build()
    lib = ctypes.CDLL(path)
    missing = [s for s in declared_symbols() if getattr(lib, s, None) is None]
    assert not missing, missing
    # the ctypes table covers exactly the header
    assert sorted(_lib.SIGNATURES) == declared_symbols()
    assert _lib.load().tt_abi_version() == 1


def test_library_is_sm100a_code():
    from paper_2304_05430_b200.build import LIB, build

    build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_param_count_matches_reference_layout():
    from paper_2304_05430_b200 import _lib

    lib = _lib.load()
    # 82,625 parameters for the default tuner
    assert lib.tt_tuner_param_count(3, 32, 6, 35) == 82625
    assert lib.tt_mlp_param_count(164) == 14785
    assert lib.tt_mlp_param_count(47) == 7297


def test_f32tc_eligibility_is_a_shape_rule():
    """The fp32 tensor-core scorer's eligibility depends on the model's shapes
    only (never on the batch), so a program's score cannot depend on which
    batch it is scored in; the workspace shrinks for small calls."""
    from paper_2304_05430_b200 import _lib

    lib = _lib.load()
    ok = lib.tt_tuner_f32tc_eligible
    assert ok(3, 32, 2, 6, 10) == 1
    assert ok(1, 32, 1, 32, 4096) == 1 and ok(8, 32, 4, 1, 1) == 1
    assert ok(3, 16, 2, 6, 10) == 0      # hidden != 32: the CUDA-core kernel
    assert ok(3, 32, 8, 6, 10) == 0      # heads 1, 2 or 4
    assert ok(3, 32, 2, 33, 10) == 0     # step width <= 32
    assert ok(3, 32, 2, 6, 4097) == 0    # max steps <= 4096
    ws = lib.tt_tuner_predict_f32tc_workspace_bytes
    small, big = ws(3, 32, 10, 1), ws(3, 32, 10, 10_000_000)
    assert 0 < small < big and small < 32 * 1024 * 1024
    assert ws(3, 32, 10, 10_000_000) == ws(3, 32, 10, 20_000_000)  # launches are chunked
