"""Stage the unmodified reference under baseline/_ref/ (git-ignored, travels
to the GPU box with the gpurun snapshot).

    python tools/stage_reference.py

* ``baseline/_ref/tensortune``  -- ``pip install --no-index --no-deps
  --target baseline/_ref`` of /root/reference/pkg (built from a /tmp copy,
  the tree is read-only);
* ``baseline/_ref/tests``       -- the reference's own pytest suite
  (pkg/tests), so ``tests/test_gpu_reference_suite.py`` can run it on the
  B200 against the kernels through ``install()``;
* ``baseline/_ref/scripts``     -- pkg/scripts (the pipeline script the
  acceptance determinism test shells out to).

Nothing here is imported by the product package; the reference is the
"reference arm" of bench.py and the parity suite's oracle.  A no-op when
/root/reference is absent (the GPU box) or the stage is already current.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")
STAMP = os.path.join(DEST, ".staged")


def stage(force: bool = False) -> str | None:
    if not os.path.isdir(REF_PKG):
        return DEST if os.path.isdir(os.path.join(DEST, "tensortune")) else None
    if not force and os.path.exists(STAMP):
        return DEST
    os.makedirs(DEST, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("frontend", "__pycache__"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--upgrade", "--target", DEST, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{r.stdout}\n{r.stderr}")
    for sub in ("tests", "scripts"):
        dst = os.path.join(DEST, sub)
        if os.path.isdir(dst):
            shutil.rmtree(dst)
        shutil.copytree(os.path.join(REF_PKG, sub), dst,
                        ignore=shutil.ignore_patterns("__pycache__"))
    with open(STAMP, "w") as fh:
        fh.write("staged from /root/reference/pkg\n")
    return DEST


if __name__ == "__main__":
    print(stage(force="-f" in sys.argv))
