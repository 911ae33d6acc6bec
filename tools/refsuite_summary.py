"""Table of the reference's own suite run on the GPU through install()
(tests/test_gpu_reference_suite.py with TT_REFSUITE_LOGDIR): per module and
precision the pytest result line and the C-ABI call counts.

    python tools/refsuite_summary.py gpurun_out/<tag>_refsuite <tag> > profiles/<tag>_reference_suite.txt
"""
import glob
import json
import os
import re
import sys


def main():
    d, tag = sys.argv[1], sys.argv[2]
    print("# The reference's own tests (baseline/_ref/tests, unmodified) on the B200 through install()")
    print(f"# tests/test_gpu_reference_suite.py, round 2 bundle {tag}; C-ABI calls = _lib.CALLS of the subprocess")
    print()
    print(f"{'module_precision':70s} {'result':42s} {'C-ABI calls':>12s}  per entry point")
    for log in sorted(glob.glob(os.path.join(d, "*.log"))):
        name = os.path.basename(log)[:-4]
        lines = [ln.strip() for ln in open(log, errors="replace") if re.search(r"\d+ (passed|failed|error)", ln)]
        res = re.sub(r"^=+\s*|\s*=+$", "", lines[-1]) if lines else "(no result line)"
        cj = os.path.join(d, name + ".calls.json")
        calls = json.load(open(cj)) if os.path.exists(cj) else {}
        print(f"{name[:70]:70s} {res[:42]:42s} {sum(calls.values()):12d}  {json.dumps(dict(sorted(calls.items())))}")


if __name__ == "__main__":
    main()
