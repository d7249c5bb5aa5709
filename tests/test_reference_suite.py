"""The reference's own test suite (/root/reference/pkg/tests, 144 tests)
run unchanged against the drop-in: ``import levsketch`` resolves to
``paper_1812_07903_b200`` (tests/refsuite/levsketch_alias.py), so every
reference test of the sketch / SVD / leverage / distributed / ordering /
matrix modules and the acceptance criteria exercises the CUDA product path.

The reference is not on the GPU box: ``__graft_entry__.build()`` stages its
tests (with the reference install itself) under baseline/_ref/, which is
git-ignored but travels with the repo snapshot.  Expected deviations, each a
deliberate scope decision, are deselected and listed here:
  * test_sketch.py::test_spec_validation — asserts SketchSpec("gaussian")
    raises; the Gaussian family is a deliberate extension (BASELINE configs
    1 and 5);
  * test_cli.py (all) and the CLI-driven acceptance criteria 9 and 10 —
    the CLI is out of scope; their calls skip.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = ROOT / "baseline" / "_ref" / "tests"
DESELECT = ["test_sketch.py::test_spec_validation"]
IGNORE = ["test_cli.py"]

pytestmark = pytest.mark.gpu


def test_reference_suite_on_dropin():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not REF_TESTS.is_dir():
        pytest.skip("reference tests not staged (build() stages them from /root/reference)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refsuite"), str(ROOT), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", str(REF_TESTS), "-p", "levsketch_alias", "-p", "no:cacheprovider",
           "-q", "-rfEs", "--rootdir", str(REF_TESTS), "-c", os.devnull]
    for d in DESELECT:
        cmd += ["--deselect", d]  # node ids relative to the rootdir
    for i in IGNORE:
        cmd += ["--ignore", str(REF_TESTS / i)]
    p = subprocess.run(cmd, cwd=str(REF_TESTS), env=env, capture_output=True, text=True, timeout=1800)
    log = p.stdout + p.stderr
    out = ROOT / "gpurun_out"
    if out.is_dir():
        (out / "refsuite.log").write_text(log)
    print(log[-4000:])
    m = re.search(r"(\d+) passed", log)
    passed = int(m.group(1)) if m else 0
    assert p.returncode == 0, log[-6000:]
    assert passed >= 100, f"only {passed} reference tests passed"
