"""pytest plugin: run the reference's own test suite against the drop-in.

Loaded with ``-p levsketch_alias`` by tests/test_reference_suite.py.  It
makes ``import levsketch`` (and its submodules) resolve to
``paper_1812_07903_b200`` — the switch a user of the reference makes — so the
reference's tests (staged by ``__graft_entry__.build()`` from
/root/reference/pkg/tests into baseline/_ref/tests, git-ignored) exercise the
CUDA product path unchanged.  ``levsketch.cli`` is out of scope for this
build: a stub whose ``main`` skips the calling test.
"""

from __future__ import annotations

import importlib
import sys
import types

import pytest

import paper_1812_07903_b200 as P

sys.modules["levsketch"] = P
for _name in ("errors", "sketch", "leverage", "svd", "order", "dist", "matrix", "config"):
    sys.modules[f"levsketch.{_name}"] = importlib.import_module(f"paper_1812_07903_b200.{_name}")

_cli = types.ModuleType("levsketch.cli")


def _cli_main(*_a, **_k):
    pytest.skip("levsketch.cli is out of scope for the B200 build (SURVEY.md §2.1)")


_cli.main = _cli_main
sys.modules["levsketch.cli"] = _cli
P.cli = _cli
