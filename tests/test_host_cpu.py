"""CPU-only checks: the C-ABI library loads and exports every declared entry
point, and the host-side logic of the drop-in API (validation, sizing,
partitioning, I/O, error classes) matches the reference contract."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native, errors
from oracle import levsketch_oracle as O

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = "\n".join(p.read_text() for p in (ROOT / "include").glob("*.h"))
    return sorted(set(re.findall(r"LVSK_API\s+[\w\s\*]+?\b(lvsk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()  # raises loudly if the .so was not built
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())
    assert lib.lvsk_abi_version() == 1


def test_inflight_hint_roundtrip():
    """lvsk_set_inflight (BatchRunner's scheduling hint) is host state only:
    round trip, range check with an error message, default restored."""
    lib = _native.lib()
    assert lib.lvsk_get_inflight() == 1
    try:
        assert lib.lvsk_set_inflight(2) == 0
        assert lib.lvsk_get_inflight() == 2
        assert lib.lvsk_set_inflight(0) == 1  # LVSK_ERR_CONFIGURATION
        assert b"passes" in lib.lvsk_last_error()
        assert lib.lvsk_get_inflight() == 2
    finally:
        assert lib.lvsk_set_inflight(1) == 0


def test_gaussian_generator_table_matches_oracle():
    """The K4 generator's host-built table (csrc/gaussian.cu) is the oracle's,
    bit for bit, so device entries can equal the oracle's exactly."""
    import ctypes

    out = np.zeros(O.gaussian_tables().size, dtype=np.uint16)
    rc = _native.lib().lvsk_gaussian_tables(out.ctypes.data_as(ctypes.c_void_p), out.size)
    assert rc == 0
    assert np.array_equal(out, O.gaussian_tables())
    # too small a buffer is refused, not overrun
    assert _native.lib().lvsk_gaussian_tables(out.ctypes.data_as(ctypes.c_void_p), out.size - 1) != 0


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        P.apply_sketch(np.ones((4, 2)), P.SketchSpec("countsketch", eps=0.5, d=2))


def test_spec_validation_and_gaussian_extension():
    with pytest.raises(errors.UnsupportedFamilyError):
        P.SketchSpec("bogus", eps=0.5, d=4)
    with pytest.raises(errors.ConfigurationError):
        P.SketchSpec("countsketch", eps=1.5, d=4)
    with pytest.raises(errors.ConfigurationError):
        P.SketchSpec("countsketch", eps=0.5, d=0)
    with pytest.raises(errors.ConfigurationError):
        P.SketchSpec("osnap", eps=0.5, d=4, osnap_s=0)
    with pytest.raises(errors.ConfigurationError):
        P.SketchSpec("countsketch", eps=0.5, d=4, seed=-1)
    # deliberate extension: the reference rejects "gaussian" (sketch.py:74-75)
    assert P.SketchSpec("gaussian", eps=0.5, d=4).family == "gaussian"


@pytest.mark.parametrize(
    "fam,kw,expect",
    [
        ("countsketch", dict(sizing_c=1.0), 1024),
        ("osnap", dict(sizing_c=1.0), 178),
        ("srht", dict(sizing_c=1.0), 256),
        ("countsketch", dict(rows_override=64), 64),
        ("osnap", dict(rows_override=64), 64),
        ("srht", dict(rows_override=64), 64),
        ("countsketch", dict(sizing_c=2.0), 2048),
    ],
)
def test_sketch_rows(fam, kw, expect):
    spec = P.SketchSpec(fam, eps=0.5, d=16, **kw)
    assert P.sketch_rows(spec) == expect
    assert P.sketch_rows(spec) == O.sketch_rows(fam, 0.5, 16, None, kw.get("rows_override"), kw.get("sizing_c"))


def test_osnap_default_s():
    assert P.SketchSpec("osnap", eps=0.5, d=16).s == 4
    assert P.SketchSpec("osnap", eps=0.5, d=1000).s == 10
    assert P.SketchSpec("countsketch", eps=0.5, d=1000).s == 1


def test_hash_keys_match_oracle():
    from paper_1812_07903_b200.sketch import _HASH_STREAM, _splitmix

    for fam in ("countsketch", "osnap"):
        for seed in (0, 1, 12345, 2**40):
            assert _splitmix(seed, _HASH_STREAM[fam], 9) == O.splitmix_keys(seed, O.HASH_TAG[fam], 9)


def test_srht_host_draw_matches_oracle(golden):
    from paper_1812_07903_b200.sketch import srht_signs_and_sample

    signs, sample = srht_signs_and_sample(0, 2**21, 4096)
    assert np.array_equal(sample, golden["srht_c3_sample"])
    assert np.array_equal(signs[:4096], golden["srht_c3_signs_head"])


def test_partition_rows():
    assert P.partition_rows(10, 2) == [(0, 5), (5, 10)]
    assert P.partition_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert P.partition_rows(5, 5) == [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)]
    with pytest.raises(errors.ConfigurationError):
        P.partition_rows(3, 4)
    with pytest.raises(errors.ConfigurationError):
        P.partition_rows(3, 0)


def test_truncate_host_logic():
    svd = P.SvdResult(u=np.eye(3), sigma=np.array([10.0, 5.0, 1e-3]), vt=np.eye(3))
    kept = P.truncate(svd, 0.01)
    assert kept.rank == 2 and np.array_equal(kept.sigma, [10.0, 5.0])
    assert P.truncate(kept, 0.01).rank == 2
    assert P.truncate(P.SvdResult(np.eye(3), np.array([2.0, 1.0, 0.0]), np.eye(3)), 0.0).rank == 2
    with pytest.raises(errors.ConfigurationError):
        P.truncate(svd, 1.0)
    with pytest.raises(errors.DegenerateInputError):
        P.truncate(P.SvdResult(np.eye(2), np.zeros(2), np.eye(2)), 0.1)


def test_approx_basis_refuses_exact_zero():
    from paper_1812_07903_b200.leverage import _approx_basis

    with pytest.raises(errors.SingularInversionError):
        _approx_basis(P.SvdResult(u=np.eye(3), sigma=np.array([2.0, 1.0, 0.0]), vt=np.eye(3)))
    b = _approx_basis(P.SvdResult(u=np.eye(2), sigma=np.array([2.0, 4.0]), vt=np.eye(2)))
    assert np.array_equal(b, np.diag([0.5, 0.25]))


def test_policy_validation_and_batches():
    with pytest.raises(errors.ConfigurationError):
        P.OrderingPolicy("sorted")
    with pytest.raises(errors.ConfigurationError):
        P.OrderingPolicy("dec", seed=-1)
    plan = P.OrderingPlan(epoch=0, indices=np.array([3, 1, 4, 0, 2]), policy=P.OrderingPolicy("dec"))
    batches = P.emit_batches(plan, 2)
    assert [len(b) for b in batches] == [2, 2, 1]
    assert np.array_equal(np.concatenate(batches), plan.indices)
    with pytest.raises(errors.ConfigurationError):
        P.emit_batches(plan, 0)


def test_mem_cap(monkeypatch):
    from paper_1812_07903_b200.config import ensure_capacity, mem_cap

    assert mem_cap() == 4 * 2**30
    monkeypatch.setenv("LVSK_MEM_CAP", "1000")
    assert mem_cap() == 1000
    with pytest.raises(errors.CapacityError):
        ensure_capacity(1001, "x")
    monkeypatch.setenv("LVSK_MEM_CAP", "abc")
    with pytest.raises(errors.ConfigurationError):
        mem_cap()


def test_matrix_io_roundtrip(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 3))
    P.save_matrix(a, tmp_path / "a.bin")
    assert np.array_equal(P.load_matrix(tmp_path / "a.bin"), a)
    P.save_matrix(a, tmp_path / "a.csv", "csv")
    assert np.array_equal(P.load_matrix(tmp_path / "a.csv"), a)
    (tmp_path / "bad.csv").write_text("1,2\n3\n")
    with pytest.raises(errors.FormatError):
        P.load_matrix(tmp_path / "bad.csv")
    (tmp_path / "nan.csv").write_text("1,x\n")
    with pytest.raises(errors.ParseError):
        P.load_matrix(tmp_path / "nan.csv")
    with pytest.raises(errors.FormatError):
        P.as_matrix(np.array([[1.0, np.nan]]))
    with pytest.raises(errors.FormatError):
        P.as_matrix(np.zeros((0, 3)))


def test_gen_synthetic_matches_reference_stream(golden):
    # lev0 in the golden set is gen_synthetic(n=4096, d=10, rank=10, seed=7)
    a = P.gen_synthetic(P.SyntheticSpec(n=4096, d=10, rank=10, seed=7))
    np.testing.assert_allclose(a, golden["lev0_x"], rtol=1e-12, atol=1e-12)


def test_error_hierarchy():
    for name in ("FormatError", "ParseError", "CapacityError", "DimensionMismatchError", "IncompatibleSketchError",
                 "DegenerateInputError", "SingularInversionError", "UnsupportedFamilyError", "ConfigurationError"):
        assert issubclass(getattr(errors, name), errors.LevsketchError)
    assert issubclass(errors.ParseError, errors.FormatError)


def test_open_lvsk_validates_header(tmp_path):
    import paper_1812_07903_b200 as P
    from paper_1812_07903_b200 import errors

    x = np.arange(12.0).reshape(4, 3)
    good = tmp_path / "g.lvsk"
    P.save_matrix(x, good)
    m = P.open_lvsk(good)
    assert m.shape == (4, 3) and np.array_equal(np.asarray(m), x)
    bad = tmp_path / "b.lvsk"
    bad.write_bytes(b"XXXX" + good.read_bytes()[4:])
    with pytest.raises(errors.FormatError):
        P.open_lvsk(bad)
    short = tmp_path / "s.lvsk"
    short.write_bytes(good.read_bytes()[:-8])
    with pytest.raises(errors.FormatError):
        P.open_lvsk(short)
