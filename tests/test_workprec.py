"""Work-precision harness (`paper_2211_08948_b200.bench`).

CPU tests pin the on-disk formats and bookkeeping (CSV header and row
formatting, `.ref` binary layout, matrix expansion, validation) as the
reference's test_bench.py:14-133 does; GPU tests run configs through the
device engines and compare every counter and the error with the CPU oracle
driving the same problem (oracle/np_integrate.adaptive).
"""

import csv
import math
import struct

import numpy as np
import pytest

from paper_2211_08948_b200 import bench as B


def test_header_pinned():
    assert B.CSV_HEADER == ("problem,param,n,integrator,scheme,tol,steps_accepted,"
                            "steps_rejected,rhs_evals,leja_iters,krylov_matvecs,substeps,"
                            "wall_time_s,l2_error")
    assert B.DEFAULT_TOLS == (1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9)


@pytest.mark.parametrize("cfg", [
    ("heat", math.nan, 16, "exprb43", "kiops", 1e-6),
    ("adr", 0.1, 16, "rk4", "kiops", 1e-6),
    ("adr", 0.1, 16, "exprb43", "chebyshev", 1e-6),
    ("adr", 0.1, 16, "exprb43", "lekry", 1e-6),   # exprb43 has no lekry
    ("adr", 0.1, 16, "exprb43", "kiops", 2.0),
    ("adr", 0.1, 16, "exprb43", "kiops", 0.0),
])
def test_validation_rejects(cfg):
    with pytest.raises(ValueError):
        B.RunConfig(*cfg).validate()


def test_validation_accepts():
    B.RunConfig("semilinear", math.nan, 16, "exprb43", "kiops", 1e-6).validate()
    B.RunConfig("adr", 0.1, 16, "epirk4s3", "lekry", 1e-6).validate()


def test_ref_file_layout_and_roundtrip(tmp_path):
    u = np.random.default_rng(3).standard_normal(41)
    p = tmp_path / "a.ref"
    B._ref_write(p, u)
    raw = p.read_bytes()
    assert len(raw) == 8 + 8 * 41
    assert struct.unpack("<Q", raw[:8])[0] == 41
    assert np.array_equal(np.frombuffer(raw[8:], dtype="<f8"), u)
    back = B._ref_read(p)
    assert np.array_equal(back, u) and back.flags.writeable
    p.write_bytes(raw[:50])  # truncated payload
    with pytest.raises(ValueError):
        B._ref_read(p)


def test_ref_key_is_sha256_of_fields():
    import hashlib
    k = B._ref_key("allen_cahn", 0.01, 12, 0.002)
    assert k == hashlib.sha256(b"allen_cahn|0.01|12|0.002").hexdigest()


def test_record_row_formats():
    rec = B.RunRecord(config=B.RunConfig("adr", 0.1, 32, "epirk4s3", "leja", 1e-6),
                      steps_accepted=5, l2_error=1.0 / 3.0)
    row = B.record_row(rec)
    assert row[:6] == ["adr", "0.10000000000000001", "32", "epirk4s3", "leja",
                       "9.9999999999999995e-07"]
    assert row[6] == "5" and row[13] == "0.33333333333333331" and row[14] == ""
    nan_row = B.record_row(B.RunRecord(
        config=B.RunConfig("semilinear", math.nan, 32, "epirk4s3", "kiops", 1e-6)))
    assert nan_row[1] == "" and nan_row[13] == "nan"


def test_write_csv_layout(tmp_path):
    cfg = B.RunConfig("adr", 0.1, 32, "epirk4s3", "leja", 1e-6)
    out = tmp_path / "w.csv"
    B.write_csv([B.RunRecord(config=cfg, error="StepFailure: x, y")], out)
    text = out.read_text(encoding="utf-8")
    assert text.split("\n")[0] == B.CSV_HEADER + ",error"
    assert "\r" not in text
    with out.open(newline="") as fh:
        rows = list(csv.reader(fh))
    assert len(rows) == 2 and len(rows[1]) == 15 and rows[1][-1] == "StepFailure: x, y"


def test_expand_matrix():
    cfgs = B.expand_matrix(B.SweepConfig(problems=["adr"], params={"adr": [0.1, 0.2]},
                                         n=32, tols=(1e-4, 1e-5)))
    # 2 params x (5 integrators x {leja, kiops} + 3 lekry) x 2 tols
    assert len(cfgs) == 2 * 13 * 2
    assert all(c.n == 32 for c in cfgs)
    assert [c.tol for c in cfgs[:2]] == [1e-4, 1e-5]
    assert not any(c.scheme == "lekry" and c.integrator == "exprb43" for c in cfgs)
    semi = B.expand_matrix(B.SweepConfig(problems=["semilinear"],
                                         params={"semilinear": [0.5]}, tols=(1e-4,)))
    assert semi and all(math.isnan(c.param) for c in semi)


# ------------------------------------------------------------------ device runs

def _oracle_run(cfg):
    from oracle import np_fields as OF, np_integrate as OI
    kw = {"n": cfg.n}
    if cfg.problem != "semilinear":
        kw["alpha"] = cfg.param
    q = OF.make(cfg.problem, **kw)
    t_final = cfg.t_final if cfg.t_final is not None else q.t_final
    return q, OI.adaptive(q.rhs, q.u0, t_final, cfg.integrator, cfg.scheme, cfg.tol,
                          jac_factory=q.jac_factory)


@pytest.mark.gpu
def test_exact_reference_semilinear():
    u = B.build_reference("semilinear", math.nan, 16)
    x = np.arange(1, 17) / 17.0
    assert np.allclose(u, x * (1.0 - x) * np.exp(1.0))


@pytest.mark.gpu
def test_reference_cache_hit(tmp_path):
    kw = dict(cache_dir=tmp_path, t_final=0.002)
    first = B.build_reference("allen_cahn", 1e-2, 12, **kw)
    files = list(tmp_path.glob("*.ref"))
    assert len(files) == 1
    assert files[0].name == B._ref_key("allen_cahn", 1e-2, 12, 0.002) + ".ref"
    stamp = files[0].stat().st_mtime_ns
    second = B.build_reference("allen_cahn", 1e-2, 12, **kw)
    assert np.array_equal(first, second)
    assert files[0].stat().st_mtime_ns == stamp


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [
    B.RunConfig("semilinear", math.nan, 16, "exprb43", "kiops", 1e-5),
    B.RunConfig("allen_cahn", 1e-2, 16, "epirk4s3", "leja", 1e-6, t_final=0.002),
    B.RunConfig("adr", 0.1, 16, "epirk4s3", "lekry", 1e-6, t_final=0.002),
])
def test_run_one_matches_oracle(cfg):
    """Leja / LeKry: counters identical to the oracle's adaptive run of the
    same config. KIOPS whole runs: the tier-3 envelope --
    accepted steps identical, work counters within 1 % (the device dots and
    norms differ from OpenBLAS ddot in the last ulp)."""
    u_ref = B.build_reference(cfg.problem, cfg.param, cfg.n, t_final=cfg.t_final)
    rec = B.run_one(cfg, u_ref=u_ref)
    assert not rec.failed, rec.error
    q, run = _oracle_run(cfg)
    for name in B._COUNTERS:
        ours, ref = getattr(rec, name), getattr(run, name)
        if cfg.scheme == "kiops" and name != "steps_accepted":
            assert abs(ours - ref) <= 0.01 * ref + 1, (name, ours, ref)
        else:
            assert ours == ref, (name, ours, ref)
    u_o = q.extract(run.u)
    err_o = np.linalg.norm(u_o - u_ref) / np.linalg.norm(u_ref)
    assert math.isclose(rec.l2_error, err_o, rel_tol=1e-3 if cfg.scheme != "kiops" else 0.5,
                        abs_tol=1e-13)
    rec2 = B.run_one(cfg, u_ref=u_ref)  # device runs are deterministic
    assert rec2.l2_error == rec.l2_error and rec2.rhs_evals == rec.rhs_evals


@pytest.mark.gpu
def test_run_one_records_failure():
    cfg = B.RunConfig("semilinear", math.nan, 16, "exprb43", "kiops", 1e-300)
    rec = B.run_one(cfg, u_ref=np.zeros(16))
    assert rec.failed and "StepFailure" in rec.error and math.isnan(rec.l2_error)


@pytest.mark.gpu
def test_run_sweep(tmp_path):
    sweep = B.SweepConfig(problems=["semilinear"], n=16, integrators=["exprb43"],
                          schemes=["kiops", "leja"], tols=(1e-4, 1e-6))
    out = tmp_path / "s.csv"
    recs = B.run_sweep(B.expand_matrix(sweep), out)
    assert len(recs) == 4 and not any(r.failed for r in recs)
    with out.open(newline="") as fh:
        rows = list(csv.reader(fh))
    assert len(rows) == 5
    for lo, hi in ((1, 2), (3, 4)):  # tighter tolerance -> smaller error
        assert float(rows[hi][13]) < float(rows[lo][13])
