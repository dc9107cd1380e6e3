"""CPU: pin the oracle restatement (oracle/urv_oracle.py) and the product's host
RNG to the real reference's frozen outputs (tests/golden, made by make_golden.py)."""

import os

import numpy as np
import pytest

from paper_1812_06007_b200 import random as prng
from paper_1812_06007_b200 import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def _same_blas(z):
    try:
        from golden.make_golden import _blas_tag  # type: ignore
    except Exception:
        import importlib.util

        spec = importlib.util.spec_from_file_location("mg", os.path.join(GOLD, "make_golden.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _blas_tag = mod._blas_tag
    return str(z["blas"]) == _blas_tag()


@pytest.mark.parametrize("gen", ["oracle", "product"])
def test_gaussian_draws_bit_exact(gen, oracle):
    z = _load("rng.npz")
    mod = oracle if gen == "oracle" else prng
    i = 0
    while f"draw{i}" in z:
        m, n = z[f"shape{i}"]
        seed = tuple(int(x) for x in z[f"seed{i}"])
        got = mod.gaussian_matrix(int(m), int(n), mod.RngSeed(*seed))
        assert np.array_equal(got, z[f"draw{i}"]), f"draw {i}"
        assert got.flags.f_contiguous
        i += 1
    spawn = [tuple(mod.RngSeed(5, 3).spawn(7)), tuple(mod.RngSeed(5, 0).spawn(1)),
             tuple(mod.RngSeed(1, 2 ** 63).spawn(2))]
    assert np.array_equal(np.array(spawn, dtype=np.uint64), z["spawn"])
    assert tuple(mod.as_seed(-1)) == tuple(int(x) for x in z["as_seed_int"])


def test_blocked_gaussian_fill_bit_exact():
    ref = prng.gaussian_matrix(300, 7, prng.RngSeed(9, 2))
    out = np.empty((300, 7), order="F")
    prng.gaussian_matrix(300, 7, prng.RngSeed(9, 2), out=out)
    assert np.array_equal(ref, out)


def test_gaussian_rejects_empty(oracle):
    for mod in (oracle, prng):
        with pytest.raises(ValueError):
            mod.gaussian_matrix(0, 3, 1)


def test_oracle_qr_matches_reference(oracle):
    z = _load("qr.npz")
    i = 0
    while f"a{i}" in z:
        res = oracle.householder_qr(z[f"a{i}"])
        if np.array_equal(res.q, z[f"q{i}"]) and np.array_equal(res.r, z[f"r{i}"]):
            pass  # bit-exact (same host BLAS)
        else:
            np.testing.assert_allclose(res.q, z[f"q{i}"], rtol=0, atol=1e-13)
            np.testing.assert_allclose(res.r, z[f"r{i}"], rtol=0, atol=1e-13 * np.abs(z[f"r{i}"]).max())
        i += 1


def test_oracle_qr_bitwise_on_fixture_host(oracle):
    z = _load("powerurv.npz")
    if not _same_blas(z):
        pytest.skip("host BLAS differs from the fixture host; bitwise check not applicable")
    q = _load("qr.npz")
    res = oracle.householder_qr(q["a2"])
    assert np.array_equal(res.q, q["q2"]) and np.array_equal(res.r, q["r2"])


def test_oracle_power_urv_matches_reference(oracle):
    z = _load("powerurv.npz")
    bitwise = _same_blas(z)
    for name in z["cases"]:
        name = str(name)
        q, reorth, seed = (int(x) for x in z[f"{name}__meta"])
        a = z[str(z[f"{name}__akey"])]
        f = oracle.power_urv(a, q=q, reorth=bool(reorth), seed=seed)
        assert list(f.provenance.warnings) == [str(w) for w in z[f"{name}__warnings"]], name
        if f"{name}__u" in z:
            for key, got in (("u", f.u), ("r", f.r), ("v", f.v)):
                ref = z[f"{name}__{key}"]
                if bitwise:
                    assert np.array_equal(got, ref), (name, key)
                else:
                    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
        d = np.diag(f.r)
        np.testing.assert_allclose(d, z[f"{name}__diag"], rtol=1e-9, atol=1e-14 * max(1.0, np.abs(d).max()))


def test_oracle_rsvd_matches_reference(oracle):
    # rsvd (factorizations.py:180-207) and lemma_check (diagnostics.py:197-214)
    z = _load("rsvd.npz")
    bitwise = _same_blas(z)
    for name in z["cases"]:
        name = str(name)
        ell, q, reorth, seed = (int(x) for x in z[f"{name}__meta"])
        a = z[str(z[f"{name}__akey"])]
        f = oracle.rsvd(a, ell, q=q, reorth=bool(reorth), seed=seed)
        assert list(f.provenance.warnings) == [str(w) for w in z[f"{name}__warnings"]], name
        for key, got in (("u", f.u), ("sigma", f.sigma), ("v", f.v)):
            ref = z[f"{name}__{key}"]
            if bitwise:
                assert np.array_equal(got, ref), (name, key)
            else:
                np.testing.assert_allclose(got, ref, rtol=0, atol=1e-10 * max(1.0, np.abs(ref).max()))
    for (i, ell, q, seed), akey, val in zip(z["lemma_cases"], z["lemma_akeys"], z["lemma_values"]):
        got = oracle.lemma_check(z[str(akey)], int(ell), q=int(q), seed=int(seed))
        assert got == val if bitwise else abs(got - val) <= 1e-13, (i, got, val)


def test_oracle_config1_summary(oracle):
    z = _load("config1.npz")
    cfg = workloads.CONFIGS[1]
    a = workloads.make_matrix(1)
    assert abs(a.sum() - float(z["a_sum"])) <= 1e-9 * abs(float(z["a_sumsq"])) ** 0.5 * a.size ** 0.5
    f = oracle.power_urv(a, q=cfg.q, reorth=True, seed=1)
    d = np.diag(f.r)
    spread = max(float(z["spread_diag"]), 1e-12)
    assert np.max(np.abs(d - z["diag"]) / np.abs(z["diag"])) <= max(1e-8, 10 * spread)
    trunc = np.array([np.linalg.norm(f.r[k:, k:]) for k in z["ks"]])
    np.testing.assert_allclose(trunc, z["trunc"], rtol=1e-8)


def test_flop_model_matches_survey():
    # F_alg for configs 1-5
    expect = {1: 1.400e10, 2: 1.4933e12, 3: 1.2186e13, 4: 1.0262e14, 5: 6.5677e15}
    for c, val in expect.items():
        cfg = workloads.CONFIGS[c]
        assert abs(workloads.flop_alg(cfg.m, cfg.n, cfg.q) / val - 1) < 5e-4, c
    assert abs(workloads.flop_paper(16384, 16384, 2) / 7.330e13 - 1) < 1e-3


def test_numpy_ziggurat_tables_located_and_verified():
    # host logic of the device Gaussian draw: NumPy's exact tables are found and
    # reproduce NumPy's standard_normal stream bit for bit (wedge + tail paths included)
    tabs = prng.ziggurat_tables()
    assert tabs is not None, "NumPy ziggurat tables could not be verified on this host"
    wi, fi, ki = tabs
    assert wi.shape == fi.shape == ki.shape == (256,)
    assert fi[0] == 1.0 and ki[1] == 0 and np.all(np.diff(fi[1:]) < 0)
    k = np.array([424242, 7], dtype=np.uint64)
    raw = [int(v) for v in np.random.Philox(key=k).random_raw(60000)]
    mine = prng._numpy_standard_normal_restated(raw, 50000, wi.tolist(), fi.tolist(), [int(v) for v in ki])
    ref = np.random.Generator(np.random.Philox(key=k)).standard_normal(50000)
    assert np.array_equal(mine, ref)


def test_oracle_profiles_match_reference(oracle):
    """oracle.error_profile / reveal_profile restate diagnostics.py:86-169 (pinned)."""
    g = np.load(os.path.join(GOLD, "profiles.npz"))
    for i in range(3):
        a, r = g[f"a{i}"], g[f"r{i}"]
        f = oracle.power_urv(a, q=int(g[f"q{i}"]), seed=int(g[f"seed{i}"]))
        sp, fro, sref = oracle.error_profile(a, f)
        scale = np.linalg.norm(a)
        np.testing.assert_allclose(fro, g[f"abs_fro{i}"], atol=1e-12 * scale)
        np.testing.assert_allclose(sp, g[f"abs_sp{i}"], atol=1e-12 * scale)
        np.testing.assert_allclose(sref, g[f"sigma_ref{i}"], rtol=1e-12, atol=1e-14 * scale)
        smin, smax = oracle.reveal_profile(r)
        np.testing.assert_allclose(smin, g[f"smin{i}"], atol=1e-12 * scale)
        np.testing.assert_allclose(smax, g[f"smax{i}"], atol=1e-12 * scale)
