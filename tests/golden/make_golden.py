"""Freeze the REAL reference's outputs into tests/golden/*.npz.

Run in the build container only (it imports the reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --configs  # + config 1/2 summaries (~1 min)
    python tests/golden/make_golden.py --rsvd     # only tests/golden/rsvd.npz
    python tests/golden/make_golden.py --profiles # only tests/golden/profiles.npz
    python tests/golden/make_golden.py --config 4 --surrogate 16384
                       # config 4 at full size and config 5's 16384^2 surrogate
                       # (each ~45 min per run on 8 cores, run twice for the spread)

The fixtures pin (a) the oracle restatement in oracle/urv_oracle.py and the
product's host RNG (tests/test_oracle_golden.py, CPU) and (b) the GPU path
(tests/test_gpu_*.py).  Inputs for the BASELINE configs are rebuilt at test
time by paper_1812_06007_b200.workloads, so only summaries (diag R, the
truncation grid, input checksums) are stored for them.
"""

from __future__ import annotations

import argparse
import functools
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def _import_reference():
    if not os.path.isdir(REF_SRC):
        raise SystemExit(f"reference not found at {REF_SRC}; fixtures can only be regenerated there")
    sys.path.insert(0, REF_SRC)
    import urv  # noqa: E402

    return urv


def _blas_tag():
    try:
        from threadpoolctl import threadpool_info

        info = [d for d in threadpool_info() if d.get("internal_api") == "openblas"]
        if info:
            return f"{info[0].get('version')}:{info[0].get('architecture')}"
    except Exception:
        pass
    return "unknown"


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max(d.get("num_threads", 0) for d in threadpool_info())
    except Exception:
        return 0


def rng_fixture(urv):
    cases = [((17, 9), (123, 4)), ((40, 40), (7, 0)), ((40, 13), (7, 0)), ((8, 8), (123, 1)),
             ((5, 3), (2 ** 64 - 1, 2 ** 63)), ((1, 1), (0, 0))]
    out = {}
    for i, ((m, n), seed) in enumerate(cases):
        out[f"draw{i}"] = urv.gaussian_matrix(m, n, urv.RngSeed(*seed))
        out[f"shape{i}"] = np.array([m, n])
        out[f"seed{i}"] = np.array(seed, dtype=np.uint64)
    out["spawn"] = np.array([tuple(urv.RngSeed(5, 3).spawn(7)), tuple(urv.RngSeed(5, 0).spawn(1)),
                             tuple(urv.RngSeed(1, 2 ** 63).spawn(2))], dtype=np.uint64)
    out["as_seed_int"] = np.array(tuple(urv.as_seed(-1)), dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def qr_fixture(urv):
    out = {}
    cases = [(50, 30, 42), (40, 40, 9), (200, 160, 9), (33, 1, 9), (70, 64, 3), (130, 97, 5)]
    for i, (m, n, s) in enumerate(cases):
        a = urv.gaussian_matrix(m, n, urv.RngSeed(s))
        res = urv.householder_qr(a)
        out[f"a{i}"], out[f"q{i}"], out[f"r{i}"] = a, res.q, res.r
    np.savez_compressed(os.path.join(HERE, "qr.npz"), **out)


def _summary(f):
    n = f.r.shape[0]
    ks = np.unique(np.round(np.linspace(0, n - 1, 10)).astype(np.int64))
    return {
        "diag": np.diag(f.r).copy(),
        "ks": ks,
        "trunc": np.array([np.linalg.norm(f.r[k:, k:]) for k in ks]),
        "warnings": np.array(list(f.provenance.warnings), dtype=object).astype(str),
    }


def powerurv_fixture(urv):
    """Small factorizations stored in full, matching the reference's own test matrices."""
    out = {}
    slow, _ = urv.gen_slow_decay(seed=0)          # 200 x 160, sigma_k = 1/k (matrices.py)
    out["slow_a"] = slow
    rank3 = (lambda m, n, r, seed: (urv.householder_qr(urv.gaussian_matrix(m, r, urv.as_seed(seed).spawn(1))).q
                                    * np.geomspace(1.0, 0.2, r))
             @ urv.householder_qr(urv.gaussian_matrix(n, r, urv.as_seed(seed).spawn(2))).q.T)(30, 20, 3, 12)
    out["rank3_a"] = rank3
    diag3 = np.zeros((5, 3))
    diag3[0, 0], diag3[1, 1], diag3[2, 2] = 4.0, 2.0, 1.0
    out["diag3_a"] = diag3
    out["rank1_a"] = np.outer(np.arange(1.0, 7.0), np.arange(1.0, 5.0))
    gauss = urv.gaussian_matrix(96, 64, urv.RngSeed(77))
    out["gauss_a"] = gauss
    cases = [
        ("slow_q1", "slow_a", 1, True, 8, True),
        ("slow_q2", "slow_a", 2, True, 8, False),
        ("slow_q0", "slow_a", 0, True, 17, False),
        ("slow_q1_noreorth", "slow_a", 1, False, 8, False),
        ("rank3_q2", "rank3_a", 2, True, 4, True),
        ("diag3_q10", "diag3_a", 10, True, 2, True),
        ("rank1_q1", "rank1_a", 1, True, 3, True),
        ("gauss_q2", "gauss_a", 2, True, 5, True),
        ("gauss_q1_noreorth", "gauss_a", 1, False, 6, True),
    ]
    names = []
    for name, akey, q, reorth, seed, full in cases:
        f = urv.power_urv(out[akey], q=q, reorth=reorth, seed=seed)
        names.append(name)
        out[f"{name}__meta"] = np.array([q, int(reorth), seed])
        out[f"{name}__akey"] = np.array(akey)
        for k, v in _summary(f).items():
            out[f"{name}__{k}"] = v
        if full:
            out[f"{name}__u"], out[f"{name}__r"], out[f"{name}__v"] = f.u, f.r, f.v
    out["cases"] = np.array(names)
    out["blas"] = np.array(_blas_tag())
    out["host"] = np.array(platform.processor() or platform.machine())
    np.savez_compressed(os.path.join(HERE, "powerurv.npz"), **out)


def rsvd_fixture(urv):
    """rsvd (factorizations.py:180-207) and lemma_check (diagnostics.py:197-214) on the
    reference's own test matrices."""
    out = {}
    pz = np.load(os.path.join(HERE, "powerurv.npz"))
    mats = {"slow_a": pz["slow_a"], "rank3_a": pz["rank3_a"], "gauss_a": pz["gauss_a"]}
    wide = urv.gaussian_matrix(40, 70, urv.RngSeed(21))
    wide[:, 35:] *= 1e-4
    mats["wide_a"] = wide
    out.update(mats)
    cases = [("slow_l60_q1", "slow_a", 60, 1, True, 0), ("slow_l60_q0", "slow_a", 60, 0, True, 3),
             ("slow_l17_q2_noreorth", "slow_a", 17, 2, False, 4), ("rank3_l3_q0", "rank3_a", 3, 0, True, 5),
             ("gauss_l20_q2", "gauss_a", 20, 2, True, 6), ("wide_l30_q1", "wide_a", 30, 1, True, 7),
             ("rank3_l10_q1", "rank3_a", 10, 1, True, 8)]
    names = []
    for name, akey, ell, q, reorth, seed in cases:
        f = urv.rsvd(mats[akey], ell, q=q, reorth=reorth, seed=seed)
        names.append(name)
        out[f"{name}__meta"] = np.array([ell, q, int(reorth), seed])
        out[f"{name}__akey"] = np.array(akey)
        out[f"{name}__u"], out[f"{name}__sigma"], out[f"{name}__v"] = f.u, f.sigma, f.v
        out[f"{name}__warnings"] = np.array(list(f.provenance.warnings), dtype=object).astype(str)
    out["cases"] = np.array(names)
    lem = [("slow_a", 60, 1, 12), ("slow_a", 60, 0, 12), ("slow_a", 5, 1, 2), ("gauss_a", 30, 2, 3)]
    out["lemma_cases"] = np.array([[i, ell, q, seed] for i, (k, ell, q, seed) in enumerate(lem)])
    out["lemma_akeys"] = np.array([k for k, *_ in lem])
    out["lemma_values"] = np.array([urv.lemma_check(mats[k], ell, q=q, seed=seed) for k, ell, q, seed in lem])
    out["blas"] = np.array(_blas_tag())
    np.savez_compressed(os.path.join(HERE, "rsvd.npz"), **out)


def config_fixture(urv, c, size=None):
    """Config c's reference run.  ``size`` scales a config down (config 5's 65536^2
    is infeasible on the CPU: its surrogate is the same iid N(0,1) construction and
    seeds at 16384^2), stored as config{c}s{size}.npz."""
    sys.path.insert(0, ROOT)
    from paper_1812_06007_b200 import workloads

    cfg = workloads.CONFIGS[c]
    if size is not None:
        cfg = workloads.Config(c, size, size, cfg.q, cfg.label)
    a = workloads.make_matrix(c, cfg.m, cfg.n)
    g = urv.gaussian_matrix(cfg.n, cfg.n, urv.RngSeed(c))
    t0 = time.perf_counter()
    f = urv.power_urv(a, q=cfg.q, reorth=True, seed=c)
    secs = time.perf_counter() - t0
    # intrinsic spread of the oracle: the same run with 64-wide panels
    fact = sys.modules["urv.factorizations"]
    orig = fact.householder_qr
    fact.householder_qr = functools.partial(orig, block_size=64)
    try:
        t0 = time.perf_counter()
        f64 = urv.power_urv(a, q=cfg.q, reorth=True, seed=c)
        secs64 = time.perf_counter() - t0
    finally:
        fact.householder_qr = orig
    s = _summary(f)
    s64 = _summary(f64)
    n = cfg.n
    out = {
        "a_sum": a.sum(), "a_sumsq": (a * a).sum(), "g_sum": g.sum(), "g_sumsq": (g * g).sum(),
        "recon": np.linalg.norm(f.u @ f.r @ f.v.T - a) / np.linalg.norm(a),
        "orth_u": np.linalg.norm(f.u.T @ f.u - np.eye(n)),
        "orth_v": np.linalg.norm(f.v.T @ f.v - np.eye(n)),
        "seconds": secs, "blas": np.array(_blas_tag()),
        "spread_diag": np.max(np.abs(s64["diag"] - s["diag"]) / np.abs(s["diag"])),
        "spread_trunc": np.max(np.abs(s64["trunc"] - s["trunc"]) / np.where(s["trunc"] > 0, s["trunc"], 1)),
    }
    out.update(s)
    out["m"], out["n"], out["q"] = np.array(cfg.m), np.array(cfg.n), np.array(cfg.q)
    out["seconds64"] = secs64
    out["threads"] = np.array(_blas_threads())
    out["host"] = np.array(platform.processor() or platform.machine())
    name = f"config{c}" if size is None else f"config{c}s{size}"
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {secs:.1f}s (block 64: {secs64:.1f}s) recon {out['recon']:.3e} "
          f"orth {out['orth_u']:.3e}/{out['orth_v']:.3e} spread diag {out['spread_diag']:.2e} "
          f"trunc {out['spread_trunc']:.2e}", flush=True)


def profiles_fixture(urv):
    """error_profile / reveal_profile (diagnostics.py:86-169) of the reference's own
    factorizations: the device profiles are checked on the reference's R (functions of
    R alone) and on the GPU factorization."""
    rng = np.random.default_rng(2024)
    out = {}
    cases = []
    m, n = 60, 40
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    cases.append(((u * np.geomspace(1.0, 1e-9, n)) @ v.T, 1, 3))                  # graded spectrum
    cases.append((rng.standard_normal((50, 6)) @ rng.standard_normal((6, 50)), 2, 5))  # rank 6 (deficient)
    cases.append((rng.standard_normal((33, 33)), 1, 7))                            # flat spectrum
    for i, (a, q, seed) in enumerate(cases):
        f = urv.power_urv(a, q=q, seed=seed)
        ep = urv.error_profile(a, f)
        rp = urv.reveal_profile(f, a)
        out[f"a{i}"] = a
        out[f"q{i}"] = np.array(q)
        out[f"seed{i}"] = np.array(seed)
        out[f"r{i}"] = f.r
        out[f"abs_sp{i}"] = ep.abs_spectral
        out[f"abs_fro{i}"] = ep.abs_frobenius
        out[f"sigma_ref{i}"] = ep.sigma_ref
        out[f"smin{i}"] = rp.smin_r11
        out[f"smax{i}"] = rp.smax_r22
    out["blas"] = np.array(_blas_tag())
    np.savez_compressed(os.path.join(HERE, "profiles.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true", help="also freeze config 1 and 2 summaries")
    ap.add_argument("--rsvd", action="store_true", help="only regenerate rsvd.npz")
    ap.add_argument("--profiles", action="store_true", help="only regenerate profiles.npz")
    ap.add_argument("--config", type=int, action="append", default=[],
                    help="freeze the summary of one more config (3: ~12 min on 8 cores)")
    ap.add_argument("--surrogate", type=int, action="append", default=[],
                    help="config 5 construction scaled to this square size (16384: ~90 min on 8 cores)")
    args = ap.parse_args()
    urv = _import_reference()
    if args.rsvd:
        rsvd_fixture(urv)
        return
    if args.profiles:
        profiles_fixture(urv)
        return
    if not args.config and not args.surrogate:
        rng_fixture(urv)
        qr_fixture(urv)
        powerurv_fixture(urv)
        rsvd_fixture(urv)
    if args.configs:
        for c in (1, 2):
            config_fixture(urv, c)
    for c in args.config:
        config_fixture(urv, c)
    for size in args.surrogate:
        config_fixture(urv, 5, size)


if __name__ == "__main__":
    main()
