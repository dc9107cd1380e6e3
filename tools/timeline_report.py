"""Summarise a tools/timeline.py capture (one power_urv call, every scope timed).

    python tools/timeline_report.py gpurun_out/timeline_c4.npz

Per kernel class and stream: launches, summed device time, flops, rate; GEMM launches
bucketed by size; the wall-clock split into "a 128x128/128x64 GEMM is running",
"only small kernels", "panel only", "idle"."""

import sys

import numpy as np

PEAK = 37.15


def union(iv):
    if len(iv) == 0:
        return 0.0, []
    iv = iv[np.argsort(iv[:, 0])]
    out = []
    s, e = iv[0]
    for a, b in iv[1:]:
        if a > e:
            out.append((s, e))
            s, e = a, b
        else:
            e = max(e, b)
    out.append((s, e))
    return sum(b - a for a, b in out), out


def main():
    z = np.load(sys.argv[1], allow_pickle=True)
    tl, names = z["tl"], list(z["names"])
    cls, stream, t0, t1, fl = tl[:, 0].astype(int), tl[:, 1].astype(int), tl[:, 2], tl[:, 3], tl[:, 4]
    dur = t1 - t0
    span = t1.max() - t0.min()
    print(f"records {len(tl)}  span {span:.1f} ms  flops {fl.sum() / 1e12:.2f} TF  "
          f"rate over span {fl.sum() / 1e9 / span:.2f} TF/s ({fl.sum() / 1e9 / span / PEAK:.1%} of {PEAK})")
    print("\nper class x stream: launches, summed ms, TF, TF/s")
    for c in sorted(set(cls)):
        for s in sorted(set(stream[cls == c])):
            m = (cls == c) & (stream == s)
            ms = dur[m].sum()
            print(f"  {names[c]:24s} s{s}  {m.sum():6d}  {ms:9.1f} ms  {fl[m].sum() / 1e12:7.2f} TF  "
                  f"{fl[m].sum() / 1e9 / ms if ms else 0:6.2f}")
    gemm = np.array([n.startswith("dgemm") for n in names])[cls]
    print("\nGEMM launches by size (flops): launches, summed ms, TF/s")
    edges = [0, 1e8, 1e9, 1e10, 1e11, 1e13]
    for lo, hi in zip(edges[:-1], edges[1:]):
        m = gemm & (fl >= lo) & (fl < hi)
        ms = dur[m].sum()
        print(f"  [{lo:.0e}, {hi:.0e})  {m.sum():6d}  {ms:9.1f} ms  {fl[m].sum() / 1e9 / ms if ms else 0:6.2f}")
    big = gemm & (fl >= 1e10)
    panel = np.array([n == "panel_geqr2" for n in names])[cls]
    u_big, _ = union(np.stack([t0[big], t1[big]], 1))
    u_any, _ = union(np.stack([t0, t1], 1))
    u_gemm, _ = union(np.stack([t0[gemm], t1[gemm]], 1))
    u_nobig = np.stack([t0[~big], t1[~big]], 1)
    # time with no big GEMM running, split into panel / other / idle by sampling
    grid = np.linspace(t0.min(), t1.max(), 200001)
    def covered(mask):
        iv = np.stack([t0[mask], t1[mask]], 1)
        _, segs = union(iv)
        cov = np.zeros_like(grid, dtype=bool)
        for a, b in segs:
            cov |= (grid >= a) & (grid < b)
        return cov
    cb, cp, ca = covered(big), covered(panel), covered(np.ones_like(big))
    print(f"\nwall {span:.1f} ms: big GEMM (>=1e10 flop) running {u_big:.1f} ms ({u_big / span:.1%}); any GEMM "
          f"{u_gemm:.1f} ms; any kernel {u_any:.1f} ms")
    print(f"  no big GEMM: panel running {np.mean(~cb & cp):.1%}, other kernels only {np.mean(~cb & ~cp & ca):.1%}, "
          f"idle {np.mean(~ca):.1%}")
    print(f"  big GEMM co-running with a panel {np.mean(cb & cp):.1%}")


if __name__ == "__main__":
    main()
