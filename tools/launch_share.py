"""Share of device time per kernel family in an ncu launch list
(`--metrics gpu__time_duration.sum --csv`; cold-cache and serialised, so compare the
SHARES with the bench line's CUDA-event `kernels` block, not the absolute times).

    python tools/launch_share.py profiles/r02_launches_c4.csv
"""

import csv
import re
import sys
from collections import defaultdict


def family(name: str) -> str:
    if "dgemm_tma_dmma" in name:
        m = re.search(r"GemmCfg<(\d+), (\d+)", name)
        tile = f"{m.group(1)}x{m.group(2)}" if m else "?"
        return {"128x128": "dgemm_tma_dmma (128x128)", "128x64": "dgemm_tma_dmma_upd (128x64)",
                "64x128": "dgemm_tma_dmma_skinny (64x128)"}.get(tile, f"dgemm {tile}")
    for key in ("panel_cl", "block_apply_cl", "panel_geqr2", "apply_t", "sum_partials", "t_merge", "splitk_reduce", "matrix_stats", "transpose",
                "load_v", "extract_r", "set_identity", "count_deficient", "gather"):
        if key in name:
            return key
    return name.split("(")[0][:40]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        f = family(r[ki])
        tot[f] += float(r[vi].replace(",", ""))
        cnt[f] += 1
    all_t = sum(tot.values())
    unit = h[h.index("Metric Unit")] if "Metric Unit" in h else ""
    print(f"{sum(cnt.values())} launches, {all_t:.4g} total ({rows[hdr + 1][h.index('Metric Unit')] if 'Metric Unit' in h else unit})")
    for f, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {f:36s} {cnt[f]:7d} launches  {100 * t / all_t:6.2f}%")


if __name__ == "__main__":
    main()
