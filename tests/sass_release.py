"""SASS check of the GEMM ring's consumer release (used by tests/test_sass_release.py).

The FP64 GEMM reads its operand ring with LDS and hands a slot back to the TMA
producer with an mbarrier arrive.  ptxas does not make that arrive wait for the
warp's outstanding LDS (the arrive's scoreboard wait mask is empty), so the next
TMA load can overwrite a slot that is still being read -- a race that showed up
as wrong 32x32 warp tiles under concurrent streams.  The kernel therefore fences
(MEMBAR.CTA) before the arrive; this checker walks `cuobjdump -sass` output and
fails if any LDS scoreboard is still pending at a consumer arrive or a CTA barrier.
"""

from __future__ import annotations

import re


def pending_loads_at_releases(sass: str):
    """[(function, address, {scoreboard: lds_address})] for every consumer arrive / BAR.SYNC."""
    lines = sass.splitlines()
    func, pending, out = None, {}, []
    i = 0
    while i < len(lines):
        ln = lines[i]
        m = re.search(r"Function : (\S+)", ln)
        if m:
            func, pending = m.group(1), {}
            i += 1
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", ln)
        if m and i + 1 < len(lines):
            m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
            if m2:
                addr, text = m.group(1), m.group(2)
                ctrl = int(m2.group(1), 16) >> 41  # Volta+ control bits of the 128-bit instruction
                wrbar, waitmask = (ctrl >> 5) & 7, (ctrl >> 11) & 63
                for b in list(pending):
                    if waitmask >> b & 1:
                        del pending[b]
                if "SYNCS.ARRIVE.TRANS64.A1T0" in text or "BAR.SYNC" in text:
                    out.append((func, addr, dict(pending)))
                if re.search(r"\bLDS", text) and wrbar != 7:
                    pending[wrbar] = addr
                i += 2
                continue
        i += 1
    return out
