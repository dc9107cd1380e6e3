"""pytest plugin (test infrastructure): run the REFERENCE's own test modules with its
hot path replaced by this repo's drop-in ("Reuse in the build").

Loaded by tests/test_gpu_reference_suite.py as ``-p dropin_plugin`` with the reference
copy (baseline/_ref/src, made by __graft_entry__.build() from /root/reference) on
PYTHONPATH.  Every ``urv`` module's binding of power_urv / ddh_urv / rsvd /
lemma_check is replaced by paper_1812_06007_b200's, so the reference's own
assertions (invariants, error paths, warnings, bitwise q=0 == ddh, thread
safety, acceptance criteria) run against the GPU implementation.
"""

import sys

# the drop-in boundary plus the SURVEY 8(f) rows built on it; the
# exception class is part of the boundary: a caller's `except urv.RankCollapseError`
# must catch what the drop-in raises
# and so are the result types (the reference's error_profile dispatches on
# isinstance(f, RsvdFactorization), diagnostics.py:125)
REPLACED = ("power_urv", "ddh_urv", "rsvd", "lemma_check", "RankCollapseError", "RsvdFactorization",
            "UrvFactorization")


def pytest_configure(config):
    import urv  # the reference (baseline/_ref/src)
    import paper_1812_06007_b200 as dropin

    assert "baseline" in urv.__file__, urv.__file__
    for name, mod in list(sys.modules.items()):
        if name == "urv" or name.startswith("urv."):
            for fn in REPLACED:
                if hasattr(mod, fn):
                    setattr(mod, fn, getattr(dropin, fn))
    print(f"[dropin] urv.{{{', '.join(REPLACED)}}} -> paper_1812_06007_b200 (GPU)", file=sys.__stderr__)
