"""Host-only guard on the ptxas report of libtilefact.so (paper_0709_1272_b200/build_ptxas.log,
written by build()): the hot register-slab / engine variants must not spill.  The persistent
kernel's noinline variants are register-allocated by ptxas across the whole call graph, and an
unrelated change can push one of them into local-memory spills (measured: an inlined
shared-memory TRSM block moved the QR slab variants to 60-220 B of spills and config 2 from
13.0 to 13.9 ms)."""
import os
import re

import pytest

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_0709_1272_b200",
                   "build_ptxas.log")

# variant (mangled-name fragment) -> spill-store budget in bytes
BUDGET = {
    "v_qr_slabILi1E": 0, "v_qr_slabILi2E": 0,          # GEQRT / TSQRT, configs 2-3 and b = 128
    "v_ssrfb_mirrorILi2E": 0, "v_larfb_regILi2E": 0,   # config 2 updates
    "v_gemmENS_3Ctx": 96, "v_syrkENS_3Ctx": 64,        # config 4 (a few bytes of spilled indices)
    "v_ssrfb_mirrorILi4E": 128,                        # config 5
}


def _spills():
    if not os.path.exists(LOG):
        pytest.skip("no build report (run build() first)")
    out, cur = {}, None
    for line in open(LOG):
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if cur and m:
            out[cur] = int(m.group(1))
            cur = None
    return out


def test_hot_variants_do_not_spill():
    sp = _spills()
    for frag, budget in BUDGET.items():
        hits = {k: v for k, v in sp.items() if frag in k}
        assert hits, f"{frag} not in the build report"
        for k, v in hits.items():
            assert v <= budget, f"{k}: {v} bytes of spill stores (budget {budget})"
