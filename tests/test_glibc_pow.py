"""The device's pow (csrc/vr_glibc_pow.h) is libm's pow bit for bit.

The reference's numba kernels evaluate `x ** y` with libm's pow (glibc 2.39:
<= 0.52 ulp, not correctly rounded); the kernels run the same algorithm on
tables extracted from libm.  Here the header is compiled for the host and
compared with libm's pow on random and special inputs, and the committed
tables are checked against the libm of this image.
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))


def test_tables_match_this_libm():
    import gen_pow_tables as g

    committed = (g.CSRC / "vr_pow_tables.h").read_text()
    ln2hi, ln2lo, poly, tab, hdr, etab = g.extract()
    assert f"#define VR_POW_LN2HI {ln2hi.hex()}" in committed
    for invc, _pad, logc, logctail in tab:
        assert f"{{{invc.hex()}, {logc.hex()}, {logctail.hex()}}}," in committed
    for x in etab[::17]:
        assert f"0x{x:016x}ull," in committed


def test_device_pow_equals_libm_pow():
    import gen_pow_tables as g

    assert g.check(3_000_000)
