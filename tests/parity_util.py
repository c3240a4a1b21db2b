"""Test infrastructure: gradient error tables in the reference's comparison
convention, max|a - b| / max|ref| (mmtplan tests/test_acceptance.py:66-68),
per module bucket and per named parameter tensor."""
from __future__ import annotations

import numpy as np

from paper_2403_07544_b200.model import bf16_round


def effective_weights(layout, master):
    """What the GPU computes with: bf16 matrices / tables, fp32 LN and biases."""
    out = master.copy()
    for p in layout.params.values():
        if p.init in ("xavier", "embed"):
            sl = slice(p.offset, p.offset + p.numel)
            out[sl] = bf16_round(master[sl])
    return out


def maxrel(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def error_table(g_eng: dict, g_ref: dict, layouts: dict, g_alt: dict = None) -> dict:
    """{module: {"engine": e, "alt": a, "tensors": {name: [e, a]}}} for every
    module whose reference gradient is non-zero; ``g_alt`` (optional) is a
    second implementation measured against the same reference."""
    rows = {}
    for k, g in g_eng.items():
        ref = g_ref.get(k)
        if ref is None:
            continue
        ref = np.asarray(ref, np.float64)
        if not np.abs(ref).max() > 0:
            continue
        alt = None if g_alt is None else np.asarray(g_alt[k], np.float64)
        row = {"engine": maxrel(g, ref), "alt": None if alt is None else maxrel(alt, ref), "tensors": {}}
        for name, p in layouts[k].params.items():
            sl = slice(p.offset, p.offset + p.numel)
            if np.abs(ref[sl]).max() > 0:
                row["tensors"][name] = [maxrel(g[sl], ref[sl]),
                                        None if alt is None else maxrel(alt[sl], ref[sl])]
        rows[str(k)] = row
    return rows
