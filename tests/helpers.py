"""Shared helpers for the parity tests (tests only)."""
import numpy as np

from oracle import oracle as O
from paper_1504_06768_b200 import configs


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind == "c":
        return np.array_equal(a.view(np.float64), b.view(np.float64))
    return np.array_equal(a, b)


def model(name, **kw):
    cfg = configs.CONFIGS[name]
    if name == "c4":
        return cfg["build"](kw.pop("i", 0), **kw)
    return cfg["build"](**kw)


def oracle_L(H, c_ops):
    return O.build_liouvillian(H.matrix, [c.matrix for c in c_ops])


def csr_equal(dev_csr, o):
    h = dev_csr.to_host()
    return (bits_equal(h.row_ptr, o.rp) and bits_equal(h.col_idx, o.ci)
            and bits_equal(h.values, o.v))
