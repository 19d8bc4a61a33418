"""Shared helpers of the GPU parity tests: stack seeded scenarios on the
device and compute the matching oracle quantities."""
import numpy as np
import scipy.sparse as sp

from oracle import pf_oracle as O


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def stack(points, key):
    return np.stack([np.asarray(p[key], dtype=np.float64) for p in points])


def dev(a, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or torch.float64, device="cuda")


def csr_dense(ptr, idx, val, shape):
    rows = np.repeat(np.arange(shape[0]), np.diff(ptr))
    D = np.zeros(shape)
    np.add.at(D, (rows, idx), val)
    return D


def oracle_khat(net, pt):
    part = O.partition(net)
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
    return O.reduce_naive(K, Gx, Gu), part
