"""CPU restatement of the max / mean aggregations (test infrastructure only: imported by
tests/ as the checker, never by the product path).

The reference implements only weighted-sum aggregation (aggregate, src/tensor.cpp:514-549),
so these two have no reference function to follow: they are PINNED ONLY TO THEIR
DEFINITIONS, which are written here loop for loop in the order include/gasb.h specifies
(parity for them is "definition-pinned", not reference-pinned):

  max_fwd : y[r] = x[c_b] for the row's first edge b, then replaced in CSR order by any strictly
            greater value (first occurrence wins; NaN survives only in first position);
            argmax[r] = that edge index; an empty row gives 0 / -1.
  max_bwd : gx[s] = fp32 sum over rows ascending of gy[r] where argmax[r] is an edge (r -> s).
  mean_fwd: y[r] = float(fp64 CSR-order sum / deg r), 0 for an empty row.
  mean coefficients: float(1.0 / deg r) per edge (the backward then is the weighted-sum
            backward, src/tensor.cpp:531-549).
"""
import numpy as np


def max_fwd(rowptr, cols, x):
    m, d = len(rowptr) - 1, x.shape[1]
    y = np.zeros((m, d), np.float32)
    arg = np.full((m, d), -1, np.int32)
    for r in range(m):
        b, e = int(rowptr[r]), int(rowptr[r + 1])
        if b == e:
            continue
        best = x[cols[b]].astype(np.float32).copy()
        bi = np.full(d, b, np.int32)
        for k in range(b + 1, e):
            v = x[cols[k]]
            gt = v > best
            best[gt] = v[gt]
            bi[gt] = k
        y[r], arg[r] = best, bi
    return y, arg


def max_bwd(rowptr, cols, arg, gy, num_src):
    d = gy.shape[1]
    gx = np.zeros((num_src, d), np.float32)
    for r in range(len(rowptr) - 1):  # rows ascending: each source's adds in ascending row order
        for k in range(int(rowptr[r]), int(rowptr[r + 1])):
            sel = arg[r] == k
            s = cols[k]
            gx[s, sel] = (gx[s, sel] + gy[r, sel]).astype(np.float32)
    return gx


def mean_fwd(rowptr, cols, x):
    m, d = len(rowptr) - 1, x.shape[1]
    y = np.zeros((m, d), np.float32)
    for r in range(m):
        b, e = int(rowptr[r]), int(rowptr[r + 1])
        if b == e:
            continue
        acc = np.zeros(d, np.float64)
        for k in range(b, e):
            acc = acc + x[cols[k]].astype(np.float64)
        y[r] = (acc / float(e - b)).astype(np.float32)
    return y


def mean_coefficients(rowptr):
    out = np.zeros(int(rowptr[-1]), np.float32)
    for r in range(len(rowptr) - 1):
        b, e = int(rowptr[r]), int(rowptr[r + 1])
        if e > b:
            out[b:e] = np.float32(1.0 / float(e - b))
    return out
