"""Helpers for GPU-vs-oracle parity tests: both sides build their hierarchies from the same
seeded cloud; comparisons are made in ORIGINAL point-id space so that neither side's
internal ordering matters.  Nothing here computes the method."""
import numpy as np


def coo_ids(ptr, col, val, row_ids, col_ids):
    """(row id, col id, value) triples sorted by (row id, col id)."""
    rows = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    r = row_ids[rows]
    c = col_ids[np.asarray(col, dtype=np.int64)]
    o = np.lexsort((c, r))
    return r[o], c[o], np.asarray(val)[o]


def relmax(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.abs(a - b).max() if a.size else 0.0
    s = np.abs(b).max() if b.size else 0.0
    return d / s if s > 0 else d


class Pair:
    """GPU hierarchy (through the C ABI) + oracle hierarchy for one workload."""

    def __init__(self, w):
        from paper_2204_06154_b200 import MGM
        import oracle as O

        self.w = w
        self.gpu = MGM(w.points, w.normals, w.stencil, w.levels)
        self.ref = O.Oracle(w.points, w.normals, w.stencil, w.levels)
        self.poisson = w.stencil.get("problem", 0) == 1
        from paper_2204_06154_b200 import mgm_export_level
        self.glv = [mgm_export_level(self.gpu.ctx, j, self.poisson) for j in range(self.gpu.p)]

    def oracle_pos(self, j):
        """orig id -> oracle row on level j"""
        ids = self.ref.levels[j].ids
        pos = np.full(len(self.w.points), -1, dtype=np.int64)
        pos[ids] = np.arange(len(ids))
        return pos

    def to_oracle_order(self, j, v_lib):
        """GPU lib-order level vector -> oracle (Morton) order, keeping the multiplier."""
        g = self.glv[j]
        pos = self.oracle_pos(j)
        n = g["n"]
        out = np.empty_like(v_lib)
        out[pos[g["ids"]]] = v_lib[:n]
        if len(v_lib) > n:
            out[n:] = v_lib[n:]
        return out

    def to_lib_order(self, j, v_mor):
        g = self.glv[j]
        pos = self.oracle_pos(j)
        n = g["n"]
        out = np.empty_like(v_mor)
        out[:n] = v_mor[pos[g["ids"]]]
        if len(v_mor) > n:
            out[n:] = v_mor[n:]
        return out

    def close(self):
        self.gpu.close()
