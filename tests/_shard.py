"""The row-sharding protocol of a multi-rank build, restated in numpy for the tests (DESIGN.md §9,
include/cleora.h cleora_build): the mirrored entry list (originals in input order, then the mirrors
of the non-self-loop edges of an undirected graph, reading B1), every row's entry count in it
(before merging duplicates), cut p = the first row whose entry prefix reaches p * total / world, and
a rank's entries = those of its rows, in list order.  Counting and filtering only: none of the
method's arithmetic (the oracle builds M from the filtered list)."""
import numpy as np


def mirrored(g):
    """(rows, cols, weights) of the mirrored entry list, in list order."""
    src = np.asarray(g.src, np.int64)
    dst = np.asarray(g.dst, np.int64)
    w = None if g.w is None else np.asarray(g.w, np.float32)
    if g.directed:
        return src, dst, w
    m = src != dst
    rows = np.concatenate([src, dst[m]])
    cols = np.concatenate([dst, src[m]])
    ws = None if w is None else np.concatenate([w, w[m]])
    return rows, cols, ws


def cuts(g, world):
    rows, _, _ = mirrored(g)
    prefix = np.zeros(g.n + 1, np.int64)
    prefix[1:] = np.cumsum(np.bincount(rows, minlength=g.n))
    tot = int(prefix[-1])
    c = [0]
    for p in range(1, world):
        c.append(int(np.argmax(prefix * world >= p * tot)))      # first row reaching p * tot / world
    c.append(g.n)
    return np.array(c, np.int64)


def shard_edges(g, r0, r1):
    """The entries of rows [r0, r1), as a directed edge list in list order."""
    rows, cols, w = mirrored(g)
    k = (rows >= r0) & (rows < r1)
    return rows[k].astype(np.int32), cols[k].astype(np.int32), None if w is None else w[k]
