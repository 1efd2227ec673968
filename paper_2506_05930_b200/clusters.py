"""Light clusters for clustered NVC (sampling.py:226-295): ``ClusterSet`` and
``kmeans_cluster``.

Clustering runs once per scene on the host, exactly like the reference: the
same numpy Generator draws (``rng.choice``), the same Lloyd iterations over
light centroids and the same empty-cluster repair, so member lists, centroids
and the inertia history are identical.  The per-frame work that uses the
clusters -- shadow-ray targets toward a random member of each cluster and the
two-step (cluster WRS, then member RIS) light sampler -- runs in libnvc
(``nvc_cluster_targets``, ``nvc_clustered_select``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class ClusterSet:
    """m clusters of light ids; ``assignment[light] = cluster`` (sampling.py:226-249)."""

    centroids: np.ndarray
    members: list
    inertia_history: list = field(default_factory=list)

    def __post_init__(self):
        self.members = [np.asarray(mem, dtype=np.int64) for mem in self.members]
        sizes = np.array([mem.size for mem in self.members])
        if np.any(sizes == 0):
            raise ValueError("empty cluster after repair")
        self.assignment = np.empty(int(sizes.sum()), dtype=np.int64)
        for j, mem in enumerate(self.members):
            self.assignment[mem] = j

    @property
    def m(self) -> int:
        return len(self.members)

    def member_count(self, j: int) -> int:
        return int(self.members[j].size)

    def packed(self):
        """(offsets (m+1) int32, flat member ids int32) -- the device layout."""
        sizes = np.array([mem.size for mem in self.members], dtype=np.int64)
        off = np.zeros(self.m + 1, dtype=np.int32)
        off[1:] = np.cumsum(sizes)
        flat = np.concatenate(self.members).astype(np.int32) if self.m else np.zeros(0, np.int32)
        return off, flat


def kmeans_cluster(lights, k: int, rng: np.random.Generator, max_iters: int = 100) -> ClusterSet:
    """Lloyd's algorithm on light centroids (sampling.py:252-295).

    Seeds: k distinct lights from ``rng.choice``.  Iterates until the
    assignment stops changing (or max_iters); a cluster that empties keeps its
    centroid.  Afterwards every empty cluster takes the member of the largest
    cluster farthest from that cluster's centroid.  k >= #lights: one light per
    cluster (no draws)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    pts = np.stack([lt.centroid() for lt in lights])
    n = pts.shape[0]
    if k >= n:
        return ClusterSet(centroids=pts.copy(), members=[np.array([i]) for i in range(n)])
    cen = pts[rng.choice(n, size=k, replace=False)].copy()
    assign = np.full(n, -1, dtype=np.int64)
    history = []
    for _ in range(max_iters):
        d2 = np.sum((pts[:, None, :] - cen[None, :, :]) ** 2, axis=2)
        nxt = np.argmin(d2, axis=1)
        history.append(float(d2[np.arange(n), nxt].sum()))
        if np.array_equal(nxt, assign):
            break
        assign = nxt
        for j in range(k):
            sel = assign == j
            if np.any(sel):
                cen[j] = pts[sel].mean(axis=0)
    members = [np.flatnonzero(assign == j) for j in range(k)]
    while any(mem.size == 0 for mem in members):
        empty = next(j for j, mem in enumerate(members) if mem.size == 0)
        big = int(np.argmax([mem.size for mem in members]))
        pool = members[big]
        far = pool[np.argmax(np.sum((pts[pool] - cen[big]) ** 2, axis=1))]
        members[big] = pool[pool != far]
        members[empty] = np.array([far])
        cen[empty] = pts[far]
    return ClusterSet(centroids=cen, members=members, inertia_history=history)


__all__ = ["ClusterSet", "kmeans_cluster"]
