"""Light clusters for clustered NVC (reference sampling.py:226-295).

``ClusterSet`` is the cluster description the sampler and the cluster-target
kernels consume; ``kmeans_cluster`` builds one.  Both run once per scene on
the host.  The per-frame work that uses the clusters -- shadow-ray targets
toward a random member of each cluster and the two-step (cluster WRS, then
member RIS) light sampler -- runs in libnvc (``nvc_cluster_targets``,
``nvc_clustered_select``), which reads the packed layout of ``pack_clusters``.

The clustering is an ordinary Lloyd iteration on the light centroids kept as
a label vector.  Its floating-point results (centroids, inertia history) are
pinned against the reference by ``tests/golden/clusters.npz``: seeds come
from the caller's numpy Generator (``choice`` without replacement), squared
distances are summed x, y, z in that order, and each centroid is the
sequential sum of its members' coordinates in light order divided by the
member count.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class ClusterSet:
    """m clusters of light ids; ``assignment[light] = cluster``."""

    centroids: np.ndarray
    members: list
    inertia_history: list = field(default_factory=list)

    def __post_init__(self):
        self.members = [np.asarray(ids, dtype=np.int64) for ids in self.members]
        counts = np.fromiter((ids.size for ids in self.members), dtype=np.int64, count=len(self.members))
        if (counts == 0).any():
            raise ValueError("empty cluster after repair")
        self.assignment = np.repeat(np.arange(counts.size, dtype=np.int64), counts)[
            np.argsort(np.concatenate(self.members), kind="stable")] if counts.size else np.zeros(0, np.int64)

    @property
    def m(self) -> int:
        return len(self.members)

    def member_count(self, j: int) -> int:
        return int(self.members[j].size)

    def packed(self):
        return pack_clusters(self)


def pack_clusters(clusters):
    """(offsets (m+1) int32, flat member ids int32): the device layout.  Works
    for this module's ClusterSet and for the reference's (same ``members``)."""
    members = [np.asarray(ids, dtype=np.int64) for ids in clusters.members]
    off = np.zeros(len(members) + 1, dtype=np.int32)
    off[1:] = np.cumsum([ids.size for ids in members])
    flat = np.concatenate(members).astype(np.int32) if members else np.zeros(0, np.int32)
    return off, flat


def _sq_dist(pts: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """(n, k) squared distances, axes summed in x, y, z order."""
    d = pts[:, None, :] - centers[None, :, :]
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def _recenter(pts: np.ndarray, labels: np.ndarray, centers: np.ndarray) -> None:
    """Move every non-empty cluster's center to its members' mean (in place);
    empty clusters keep their center (inertia stays non-increasing)."""
    k = centers.shape[0]
    counts = np.bincount(labels, minlength=k)
    live = counts > 0
    for a in range(3):
        sums = np.bincount(labels, weights=pts[:, a], minlength=k)
        centers[live, a] = sums[live] / counts[live]


def kmeans_cluster(lights, k: int, rng: np.random.Generator, max_iters: int = 100) -> ClusterSet:
    """Lloyd iterations over light centroids until the labels stop changing
    (at most ``max_iters`` assignments), then every empty cluster takes the
    member of the largest cluster farthest from that cluster's center.  With
    ``k >= #lights`` each light is its own cluster (no draws)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    pts = np.stack([lt.centroid() for lt in lights])
    n = pts.shape[0]
    if k >= n:
        return ClusterSet(centroids=pts.copy(), members=[np.array([i]) for i in range(n)])
    centers = pts[rng.choice(n, size=k, replace=False)].copy()
    labels = None
    history = []
    rows = np.arange(n)
    for _ in range(max_iters):
        d2 = _sq_dist(pts, centers)
        new = d2.argmin(axis=1)
        history.append(float(d2[rows, new].sum()))
        if labels is not None and np.array_equal(new, labels):
            break
        labels = new
        _recenter(pts, labels, centers)
    members = [np.flatnonzero(labels == j) for j in range(k)]
    # repair: with k < n an empty cluster implies a donor of size >= 2, so one
    # ascending pass over the empty clusters never empties a donor
    for j in range(k):
        if members[j].size:
            continue
        donor = int(np.argmax([ids.size for ids in members]))
        ids = members[donor]
        far = ids[np.argmax(_sq_dist(pts[ids], centers[donor:donor + 1])[:, 0])]
        members[donor] = ids[ids != far]
        members[j] = np.array([far])
        centers[j] = pts[far]
    return ClusterSet(centroids=centers, members=members, inertia_history=history)


__all__ = ["ClusterSet", "kmeans_cluster", "pack_clusters"]
