"""Element partitioning for multi-GPU runs (the
reference has no distributed path, hybridwave/SPEC.md:440).

A rank's local mesh holds its owned elements followed by ghost copies of
the off-rank face neighbours, per element type:

    [ owned interior | owned boundary | ghosts from rank s0 | ghosts from s1 | ... ]

(owned boundary = owned elements with an off-rank face neighbour).  Building
it as an ordinary HybridMesh re-derives the face links and orientation codes,
so the device kernels run unchanged on the owned subset; a ghost's faces
towards non-local elements become (unused) boundary faces.  Per stage the
owned boundary states listed in ``send[s][t]`` travel to rank s and land in
the contiguous ghost range ``recv[s][t]`` of the receiver's state arrays,
in global element order on both sides.
"""

from dataclasses import dataclass, field

import numpy as np

from .mesh import HybridMesh
from .refelem import ELEMENT_TYPES

__all__ = ["partition_elements", "LocalPart", "build_local_parts", "TYPE_NAMES"]

TYPE_NAMES = list(ELEMENT_TYPES)            # hex, wedge, pyramid, tet
_COST = {"hex": 1.0, "wedge": 1.6, "pyramid": 1.4, "tet": 1.0}   # per-DOF cost weights


def _centroids(mesh, t):
    return mesh.element_vertices(t).mean(axis=1)


def partition_elements(mesh, nparts, method="rcb", N=3):
    """Rank of every element: dict t -> (K,) int.  'xslab' cuts x into
    equal-width slabs (the structured generators' natural cut); 'rcb' is a
    recursive coordinate bisection weighted by per-type cost x Np."""
    from .basis import basis_dimension
    if nparts == 1:
        return {t: np.zeros(len(mesh.blocks[t]), dtype=np.int64) for t in mesh.elem_types}
    cents = np.vstack([_centroids(mesh, t) for t in mesh.elem_types])
    owners = np.concatenate([np.full(len(mesh.blocks[t]), i)
                             for i, t in enumerate(mesh.elem_types)])
    if method == "xslab":
        lo, hi = mesh.vertices[:, 0].min(), mesh.vertices[:, 0].max()
        rank = np.clip(((cents[:, 0] - lo) / (hi - lo) * nparts).astype(np.int64), 0, nparts - 1)
    elif method == "rcb":
        w = np.concatenate([np.full(len(mesh.blocks[t]),
                                    _COST[t] * basis_dimension(t, N)) for t in mesh.elem_types])
        rank = np.zeros(len(cents), dtype=np.int64)

        def split(idx, r0, nr):
            if nr == 1:
                rank[idx] = r0
                return
            ext = cents[idx].max(axis=0) - cents[idx].min(axis=0)
            ax = int(np.argmax(ext))
            order = idx[np.argsort(cents[idx, ax], kind="stable")]
            left = nr // 2
            cw = np.cumsum(w[order])
            cut = int(np.searchsorted(cw, cw[-1] * left / nr))
            split(order[:cut], r0, left)
            split(order[cut:], r0 + left, nr - left)

        split(np.arange(len(cents)), 0, nparts)
    else:
        raise ValueError(f"unknown partition method {method!r}")
    out, off = {}, 0
    for i, t in enumerate(mesh.elem_types):
        K = len(mesh.blocks[t])
        out[t] = rank[off:off + K]
        off += K
    return out


@dataclass
class LocalPart:
    rank: int
    mesh: HybridMesh
    n_owned: dict                      # t -> owned count
    n_interior: dict                   # t -> owned elements without off-rank neighbours
    global_ids: dict                   # t -> (K_local,) global element index
    send: dict = field(default_factory=dict)   # peer -> t -> local indices (owned), in order
    recv: dict = field(default_factory=dict)   # peer -> t -> (start, stop) local ghost range
    # face-level halo: peer -> t -> (n, 2) (local element, face) pairs, the
    # owned faces a peer's elements touch (send) / the ghost faces my owned
    # elements touch (recv), both in global (element, face) order
    send_faces: dict = field(default_factory=dict)
    recv_faces: dict = field(default_factory=dict)

    @property
    def types(self):
        return self.mesh.elem_types


def build_local_parts(mesh, rank_of, ranks=None):
    """LocalPart objects (host, vectorised) for `ranks` (default: all; the
    others are None — a distributed run builds only its own)."""
    nparts = int(max(int(v.max(initial=0)) for v in rank_of.values())) + 1
    types = mesh.elem_types
    # (type of needed element, element, needing rank) over every cut face,
    # and the same with the needed element's face
    pairs = {t: [] for t in types}
    fpairs = {t: [] for t in types}
    has_off = {t: np.zeros(len(mesh.blocks[t]), dtype=bool) for t in types}
    for t in types:
        nbr = mesh.nbr[t]
        r_me = rank_of[t]
        for f in range(nbr.shape[1]):
            for tid2, t2 in enumerate(ELEMENT_TYPES):
                sel = nbr[:, f, 0] == tid2
                if not sel.any():
                    continue
                k2 = nbr[sel, f, 1]
                f2 = nbr[sel, f, 2]
                rm = r_me[sel]
                diff = rank_of[t2][k2] != rm
                has_off[t][np.flatnonzero(sel)[diff]] = True
                pairs[t2].append(np.column_stack([k2[diff], rm[diff]]))
                fpairs[t2].append(np.column_stack([k2[diff], f2[diff], rm[diff]]))
    need, need_f = {}, {}
    for t in types:
        a = np.vstack(pairs[t]) if pairs[t] else np.zeros((0, 2), dtype=np.int64)
        need[t] = np.unique(a, axis=0)          # rows (element, needing rank), sorted by element
        a = np.vstack(fpairs[t]) if fpairs[t] else np.zeros((0, 3), dtype=np.int64)
        need_f[t] = np.unique(a, axis=0)        # rows (element, face, needing rank)
    parts = []
    for r in range(nparts):
        if ranks is not None and r not in ranks:
            parts.append(None)
            continue
        blocks, mats, gids, n_owned, n_int, glist = {}, {}, {}, {}, {}, {}
        for t in types:
            own = np.flatnonzero(rank_of[t] == r)
            interior = own[~has_off[t][own]]
            boundary = own[has_off[t][own]]
            g = need[t][need[t][:, 1] == r, 0]
            g = g[np.lexsort((g, rank_of[t][g]))]      # by owner rank, then global id
            glist[t] = g
            ids = np.concatenate([interior, boundary, g])
            gids[t] = ids
            blocks[t] = mesh.blocks[t][ids]
            mats[t] = np.asarray(mesh.materials[t])[ids].copy()
            n_owned[t] = len(own)
            n_int[t] = len(interior)
        lm = HybridMesh(mesh.vertices, {t: blocks[t] for t in types if len(blocks[t])},
                        materials={t: mats[t] for t in types if len(blocks[t])})
        part = LocalPart(r, lm, n_owned, n_int, gids)
        for t in types:
            g = glist[t]
            src = rank_of[t][g]
            for sr in np.unique(src):
                idx = np.flatnonzero(src == sr)
                part.recv.setdefault(int(sr), {})[t] = (n_owned[t] + int(idx[0]),
                                                        n_owned[t] + int(idx[-1]) + 1)
        parts.append(part)
    # send lists: owned elements of r needed by s, in global order (matches
    # the receiver's ghost order)
    for r, part in enumerate(parts):
        if part is None:
            continue
        for t in types:
            own_ids = part.global_ids[t][:part.n_owned[t]]
            lookup = np.full(len(mesh.blocks[t]), -1, dtype=np.int64)
            lookup[own_ids] = np.arange(len(own_ids))
            nt = need[t]
            mine = nt[rank_of[t][nt[:, 0]] == r]
            for sr in np.unique(mine[:, 1]):
                ks = np.sort(mine[mine[:, 1] == sr, 0])
                part.send.setdefault(int(sr), {})[t] = lookup[ks]
            # face-level lists: sent (owned element, face) pairs, and the
            # received ghost (element, face) pairs in the same global order
            nf = need_f[t]
            mine = nf[rank_of[t][nf[:, 0]] == r]
            for sr in np.unique(mine[:, 2]):
                rows = mine[mine[:, 2] == sr]
                part.send_faces.setdefault(int(sr), {})[t] = np.column_stack(
                    [lookup[rows[:, 0]], rows[:, 1]])
            theirs = nf[nf[:, 2] == r]
            if len(theirs):
                glookup = np.full(len(mesh.blocks[t]), -1, dtype=np.int64)
                gl = part.global_ids[t]
                glookup[gl[part.n_owned[t]:]] = np.arange(part.n_owned[t], len(gl))
                src = rank_of[t][theirs[:, 0]]
                for sr in np.unique(src):
                    rows = theirs[src == sr]
                    part.recv_faces.setdefault(int(sr), {})[t] = np.column_stack(
                        [glookup[rows[:, 0]], rows[:, 1]])
    return parts
