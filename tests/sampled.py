"""TEST INFRASTRUCTURE: oracle RHS on a sampled sub-mesh.

The RHS of an element depends only on its own state, geometry and material
and on its face neighbours' states and materials (hybridwave/dg.py:299-354:
traces, the mapP gather, the flux with avg(rho c)).  So the oracle RHS of a
sample S of a large mesh is exact when computed on the sub-mesh S ∪ N(S)
(N = face neighbours) — rows of S only; the rows of N(S) see artificial
boundary faces and are discarded.  This makes full-size parity (hybrid:38,
hexdom:120) affordable on the host.
"""

import numpy as np

from paper_1507_02557_b200.mesh import HybridMesh, TYPE_IDS


def default_sample(mesh, n_random=192, n_edge=48, seed=0):
    """Per type: the first and last n_edge elements (block boundaries, the
    largest offsets) and n_random random ones."""
    rng = np.random.default_rng(seed)
    out = {}
    for t in mesh.elem_types:
        K = len(mesh.blocks[t])
        ids = np.concatenate([np.arange(min(n_edge, K)), np.arange(max(0, K - n_edge), K),
                              rng.choice(K, size=min(n_random, K), replace=False)])
        out[t] = np.unique(ids)
    return out


def neighbour_closure(mesh, sample):
    keep = {t: set(np.asarray(sample.get(t, []), dtype=np.int64).tolist())
            for t in mesh.elem_types}
    for t, ids in sample.items():
        nb = mesh.nbr[t][np.asarray(ids, dtype=np.int64)]          # (n, nf, 3)
        for t2 in mesh.elem_types:
            sel = nb[:, :, 0] == TYPE_IDS[t2]
            keep[t2].update(nb[:, :, 1][sel].tolist())
    return {t: np.array(sorted(v), dtype=np.int64) for t, v in keep.items() if v}


def submesh(mesh, keep):
    blocks = {t: mesh.blocks[t][ids] for t, ids in keep.items()}
    mats = {t: np.array(mesh.materials[t][ids], copy=True) for t, ids in keep.items()}
    return HybridMesh(mesh.vertices, blocks, materials=mats)


def sampled_oracle_rhs(disc, state_rows, sample, **disc_kw):
    """Oracle RHS rows of ``sample`` (dict t -> element ids) of ``disc``'s
    mesh.  ``state_rows(t, ids) -> (len(ids), 4, Np)`` fp64 host array.
    Returns dict t -> (len(sample[t]), 4, Np)."""
    import oracle
    from paper_1507_02557_b200.dg import Discretization
    keep = neighbour_closure(disc.mesh, sample)
    sub = submesh(disc.mesh, keep)
    d = Discretization(sub, disc.N, disc.formulation.kind, forms_override=disc.forms,
                       penalty_scale=disc.penalty_scale, device="cpu", **disc_kw)
    st = {t: state_rows(t, keep[t]) for t in sub.elem_types}
    r = oracle.compute_rhs(d, st)
    out = {}
    for t, ids in sample.items():
        pos = np.searchsorted(keep[t], ids)
        out[t] = r[t][pos]
    return out
