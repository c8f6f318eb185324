"""Hybrid meshes: typed element blocks, vectorised face connectivity,
structured generators and a GMSH v2.2 reader (host setup).

Element and vertex numbering of the generators reproduce the reference's
(hybridwave/mesh.py:183-340) so states are interchangeable with it; the
construction is vectorised (the reference walks cells in Python and takes
~30 s at n=38; the 2.2M-element hex-dominant mesh of BASELINE config 4 needs
this).  Connectivity is sorted-key matching over all faces at once instead
of a per-face dictionary (mesh.py:121-160).
"""

import itertools
import os

import numpy as np

from .refelem import ELEMENT_TYPES, FACES, N_VERTS, REF_VERTS

__all__ = ["HybridMesh", "FaceLink", "NonconformingMeshError", "GmshParseError",
           "build_connectivity", "uniform_cube_mesh", "hybrid_band_layout",
           "structured_hybrid_mesh", "layered_hybrid_mesh", "hex_dominant_mesh",
           "graded_hybrid_mesh", "read_gmsh", "mesh_volume", "TYPE_IDS"]

TYPE_IDS = {t: i for i, t in enumerate(ELEMENT_TYPES)}   # hex 0, wedge 1, pyramid 2, tet 3

_TRI_PERMS = [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]
_QUAD_PERMS = [(0, 1, 2, 3), (1, 2, 3, 0), (2, 3, 0, 1), (3, 0, 1, 2),
               (0, 3, 2, 1), (3, 2, 1, 0), (2, 1, 0, 3), (1, 0, 3, 2)]


class NonconformingMeshError(ValueError):
    pass


class GmshParseError(ValueError):
    pass


class FaceLink:
    """Connectivity record of one face (hybridwave/mesh.py:57-73):
    neighbor = (type, element, face) or None; orientation = index of the
    vertex permutation p with my_face[p[i]] == neighbor_face[i]."""

    __slots__ = ("neighbor", "orientation")

    def __init__(self, neighbor=None, orientation=0):
        self.neighbor = neighbor
        self.orientation = orientation

    @property
    def is_boundary(self):
        return self.neighbor is None


def _face_vertex_ids(mesh, t):
    conn = mesh.blocks[t]
    return [conn[:, list(ix)] for _, ix in FACES[t]]


def build_connectivity(mesh):
    """Vectorised face matching.

    Returns dict t -> (nbr (K, nf, 3) int64 [type id, element, face] with -1
    on the boundary, code (K, nf) int8 = my orientation code c with
    my_face[i] == nbr_face[PERMS[c][i]], refcode (K, nf) int8 = the
    reference's FaceLink.orientation)."""
    keys, owners, verts_list = [], [], []
    for t in mesh.elem_types:
        for f, fv in enumerate(_face_vertex_ids(mesh, t)):
            K = len(fv)
            k4 = np.full((K, 4), -1, dtype=np.int64)
            k4[:, :fv.shape[1]] = np.sort(fv, axis=1)
            keys.append(k4)
            owners.append(np.column_stack([np.full(K, TYPE_IDS[t]), np.arange(K),
                                           np.full(K, f)]))
            v4 = np.full((K, 4), -1, dtype=np.int64)
            v4[:, :fv.shape[1]] = fv
            verts_list.append(v4)
    out = {t: (np.full((len(mesh.blocks[t]), len(FACES[t]), 3), -1, dtype=np.int64),
               np.zeros((len(mesh.blocks[t]), len(FACES[t])), dtype=np.int8),
               np.zeros((len(mesh.blocks[t]), len(FACES[t])), dtype=np.int8))
           for t in mesh.elem_types}
    if not keys:
        return out
    keys = np.vstack(keys)
    owners = np.vstack(owners)
    fverts = np.vstack(verts_list)
    order = np.lexsort(keys.T[::-1])
    sk = keys[order]
    newgrp = np.ones(len(sk), dtype=bool)
    newgrp[1:] = np.any(sk[1:] != sk[:-1], axis=1)
    gid = np.cumsum(newgrp) - 1
    counts = np.bincount(gid)
    if counts.max() > 2:
        bad = sk[np.flatnonzero(counts[gid] > 2)[0]]
        raise NonconformingMeshError(
            f"face {tuple(int(v) for v in bad if v >= 0)} shared by {counts.max()} elements")
    first = np.flatnonzero(newgrp)
    pair = first[counts[gid[first]] == 2]
    ia, ib = order[pair], order[pair + 1]
    va, vb = fverts[ia], fverts[ib]
    na, nb = (va >= 0).sum(1), (vb >= 0).sum(1)
    if np.any(na != nb):
        raise NonconformingMeshError("face links a triangle to a quadrilateral")
    codes_ab = np.full(len(ia), -1)     # mine: va[i] == vb[P[c][i]]
    codes_ba = np.full(len(ia), -1)
    ref_ab = np.full(len(ia), -1)       # reference: va[P[c][i]] == vb[i]
    ref_ba = np.full(len(ia), -1)
    for nvf, perms in ((3, _TRI_PERMS), (4, _QUAD_PERMS)):
        sel = na == nvf
        if not sel.any():
            continue
        A, B = va[sel][:, :nvf], vb[sel][:, :nvf]
        for c, p in enumerate(perms):
            p = list(p)
            for arr, X, Y in ((codes_ab, A, B[:, p]), (codes_ba, B, A[:, p]),
                              (ref_ab, A[:, p], B), (ref_ba, B[:, p], A)):
                hit = np.all(X == Y, axis=1)
                idx = np.flatnonzero(sel)[hit]
                arr[idx] = np.where(arr[idx] < 0, c, arr[idx])
    if np.any(codes_ab < 0) or np.any(codes_ba < 0):
        raise NonconformingMeshError("faces are not related by a dihedral map")
    oa, ob = owners[ia], owners[ib]
    for (src, dst, code, rcode) in ((oa, ob, codes_ab, ref_ab), (ob, oa, codes_ba, ref_ba)):
        for tid, t in enumerate(ELEMENT_TYPES):
            if t not in out:
                continue
            m = src[:, 0] == tid
            nbr, cd, rc = out[t]
            nbr[src[m, 1], src[m, 2]] = dst[m]
            cd[src[m, 1], src[m, 2]] = code[m]
            rc[src[m, 1], src[m, 2]] = rcode[m]
    return out


class HybridMesh:
    """Vertices, typed element blocks, materials (rho, kappa) and face
    connectivity (hybridwave/mesh.py:76-115).  ``nbr``/``face_code`` hold the
    connectivity as arrays; ``face_links`` builds the reference's per-face
    FaceLink objects on first use."""

    def __init__(self, vertices, blocks, materials=None, physical=None):
        self.vertices = np.asarray(vertices, dtype=float)
        self.blocks = {t: np.asarray(v, dtype=np.int64).reshape(-1, N_VERTS[t])
                       for t, v in blocks.items() if len(v)}
        if materials is None:
            materials = {t: np.ones((len(v), 2)) for t, v in self.blocks.items()}
        self.materials = materials
        self.physical = physical or {}
        conn = build_connectivity(self)
        self.nbr = {t: c[0] for t, c in conn.items()}
        self.face_code = {t: c[1] for t, c in conn.items()}
        self._ref_code = {t: c[2] for t, c in conn.items()}
        self._links = None

    @property
    def elem_types(self):
        return [t for t in ELEMENT_TYPES if t in self.blocks]

    @property
    def n_elements(self):
        return sum(len(v) for v in self.blocks.values())

    def element_vertices(self, elem_type):
        return self.vertices[self.blocks[elem_type]]

    @property
    def face_links(self):
        if self._links is None:
            links = {}
            for t in self.elem_types:
                nb, rc = self.nbr[t], self._ref_code[t]
                rows = []
                for k in range(len(nb)):
                    row = []
                    for f in range(nb.shape[1]):
                        if nb[k, f, 0] < 0:
                            row.append(FaceLink())
                        else:
                            row.append(FaceLink((ELEMENT_TYPES[nb[k, f, 0]], int(nb[k, f, 1]),
                                                 int(nb[k, f, 2])), int(rc[k, f])))
                    rows.append(row)
                links[t] = rows
            self._links = links
        return self._links

    def set_materials(self, table):
        for t in self.blocks:
            groups = self.physical.get(t)
            if groups is None:
                continue
            for k, g in enumerate(groups):
                if g in table:
                    self.materials[t][k] = table[g]


# ---------------------------------------------------------------- generators

def _kuhn_local():
    """Local corner indices (hex order) of the 6 Kuhn tets of a cell, in the
    reference's permutation order, positively oriented on an axis-aligned
    cell (hybridwave/mesh.py:217-239)."""
    remap = {0: 0, 1: 1, 3: 2, 2: 3, 4: 4, 5: 5, 7: 6, 6: 7}
    cube = REF_VERTS["hex"]
    out = []
    for perm in itertools.permutations(range(3)):
        p = np.zeros(3)
        ids = [0]
        for d in perm:
            p = p.copy()
            p[d] = 1
            ids.append(int(p[0]) + 2 * int(p[1]) + 4 * int(p[2]))
        tet = [remap[i] for i in ids]
        v = cube[tet]
        if np.linalg.det(np.column_stack([v[1] - v[0], v[2] - v[0], v[3] - v[0]])) < 0:
            tet[2], tet[3] = tet[3], tet[2]
        out.append(tet)
    return np.array(out)


_WEDGE_LOCAL = np.array([[0, 7, 3, 1, 6, 2], [0, 4, 7, 1, 5, 6]])


def _orient_tets(conn, X):
    v = X[conn]
    det = np.linalg.det(np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0],
                                  v[:, 3] - v[:, 0]], axis=2))
    conn = conn.copy()
    neg = det < 0
    conn[neg, 2], conn[neg, 3] = conn[neg, 3].copy(), conn[neg, 2].copy()
    return conn


def layered_hybrid_mesh(n, kinds, zs=None, nx=None):
    """Box mesh of nx x n cells per z-layer (unit cube when nx = n; for
    nx = m n the box is [0, m] x [0, 1] x [0, 1] with the same cell size, the
    weak-scaling extension of the reference's cube); kinds[k] in {"hex",
    "wedge", "pyrtop", "pyr", "tet"} selects the cell decomposition of layer
    k ("pyrtop" = 5 pyramids + the top pyramid split into 2 tets, the
    reference's transition layer; "pyr" = 6 pyramids).  Vertex and element
    numbering follow the reference's cell walk (k outer, then j, then i)."""
    nz = len(kinds)
    zs = np.linspace(0.0, 1.0, nz + 1) if zs is None else np.asarray(zs, dtype=float)
    nx = n if nx is None else int(nx)
    xs = np.linspace(0.0, nx / n, nx + 1)
    ys = np.linspace(0.0, 1.0, n + 1)
    gx, gy, gz = np.meshgrid(xs, ys, zs, indexing="ij")
    # pool order: z outer, y, x inner
    grid = np.column_stack([gx.transpose(2, 1, 0).ravel(), gy.transpose(2, 1, 0).ravel(),
                            gz.transpose(2, 1, 0).ravel()])
    nv = len(grid)

    def vid(i, j, k):
        return (k * (n + 1) + j) * (nx + 1) + i

    jj, ii = np.meshgrid(np.arange(n), np.arange(nx), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()                 # cell order within a layer: j outer, i inner
    blocks = {t: [] for t in ELEMENT_TYPES}
    extra = []
    kuhn = _kuhn_local()
    hexf = FACES["hex"]
    for k, kind in enumerate(kinds):
        kk = np.full_like(ii, k)
        c = np.column_stack([vid(ii, jj, kk), vid(ii + 1, jj, kk), vid(ii + 1, jj + 1, kk),
                             vid(ii, jj + 1, kk), vid(ii, jj, kk + 1), vid(ii + 1, jj, kk + 1),
                             vid(ii + 1, jj + 1, kk + 1), vid(ii, jj + 1, kk + 1)])
        if kind == "hex":
            blocks["hex"].append(c)
        elif kind == "wedge":
            blocks["wedge"].append(c[:, _WEDGE_LOCAL].reshape(-1, 6))
        elif kind == "tet":
            blocks["tet"].append(c[:, kuhn].reshape(-1, 4))
        elif kind in ("pyr", "pyrtop"):
            cx = grid[c].mean(axis=1)
            apex = nv + sum(len(e) for e in extra) + np.arange(len(c))
            extra.append(cx)
            pyrs, tets = [], []
            for f, (_, ix) in enumerate(hexf):
                base_in = c[:, list(ix)][:, ::-1]
                if kind == "pyrtop" and f == 5:
                    a, b, cc, d = base_in.T
                    tets = [np.column_stack([a, b, d, apex]), np.column_stack([b, cc, d, apex])]
                else:
                    pyrs.append(np.column_stack([base_in, apex]))
            blocks["pyramid"].append(np.stack(pyrs, axis=1).reshape(-1, 5))
            if tets:
                X = np.vstack([grid] + extra)
                t2 = np.stack([_orient_tets(tt, X) for tt in tets], axis=1).reshape(-1, 4)
                blocks["tet"].append(t2)
        else:
            raise ValueError(f"unknown layer kind {kind!r}")
    X = np.vstack([grid] + extra)
    return HybridMesh(X, {t: np.vstack(v) for t, v in blocks.items() if v})


def uniform_cube_mesh(elem_type, n):
    """n^3 hexes, 2n^3 wedges, 6n^3 pyramids or 6n^3 Kuhn tets on the unit
    cube (hybridwave/mesh.py:272-297)."""
    if n < 1:
        raise ValueError("need at least one cell per axis")
    kind = {"hex": "hex", "wedge": "wedge", "pyramid": "pyr", "tet": "tet"}.get(elem_type)
    if kind is None:
        raise ValueError(f"unknown element type {elem_type!r}")
    return layered_hybrid_mesh(n, [kind] * n)


def hybrid_band_layout(n):
    """(hex, wedge, pyramid, tet) layer counts (hybridwave/mesh.py:300-307)."""
    nz = max(n, 4)
    t_l = max(1, nz // 2 - 1)
    w_l = max(1, (nz - t_l - 1) // 2)
    return nz - t_l - 1 - w_l, w_l, 1, t_l


def structured_hybrid_mesh(n, nx=None):
    """The reference's hybrid cube: hex slab, wedge slab, one pyramid
    transition layer, Kuhn tets (hybridwave/mesh.py:310-340).  nx > n
    extends the box along x with the same cells (weak scaling)."""
    if n < 2:
        raise ValueError("hybrid cube needs n >= 2")
    h, w, p, t = hybrid_band_layout(n)
    return layered_hybrid_mesh(n, ["hex"] * h + ["wedge"] * w + ["pyrtop"] * p + ["tet"] * t,
                               nx=nx)


def hex_dominant_mesh(n, layers=(110, 4, 1, 5)):
    """BASELINE config 4 (not in the reference): the same bands with a
    hex-dominant layer split; n=120 with layers (110, 4, 1, 5) gives
    1,584,000 hex / 115,200 wedge / 72,000 pyramid / 460,800 tet."""
    h, w, p, t = layers
    return layered_hybrid_mesh(n, ["hex"] * h + ["wedge"] * w + ["pyrtop"] * p + ["tet"] * t)


def graded_hybrid_mesh(n, layers=None, ratio=0.5, nx=None):
    """BASELINE config 5 (not in the reference): the reference's band
    layout with geometrically graded z-spacing, finest in the pyramid/tet
    refinement zone, so local timesteps span several MRAB levels."""
    h, w, p, t = layers or hybrid_band_layout(n)
    nz = h + w + p + t
    # spacing shrinks by `ratio` across the hex/wedge bands towards the tets
    s = np.ones(nz)
    s[:h] = 4.0
    s[h:h + w] = 2.0
    s[h + w:] = 1.0
    s = s ** (np.log(1 / ratio) / np.log(2.0))
    zs = np.concatenate([[0.0], np.cumsum(s)]) / s.sum()
    return layered_hybrid_mesh(n, ["hex"] * h + ["wedge"] * w + ["pyrtop"] * p + ["tet"] * t,
                               zs=zs, nx=nx)


# ---------------------------------------------------------------- GMSH

# msh 2.2 element code -> (type, vertex count); lower-dimensional codes that a
# volume mesh may carry (line, triangle, quad, point) are skipped
_MSH_VOLUME = {4: ("tet", 4), 5: ("hex", 8), 6: ("wedge", 6), 7: ("pyramid", 5)}
_MSH_SKIPPED = frozenset((1, 2, 3, 15))
# gmsh's prism runs its triangle the other way round from our (r, t)
# triangle: reversing corners 1 <-> 2 on both triangles keeps J > 0
_MSH_PRISM_ORDER = np.array([0, 2, 1, 3, 5, 4])


class _MshCursor:
    """Line cursor over a .msh file; every error names the 1-based line."""

    def __init__(self, path):
        self.path = path
        with open(path) as fh:
            self.rows = fh.read().splitlines()
        self.i = 0

    def error(self, what):
        return GmshParseError(f"{self.path}:{self.i + 1}: {what}")

    def marker(self, name):
        while self.i < len(self.rows) and not self.rows[self.i].strip():
            self.i += 1
        if self.i >= len(self.rows) or self.rows[self.i].strip() != name:
            raise self.error(f"expected {name}")
        self.i += 1

    def fields(self, what, min_len=1):
        if self.i >= len(self.rows):
            raise self.error(what)
        f = self.rows[self.i].split()
        if len(f) < min_len or f[0].startswith("$"):
            raise self.error(what)
        self.i += 1
        return f

    def count(self, what):
        try:
            return int(self.fields(what)[0])
        except ValueError:
            self.i -= 1
            raise self.error(what) from None


def read_gmsh(path):
    """Linear volume mesh from a GMSH 2.2 ASCII file (reference interface:
    hybridwave/mesh.py:359-442).  Element codes 4/5/6/7 become tet, hex,
    wedge, pyramid blocks (prism corners reordered to our orientation);
    the first element tag is kept as the physical group; lines, triangles,
    quads and points are ignored; anything else raises GmshParseError with
    the offending line number."""
    cur = _MshCursor(path)
    cur.marker("$MeshFormat")
    version = cur.fields("only msh format 2.2 is supported")[0]
    if not version.startswith("2.2"):
        cur.i -= 1
        raise cur.error("only msh format 2.2 is supported")
    cur.marker("$EndMeshFormat")

    cur.marker("$Nodes")
    n_nodes = cur.count("bad node count")
    tags = np.empty(n_nodes, dtype=np.int64)
    xyz = np.empty((n_nodes, 3))
    for r in range(n_nodes):
        f = cur.fields("truncated $Nodes section" if cur.i >= len(cur.rows)
                       else "bad node line", 4)
        tags[r] = int(f[0])
        xyz[r] = f[1:4]
    cur.marker("$EndNodes")
    row_of = dict(zip(tags.tolist(), range(n_nodes)))

    cur.marker("$Elements")
    n_items = cur.count("bad element count")
    conn = {t: [] for t in ELEMENT_TYPES}
    group = {t: [] for t in ELEMENT_TYPES}
    for _ in range(n_items):
        f = cur.fields("truncated $Elements section", 1)
        if len(f) < 3:
            cur.i -= 1
            raise cur.error("bad element line")
        code, ntag = int(f[1]), int(f[2])
        if code in _MSH_SKIPPED:
            continue
        if code not in _MSH_VOLUME:
            cur.i -= 1
            raise cur.error(f"unsupported element code {code}")
        kind, nv = _MSH_VOLUME[code]
        verts = f[3 + ntag:]
        if len(verts) != nv:
            cur.i -= 1
            raise cur.error(f"{kind} element needs {nv} nodes, got {len(verts)}")
        missing = [v for v in verts if int(v) not in row_of]
        if missing:
            cur.i -= 1
            raise cur.error(f"unknown node id {missing[0]}")
        row = np.array([row_of[int(v)] for v in verts])
        conn[kind].append(row[_MSH_PRISM_ORDER] if kind == "wedge" else row)
        group[kind].append(int(f[3]) if ntag else 0)
    cur.marker("$EndElements")
    present = [t for t in ELEMENT_TYPES if conn[t]]
    return HybridMesh(xyz, {t: np.array(conn[t]) for t in present},
                      physical={t: np.array(group[t]) for t in present})


def mesh_volume(mesh, N=2):
    """Total volume as the sum over types of w . J at an exact-degree
    element rule (the reference's mesh check, hybridwave/mesh.py:449-459)."""
    from .quadrature import element_rule
    from .refelem import jacobian_det_fast
    vol = {}
    for t in mesh.elem_types:
        rule = element_rule(t, N)
        vol[t] = jacobian_det_fast(t, mesh.element_vertices(t), rule.collapsed) @ rule.weights
    return float(sum(v.sum() for v in vol.values()))


def wedge_tet_columns_mesh(nx=4, ny=2, nz=2):
    """Test mesh (not in the reference): nx x ny x nz cells of the unit box
    whose x-columns alternate between wedge pairs and Kuhn tets, so wedge
    triangle faces meet tet faces (the wedge triangles lie on the cells'
    x-faces and their diagonals match the Kuhn split).  Jittering the
    interior vertices makes those wedges non-affine."""
    xs, ys, zs = (np.linspace(0.0, 1.0, n + 1) for n in (nx, ny, nz))
    gx, gy, gz = np.meshgrid(xs, ys, zs, indexing="ij")
    X = np.column_stack([gx.transpose(2, 1, 0).ravel(), gy.transpose(2, 1, 0).ravel(),
                         gz.transpose(2, 1, 0).ravel()])

    def vid(i, j, k):
        return (k * (ny + 1) + j) * (nx + 1) + i

    wed, tet = [], []
    kuhn = _kuhn_local()
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                c = np.array([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k),
                              vid(i, j + 1, k), vid(i, j, k + 1), vid(i + 1, j, k + 1),
                              vid(i + 1, j + 1, k + 1), vid(i, j + 1, k + 1)])
                if i % 2 == 0:
                    wed.append(c[_WEDGE_LOCAL].reshape(-1, 6))
                else:
                    tet.append(_orient_tets(c[kuhn].reshape(-1, 4), X))
    return HybridMesh(X, {"wedge": np.vstack(wed), "tet": np.vstack(tet)})


def _orient_wedges(conn, X):
    """Wedges (two triangles, corresponding corners) in the orientation of
    _WEDGE_LOCAL's: flip both triangles where the sign differs."""
    def sign(c):
        v = X[c]
        return np.sign(np.einsum("ij,ij->i", np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]),
                                 v[:, 3] - v[:, 0]))
    ref = REF_VERTS["hex"][_WEDGE_LOCAL[0]]
    want = np.sign(np.dot(np.cross(ref[1] - ref[0], ref[2] - ref[0]), ref[3] - ref[0]))
    conn = conn.copy()
    bad = sign(conn) != want
    conn[bad] = conn[bad][:, [0, 2, 1, 3, 5, 4]]
    return conn


def wedge_pyramid_columns_mesh(ny=2, jitter=0.0, seed=0):
    """Test mesh (not in the reference): ny rows of four cells along x,
    [pyramids | wedges | wedges | pyramids], one cell thick in z.  A
    pyramid cell is the cube split into 3 pyramids with a common apex at a
    corner on its wedge-side x-face, whose two triangles then meet the
    wedge pair's triangles (the wedge diagonal goes through the apex corner;
    rows alternate the apex's y side so the pyramid cells stay conforming).
    jitter > 0 moves the vertices of the middle x-plane (shared by wedges
    only): the wedges become non-affine, the pyramids stay affine."""
    nx, nz = 4, 1
    xs, ys, zs = np.linspace(0.0, 1.0, nx + 1), np.linspace(0.0, 1.0, ny + 1), np.array([0.0, 1.0 / ny])
    gx, gy, gz = np.meshgrid(xs, ys, zs, indexing="ij")
    X = np.column_stack([gx.transpose(2, 1, 0).ravel(), gy.transpose(2, 1, 0).ravel(),
                         gz.transpose(2, 1, 0).ravel()])

    def vid(i, j, k):
        return (k * (ny + 1) + j) * (nx + 1) + i

    hexf = FACES["hex"]
    wed, pyr = [], []
    for j in range(ny):
        low = j % 2 == 0                 # apex (and wedge diagonal) on the row's low-y side
        for i in range(nx):
            c = np.array([vid(i, j, 0), vid(i + 1, j, 0), vid(i + 1, j + 1, 0),
                          vid(i, j + 1, 0), vid(i, j, 1), vid(i + 1, j, 1),
                          vid(i + 1, j + 1, 1), vid(i, j + 1, 1)])
            if i in (1, 2):
                # x-face diagonal (y_a, z0)-(y_b, z1): through local 0-7 (low) or 3-4
                loc = _WEDGE_LOCAL if low else np.array([[3, 4, 0, 2, 5, 1], [3, 7, 4, 2, 6, 5]])
                wed.append(c[loc])
            else:
                # apex corner: on the x-face towards the wedges, at z0 and the row's y side
                xi = 1 if i == 0 else 0
                apex_local = {(0, True): 0, (1, True): 1, (0, False): 3, (1, False): 2}[(xi, low)]
                for f, (_, ix) in enumerate(hexf):
                    if apex_local in ix:
                        continue
                    pyr.append(np.concatenate([c[list(ix)][::-1], [c[apex_local]]]))
    wed = _orient_wedges(np.vstack(wed), X)
    if jitter > 0:
        rng = np.random.default_rng(seed)
        mid = np.abs(X[:, 0] - xs[2]) < 1e-12
        X = X.copy()
        X[mid] += jitter / nx * rng.uniform(-1, 1, (int(mid.sum()), 3)) * np.array([1.0, 0.0, 0.0])
    return HybridMesh(X, {"wedge": wed, "pyramid": np.array(pyr)})
