"""Synthetic FEM matrices of the shapes BASELINE.json names (host-side input
synthesis only; the SpMV / CG under test never runs here).

All meshes are the reference's structured tetrahedral box
(fem/mesh.cpp:33-71): (nx+1)(ny+1)(nz+1) nodes numbered
(k*(ny+1)+j)*(nx+1)+i, each cell split into six tetrahedra around its main
diagonal (Freudenthal). P1 elements couple every node with itself and the
14 neighbours at offsets +-x, +-y, +-z, +-(x+y), +-(y+z), +-(x+z),
+-(x+y+z): a 15-point stencil, 5..15 entries per row on the box.

* ``laplacian_box``   -- config 1: P1 stiffness (element_geometry gradients,
  fem/element.cpp:7-47) + sigma * lumped mass; SPD. box(63,63,63) gives
  262,144 rows and 3,834,622 nonzeros.
* ``elasticity_box``  -- config 2: 3-DOF linear elasticity (E, nu), 3x3
  blocks on the same stencil + sigma * lumped mass; SPD.
* ``ventricle_box``   -- config 4: config-1 operator on a mesh whose nodes
  are jittered (per-element geometry) and whose unknowns are renumbered by a
  seeded random permutation.

Every generator returns (nrows, ncols, row_offsets[int64], col_indices[int64],
values[float64]) with strictly increasing columns per row (canonical CSR).
"""
from __future__ import annotations

import numpy as np

# Freudenthal split (fem/mesh.cpp:52-71): corner walks of the six tetrahedra
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def _tet_corners():
    """Per tetrahedron, its 4 corner offsets (di, dj, dk) in the cell."""
    tets = []
    for perm in _PERMS:
        at = [0, 0, 0]
        corners = [tuple(at)]
        for s in range(3):
            at[perm[s]] += 1
            corners.append(tuple(at))
        tets.append(corners)
    return tets


_STENCIL = sorted({(a[0] - b[0], a[1] - b[1], a[2] - b[2])
                   for t in _tet_corners() for a in t for b in t})
assert len(_STENCIL) == 15


def _p1_gradients(xyz):
    """P1 shape-function gradients and volumes for tets given as (..., 4, 3)
    coordinates (element_geometry, fem/element.cpp:7-47)."""
    e = xyz[..., 1:, :] - xyz[..., :1, :]  # rows: edge vectors from node 0
    det = np.linalg.det(e)
    inv = np.linalg.inv(e)  # columns: d xi / d x ... grad N_{1..3} are columns of inv^T rows
    g123 = np.swapaxes(inv, -1, -2)  # (..., 3 nodes, 3 coords)
    g0 = -g123.sum(axis=-2, keepdims=True)
    grads = np.concatenate([g0, g123], axis=-2)
    return grads, np.abs(det) / 6.0


def _stencil_csr(nx, ny, nz, block, accumulate):
    """CSR over the 15-point stencil with `block` x `block` node couplings.
    accumulate(dense) fills dense[node, stencil_dir, a, b]."""
    n1, n2, n3 = nx + 1, ny + 1, nz + 1
    nn = n1 * n2 * n3
    dense = np.zeros((nn, len(_STENCIL), block, block), np.float64)
    accumulate(dense)
    ii, jj, kk = np.meshgrid(np.arange(n1), np.arange(n2), np.arange(n3), indexing="ij")
    ii, jj, kk = (a.transpose(2, 1, 0).ravel() for a in (ii, jj, kk))  # node order k, j, i
    present = np.zeros((nn, len(_STENCIL)), bool)
    offs = np.zeros(len(_STENCIL), np.int64)
    for d, (di, dj, dk) in enumerate(_STENCIL):
        present[:, d] = ((ii + di >= 0) & (ii + di < n1) & (jj + dj >= 0) & (jj + dj < n2)
                         & (kk + dk >= 0) & (kk + dk < n3))
        offs[d] = (dk * n2 + dj) * n1 + di
    order = np.argsort(offs, kind="stable")  # ascending column within a node row
    present, offs, dense = present[:, order], offs[order], dense[:, order]
    node = np.arange(nn, dtype=np.int64)
    # rows are (node, a); columns (node + off) * block + b, ascending per row
    cnt_node = present.sum(axis=1) * block
    row_len = np.repeat(cnt_node, block)
    ro = np.zeros(nn * block + 1, np.int64)
    np.cumsum(row_len, out=ro[1:])
    cols = ((node[:, None] + offs[None, :])[:, :, None] * block + np.arange(block)[None, None, :])
    cols = np.broadcast_to(cols[:, None, :, :], (nn, block, len(_STENCIL), block))
    vals = np.transpose(dense, (0, 2, 1, 3))  # (node, a, dir, b)
    mask = np.broadcast_to(present[:, None, :, None], (nn, block, len(_STENCIL), block))
    ci = cols[mask].astype(np.int64)
    v = vals[mask].astype(np.float64)
    return nn * block, nn * block, ro, ci, v


def _cells(nx, ny, nz):
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    return (a.transpose(2, 1, 0).ravel() for a in (ci, cj, ck))


def _node_id(i, j, k, nx, ny):
    return (k * (ny + 1) + j) * (nx + 1) + i


def _dir_index(d):
    return _STENCIL.index(d)


def laplacian_box(nx=63, ny=63, nz=63, sigma=1e-3):
    """Config 1: P1 Laplacian stiffness + sigma * lumped mass, unit cells."""
    tets = _tet_corners()

    def acc(dense):
        ci, cj, ck = _cells(nx, ny, nz)
        base = _node_id(ci, cj, ck, nx, ny)
        for corners in tets:
            xyz = np.array(corners, np.float64)
            g, vol = _p1_gradients(xyz)
            ke = vol * g @ g.T
            for a in range(4):
                na = base + _node_id(*corners[a], nx, ny)
                for b in range(4):
                    d = _dir_index(tuple(np.subtract(corners[b], corners[a])))
                    val = ke[a, b] + (sigma * vol / 4.0 if a == b else 0.0)
                    # for a fixed corner every cell maps to a distinct node, so
                    # a plain fancy-index add has no repeated indices
                    dense[na, d, 0, 0] += val

    return _stencil_csr(nx, ny, nz, 1, acc)


def _elastic_d(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2 * mu
    D[np.arange(3, 6), np.arange(3, 6)] = mu
    return D


def _strain_b(g):
    """6 x 12 strain-displacement matrix of a P1 tet (Voigt xx,yy,zz,xy,yz,xz)."""
    B = np.zeros((6, 12))
    for a in range(4):
        gx, gy, gz = g[a]
        c = 3 * a
        B[0, c] = gx
        B[1, c + 1] = gy
        B[2, c + 2] = gz
        B[3, c], B[3, c + 1] = gy, gx
        B[4, c + 1], B[4, c + 2] = gz, gy
        B[5, c], B[5, c + 2] = gz, gx
    return B


def elasticity_box(nx=86, ny=86, nz=86, E=1.0, nu=0.3, sigma=1e-3):
    """Config 2: 3-DOF linear elasticity + sigma * lumped mass (SPD)."""
    tets = _tet_corners()
    D = _elastic_d(E, nu)

    def acc(dense):
        ci, cj, ck = _cells(nx, ny, nz)
        base = _node_id(ci, cj, ck, nx, ny)
        for corners in tets:
            xyz = np.array(corners, np.float64)
            g, vol = _p1_gradients(xyz)
            B = _strain_b(g)
            ke = vol * B.T @ D @ B
            for a in range(4):
                na = base + _node_id(*corners[a], nx, ny)
                for b in range(4):
                    d = _dir_index(tuple(np.subtract(corners[b], corners[a])))
                    blk = ke[3 * a:3 * a + 3, 3 * b:3 * b + 3].copy()
                    if a == b:
                        blk[np.arange(3), np.arange(3)] += sigma * vol / 4.0
                    dense[na, d] += blk

    return _stencil_csr(nx, ny, nz, 3, acc)


def _element_matrix(kind, corners, E=1.0, nu=0.3, sigma=1e-3):
    """Element matrix (4b x 4b) of a unit-cell tet incl. the lumped mass shift."""
    g, vol = _p1_gradients(np.array(corners, np.float64))
    if kind == "laplacian":
        ke = vol * g @ g.T
        ke[np.arange(4), np.arange(4)] += sigma * vol / 4.0
        return ke
    B = _strain_b(g)
    ke = vol * B.T @ _elastic_d(E, nu) @ B
    ke[np.arange(12), np.arange(12)] += sigma * vol / 4.0
    return ke


def box_rows(kind, nx, ny, nz, k0=0, k1=None, **kw):
    """Rows of the node layers [k0, k1) of the `kind` ("laplacian" or
    "elasticity") operator on box(nx, ny, nz), with GLOBAL column ids: the row
    block one rank of the partitioned solver owns (slab partition along z).
    Returns (row_begin, nrows_global, ro, ci, v); box_rows(kind, ..., 0,
    nz + 1) equals laplacian_box / elasticity_box."""
    k1 = nz + 1 if k1 is None else k1
    blk = 1 if kind == "laplacian" else 3
    n1, n2, n3 = nx + 1, ny + 1, nz + 1
    nzw = k1 - k0
    ns = len(_STENCIL)
    dense = np.zeros((nzw, n2, n1, ns, blk, blk), np.float64)
    for corners in _tet_corners():
        ke = _element_matrix(kind, corners, **kw)
        for a, ca in enumerate(corners):
            lo, hi = max(k0 - ca[2], 0), min(k1 - ca[2], nz)  # cell layers whose corner a is in the window
            if lo >= hi:
                continue
            tgt = dense[lo + ca[2] - k0:hi + ca[2] - k0, ca[1]:ny + ca[1], ca[0]:nx + ca[0]]
            for b, cb in enumerate(corners):
                d = _dir_index(tuple(np.subtract(cb, ca)))
                tgt[..., d, :, :] += ke[blk * a:blk * (a + 1), blk * b:blk * (b + 1)]
    nn = nzw * n2 * n1
    dense = dense.reshape(nn, ns, blk, blk)
    kk, jj, ii = np.meshgrid(np.arange(k0, k1), np.arange(n2), np.arange(n1), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    present = np.zeros((nn, ns), bool)
    offs = np.zeros(ns, np.int64)
    for d, (di, dj, dk) in enumerate(_STENCIL):
        present[:, d] = ((ii + di >= 0) & (ii + di < n1) & (jj + dj >= 0) & (jj + dj < n2)
                         & (kk + dk >= 0) & (kk + dk < n3))
        offs[d] = (dk * n2 + dj) * n1 + di
    order = np.argsort(offs, kind="stable")
    present, offs, dense = present[:, order], offs[order], dense[:, order]
    node = k0 * n2 * n1 + np.arange(nn, dtype=np.int64)
    ro = np.zeros(nn * blk + 1, np.int64)
    np.cumsum(np.repeat(present.sum(axis=1) * blk, blk), out=ro[1:])
    cols = (node[:, None] + offs[None, :])[:, :, None] * blk + np.arange(blk)[None, None, :]
    cols = np.broadcast_to(cols[:, None, :, :], (nn, blk, ns, blk))
    mask = np.broadcast_to(present[:, None, :, None], (nn, blk, ns, blk))
    ci = cols[mask].astype(np.int64)
    v = np.transpose(dense, (0, 2, 1, 3))[mask].astype(np.float64)
    return k0 * n2 * n1 * blk, n1 * n2 * n3 * blk, ro, ci, v


def _slab_row_lengths(kind, nx, ny, nz, k0, k1):
    """Row lengths of node layers [k0, k1) (stencil presence only; cheap)."""
    blk = 1 if kind == "laplacian" else 3
    n1, n2, n3 = nx + 1, ny + 1, nz + 1
    kk, jj, ii = np.meshgrid(np.arange(k0, k1), np.arange(n2), np.arange(n1), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    cnt = np.zeros(ii.size, np.int64)
    for di, dj, dk in _STENCIL:
        cnt += ((ii + di >= 0) & (ii + di < n1) & (jj + dj >= 0) & (jj + dj < n2)
                & (kk + dk >= 0) & (kk + dk < n3))
    return np.repeat(cnt * blk, blk)


def box_csr_slabbed(kind, nx, ny, nz, nslabs=16, workers=1, **kw):
    """The whole box operator built slab by slab straight into its final
    arrays (row offsets from the stencil presence first, then each slab's
    columns and values, `workers` slabs at a time on threads): for the
    100M-row config 5 on one GPU, without holding a second copy. Equals
    elasticity_box / laplacian_box."""
    _, n, ro, ci, v = box_rows_slabbed(kind, nx, ny, nz, 0, nz + 1, nslabs=nslabs, workers=workers, **kw)
    return n, n, ro, ci, v


def box_rows_slabbed(kind, nx, ny, nz, k0=0, k1=None, nslabs=None, workers=8, **kw):
    """box_rows(kind, nx, ny, nz, k0, k1) built `nslabs` node-layer slabs at a
    time straight into the final arrays (`workers` slabs concurrently on
    threads): a partitioned solver's row block of config 5 without the
    dense per-stencil staging of the whole block. Returns (row_begin,
    nrows_global, ro, ci, v) with global column ids, equal to box_rows."""
    blk = 1 if kind == "laplacian" else 3
    k1 = nz + 1 if k1 is None else k1
    nl = k1 - k0
    if nslabs is None:
        nslabs = max(1, nl // 8)
    nrow_layer = (nx + 1) * (ny + 1) * blk
    n = nl * nrow_layer
    layers = [k0 + round(s * nl / nslabs) for s in range(nslabs + 1)]
    ro = np.empty(n + 1, np.int64)
    ro[0] = 0
    start = 0
    for s in range(nslabs):
        lens = _slab_row_lengths(kind, nx, ny, nz, layers[s], layers[s + 1])
        np.cumsum(lens, out=ro[start + 1:start + 1 + lens.size])
        ro[start + 1:start + 1 + lens.size] += ro[start]
        start += lens.size
    nnz = int(ro[n])
    ci = np.empty(nnz, np.int64)
    v = np.empty(nnz, np.float64)
    row0 = k0 * nrow_layer

    def fill(slab):
        a, b = layers[slab], layers[slab + 1]
        if b <= a:
            return
        rb, _, r, c, vv = box_rows(kind, nx, ny, nz, a, b, **kw)
        at = ro[rb - row0]
        ci[at:at + c.size] = c
        v[at:at + c.size] = vv

    if workers <= 1:
        for slab in range(nslabs):
            fill(slab)
    else:
        # numpy releases the GIL in the bulk array work: threads share the
        # output arrays, no copies
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(fill, range(nslabs)))
    return row0, (nx + 1) * (ny + 1) * (nz + 1) * blk, ro, ci, v


def elasticity_box_slabbed(nx=321, ny=321, nz=321):
    """Config 5 on one GPU: the 100M-row elasticity box, built slab by slab."""
    return box_csr_slabbed("elasticity", nx, ny, nz, nslabs=max(1, (nz + 1) // 8), workers=8)


def slab_layers(nz, nparts):
    """Node-layer boundaries of a z-slab partition of box(., ., nz)."""
    return [round(g * (nz + 1) / nparts) for g in range(nparts + 1)]


def _tet_grad_vol(p0, p1, p2, p3):
    """Closed-form P1 gradients (4 x (..., 3)) and volumes of tets whose corner
    coordinates are (..., 3) arrays (element_geometry, fem/element.cpp:7-47)."""
    e1, e2, e3 = p1 - p0, p2 - p0, p3 - p0
    c23 = np.cross(e2, e3)
    c31 = np.cross(e3, e1)
    c12 = np.cross(e1, e2)
    det = np.einsum("...j,...j->...", e1, c23)
    g1 = c23 / det[..., None]
    g2 = c31 / det[..., None]
    g3 = c12 / det[..., None]
    g0 = -(g1 + g2 + g3)
    return (g0, g1, g2, g3), np.abs(det) / 6.0


def ventricle_box(nx=170, ny=170, nz=170, jitter=0.3, sigma=1e-3, seed=4, slab=16):
    """Config 4: jittered P1 operator, unknowns renumbered at random."""
    rng = np.random.default_rng(seed)
    n1, n2, n3 = nx + 1, ny + 1, nz + 1
    kk, jj, ii = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    xyz = np.stack([ii, jj, kk], axis=-1).astype(np.float64)  # (n3, n2, n1, 3)
    xyz += rng.uniform(-jitter, jitter, size=xyz.shape)
    tets = _tet_corners()

    def acc(dense):
        d3 = dense.reshape(n3, n2, n1, len(_STENCIL))
        for k0 in range(0, nz, slab):
            k1 = min(nz, k0 + slab)
            for corners in tets:
                pts = [xyz[k0 + c[2]:k1 + c[2], c[1]:ny + c[1], c[0]:nx + c[0]] for c in corners]
                grads, vol = _tet_grad_vol(*pts)
                for a in range(4):
                    ca = corners[a]
                    tgt = d3[k0 + ca[2]:k1 + ca[2], ca[1]:ny + ca[1], ca[0]:nx + ca[0]]
                    for b in range(4):
                        d = _dir_index(tuple(np.subtract(corners[b], corners[a])))
                        val = vol * np.einsum("...j,...j->...", grads[a], grads[b])
                        if a == b:
                            val += sigma * vol / 4.0
                        tgt[..., d] += val

    n, _, ro, ci, v = _stencil_csr(nx, ny, nz, 1, acc)
    perm = rng.permutation(n).astype(np.int64)  # new id of old unknown
    return renumber(n, ro, ci, v, perm)


def renumber(n, ro, ci, v, new_of_old):
    """Symmetric renumbering P A P^T with columns re-sorted per row."""
    lens = np.diff(ro)
    width = int(lens.max()) if n else 0
    old_of_new = np.empty(n, np.int64)
    old_of_new[new_of_old] = np.arange(n, dtype=np.int64)
    new_lens = lens[old_of_new]
    ro2 = np.zeros(n + 1, np.int64)
    np.cumsum(new_lens, out=ro2[1:])
    # rows padded to `width`, sorted by new column, padding sorts last
    slot = np.arange(width)[None, :]
    src = ro[old_of_new][:, None] + slot
    valid = slot < new_lens[:, None]
    src = np.where(valid, src, 0)
    cols = np.where(valid, new_of_old[ci[src]], np.iinfo(np.int64).max)
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(v[src], order, axis=1)
    keep = np.take_along_axis(valid, order, axis=1)
    return n, n, ro2, cols[keep], vals[keep]


def random_x(n, seed=1):
    """x = U(0.1, 1), the bench input (bench.cpp:27-33 draws it with
    mt19937_64; any fixed seeded draw serves the throughput runs)."""
    return np.random.default_rng(seed).uniform(0.1, 1.0, n)


def stats(ro):
    lens = np.diff(ro)
    return dict(nrows=int(lens.size), nnz=int(ro[-1]), minrow=int(lens.min()), maxrow=int(lens.max()),
                mean=float(lens.mean()))


# ---------------------------------------------------------------------------
# Config 3: the paper's 15-matrix suite at its Table 2 sizes
# ---------------------------------------------------------------------------
# PAPER.md:526-542 (Table 2): name, nz, nrows, minrow, maxrow. The matrices
# themselves are not available (no network): each is a seeded synthetic
# stand-in of the same kind the reference's registry uses
# (bench/fetch.cpp:16-46: powerlaw_rows for circuit / economics / webbase,
# uniform_band for qcd, a mesh-like graph for the FEM and heart matrices),
# with its parameters chosen so that nz, nrows, minrow and maxrow land on
# Table 2 (tests/test_workloads.py checks them within 5%, most exactly).
TABLE2 = [
    ("circuit", 958_936, 170_998, 1, 353),
    ("economics", 1_273_389, 206_500, 1, 44),
    ("epidemiology", 2_100_225, 525_825, 2, 4),
    ("accelerator", 2_624_331, 121_192, 8, 81),
    ("cantilever", 4_007_383, 62_451, 1, 78),
    ("harbor", 2_374_001, 46_835, 4, 145),
    ("ship", 7_813_404, 140_874, 24, 102),
    ("spheres", 6_010_480, 83_334, 1, 81),
    ("heart3k", 37_035, 3_129, 5, 21),
    ("heart5k", 52_715, 4_563, 6, 22),
    ("heart30k", 367_443, 28_639, 6, 24),
    ("protein", 4_344_765, 36_417, 18, 204),
    ("qcd", 1_916_928, 49_152, 39, 39),
    ("webbase", 3_105_536, 1_000_005, 1, 4700),
    ("windtunnel", 11_634_424, 217_918, 2, 180),
]
_TABLE2_SEED = {name: 11 + i for i, (name, *_rest) in enumerate(TABLE2)}


def powerlaw_lengths(nrows, alpha, maxrow, ncols=0):
    """Row lengths powerlaw_rows draws before its shuffle (synth.cpp:83-93)."""
    ncols = ncols if ncols > 0 else max(nrows, maxrow)
    cap = min(maxrow, ncols)
    k = np.arange(1, nrows + 1, dtype=np.float64)
    return np.clip(np.floor(cap * k ** -alpha + 0.5), 1, cap).astype(np.int64)


def powerlaw_alpha(nrows, maxrow, nnz):
    """The exponent for which powerlaw_rows(nrows, alpha, maxrow) has `nnz`
    entries (bisection; nnz is decreasing in alpha)."""
    lo, hi = 1e-3, 8.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if powerlaw_lengths(nrows, mid, maxrow).sum() > nnz:
            lo = mid
        else:
            hi = mid
    a, b = powerlaw_lengths(nrows, lo, maxrow).sum(), powerlaw_lengths(nrows, hi, maxrow).sum()
    return lo if abs(a - nnz) <= abs(b - nnz) else hi


def powerlaw_rows_scaled(nrows, alpha, scale, maxrow, seed):
    """powerlaw_rows' row-length law with its scale decoupled from the cap:
    lengths clamp(round(scale * k^-alpha), 1, maxrow), shuffled, each row's
    columns distinct and uniform over [0, nrows), ascending (synth.cpp:76-128
    ties scale to maxrow, which cannot give Circuit / Economics both their
    Table 2 nz and a shortest row of 1). Values U(0.1, 1)."""
    rng = np.random.default_rng(seed)
    k = np.arange(1, nrows + 1, dtype=np.float64)
    L = np.clip(np.floor(scale * k ** -alpha + 0.5), 1, maxrow).astype(np.int64)
    L = L[rng.permutation(nrows)]
    need = L.copy()
    got_r, got_c = [], []
    rows = np.arange(nrows)
    while need.sum() > 0:
        rr = np.repeat(rows, need)
        cc = rng.integers(0, nrows, rr.size)
        got_r.append(rr)
        got_c.append(cc)
        r = np.concatenate(got_r)
        c = np.concatenate(got_c)
        key = np.unique(r * nrows + c)  # sorted, distinct (row, col)
        r, c = key // nrows, key % nrows
        cnt = np.bincount(r, minlength=nrows)
        # keep at most L[row] per row (the first, i.e. smallest, columns are
        # as random as any: draws are uniform)
        start = np.zeros(nrows + 1, np.int64)
        np.cumsum(cnt, out=start[1:])
        pos = np.arange(r.size) - start[r]
        keep = pos < L[r]
        r, c = r[keep], c[keep]
        got_r, got_c = [r], [c]
        need = L - np.bincount(r, minlength=nrows)
    ro = np.zeros(nrows + 1, np.int64)
    np.cumsum(L, out=ro[1:])
    v = rng.uniform(0.1, 1.0, c.size)
    return nrows, nrows, ro, c.astype(np.int64), v


def powerlaw_scaled_fit(nrows, maxrow, nnz):
    """(alpha, scale) with scale * nrows^-alpha = 1 (the longest-k rows
    reach length 1) and sum of lengths = nnz (bisection on alpha)."""
    def total(a):
        sc = float(nrows) ** a
        k = np.arange(1, nrows + 1, dtype=np.float64)
        return np.clip(np.floor(sc * k ** -a + 0.5), 1, maxrow).sum(), sc

    lo, hi = 1e-3, 4.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if total(mid)[0] < nnz:
            lo = mid
        else:
            hi = mid
    a = lo if abs(total(lo)[0] - nnz) <= abs(total(hi)[0] - nnz) else hi
    return a, total(a)[1]


def grid2d(nx, ny):
    """4-neighbour grid graph (a 2D Markov chain like Epidemiology's mc2depi:
    2 entries per corner row, 3 per edge row, 4 inside; no diagonal)."""
    n = nx * ny
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    i, j = i.ravel(), j.ravel()
    node = np.arange(n, dtype=np.int64)
    nb = []
    for di, dj, off in ((0, -1, -nx), (-1, 0, -1), (1, 0, 1), (0, 1, nx)):  # ascending column
        ok = (i + di >= 0) & (i + di < nx) & (j + dj >= 0) & (j + dj < ny)
        nb.append(np.where(ok, node + off, -1))
    cols = np.stack(nb, axis=1)
    keep = cols >= 0
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(keep.sum(axis=1), out=ro[1:])
    ci = cols[keep]
    v = np.full(ci.size, 0.25)
    return n, n, ro, ci, v


def fem_rows(n, minrow, maxrow, nnz, seed, window=None):
    """A mesh-like sparse matrix with exactly `nnz` entries, row lengths in
    [minrow, maxrow] (both attained) from a clamped normal whose mean is
    nnz / n, and each row's off-diagonal columns drawn without replacement
    from a window of +-window around the diagonal (the locality of a banded
    FEM numbering, as fem_tet_graph's window, synth.cpp:56-70). Columns
    ascending; diagonal L + 0.5, off-diagonal -U(0.1, 1)."""
    rng = np.random.default_rng(seed)
    sd = (maxrow - minrow) / 6.0 + 0.5
    z = rng.standard_normal(n)

    def lens(mu):
        return np.clip(np.floor(mu + sd * z + 0.5), minrow, maxrow).astype(np.int64)

    lo, hi = minrow - 4 * sd, maxrow + 4 * sd
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if lens(mid).sum() < nnz:
            lo = mid
        else:
            hi = mid
    L = lens(hi)
    L[int(np.argmin(z))] = minrow
    L[int(np.argmax(z))] = maxrow
    fixed = {int(np.argmin(z)), int(np.argmax(z))}
    # move the total onto nnz one entry at a time on random free rows
    d = int(L.sum()) - nnz
    order = rng.permutation(n)
    for r in order:
        if d == 0:
            break
        if int(r) in fixed:
            continue
        if d > 0 and L[r] > minrow:
            step = min(d, int(L[r] - minrow))
            L[r] -= step
            d -= step
        elif d < 0 and L[r] < maxrow:
            step = min(-d, int(maxrow - L[r]))
            L[r] += step
            d += step
    W = window or max(2 * maxrow, 32)
    offs = np.concatenate([np.arange(-W, 0), np.arange(1, W + 1)])
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(L, out=ro[1:])
    ci = np.empty(int(ro[-1]), np.int64)
    v = np.empty(int(ro[-1]), np.float64)
    chunk = max(1, (1 << 22) // (2 * W))
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        rows = np.arange(a, b)
        cand = rows[:, None] + offs[None, :]
        key = rng.random(cand.shape)
        key[(cand < 0) | (cand >= n)] = np.inf
        pick = np.argsort(key, axis=1, kind="stable")
        cand = np.take_along_axis(cand, pick, axis=1)
        take = np.arange(2 * W)[None, :] < (L[a:b] - 1)[:, None]
        cand = np.where(take, cand, np.iinfo(np.int64).max)
        full = np.concatenate([cand, rows[:, None]], axis=1)  # + the diagonal
        full.sort(axis=1)
        keep = full != np.iinfo(np.int64).max
        ci[ro[a]:ro[b]] = full[keep]
        vals = -rng.uniform(0.1, 1.0, full.shape)
        vals[full == rows[:, None]] = (L[a:b] + 0.5)[:, None].repeat(full.shape[1], axis=1)[full == rows[:, None]]
        v[ro[a]:ro[b]] = vals[keep]
    return n, n, ro, ci, v


def table2_spec(name):
    """(kind, parameters) of config 3's stand-in for Table 2 matrix `name`."""
    row = {t[0]: t for t in TABLE2}[name]
    _, nnz, n, mn, mx = row
    seed = _TABLE2_SEED[name]
    if name == "webbase":
        return "powerlaw_rows", dict(nrows=n, alpha=powerlaw_alpha(n, mx, nnz), maxrow=mx, seed=seed)
    if name in ("circuit", "economics"):
        a, sc = powerlaw_scaled_fit(n, mx, nnz)
        return "powerlaw_rows_scaled", dict(nrows=n, alpha=a, scale=sc, maxrow=mx, seed=seed)
    if name == "epidemiology":
        return "grid2d", dict(nx=675, ny=779)  # 675 x 779 = 525,825 rows
    if name == "qcd":
        return "uniform_band", dict(n=n, row_len=mx)
    return "fem_rows", dict(n=n, minrow=mn, maxrow=mx, nnz=nnz, seed=seed)


def table2_matrix(name, ew_mod=None):
    """Config 3's stand-in for Table 2 matrix `name` as (nrows, ncols, ro,
    ci, v). powerlaw_rows runs the reference's generator (our seed-identical
    C++ port, through _ellwarp)."""
    kind, p = table2_spec(name)
    if kind == "powerlaw_rows":
        if ew_mod is None:
            from paper_1501_00324_b200 import load_ellwarp

            ew_mod = load_ellwarp()
        m = ew_mod.powerlaw_rows(p["nrows"], p["alpha"], p["maxrow"], p["seed"])
        return (m.nrows, m.ncols, np.asarray(m.row_offsets, np.int64), np.asarray(m.col_indices, np.int64),
                np.asarray(m.values, np.float64))
    if kind == "powerlaw_rows_scaled":
        return powerlaw_rows_scaled(**p)
    if kind == "grid2d":
        return grid2d(p["nx"], p["ny"])
    if kind == "uniform_band":
        n, L = p["n"], p["row_len"]
        ro = np.arange(n + 1, dtype=np.int64) * L
        cols = (np.arange(n)[:, None] + np.arange(L)[None, :]) % n
        cols.sort(axis=1)
        v = np.where(cols == np.arange(n)[:, None], 2.0 * L, -1.0)  # synth.cpp:130-140
        return n, n, ro, cols.ravel().astype(np.int64), v.ravel()
    return fem_rows(**p)
