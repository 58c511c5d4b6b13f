"""P1 finite-element assembly on structured simplicial meshes (oracle; test infra only).

PAPER.md:218-223 (§3): "H^1-conforming finite element spaces V_h ⊂ V constructed in
terms of P1 elements ... T_h is a discrete trace operator ... the discrete trace space
V_{Γ,h} = Q_h built likewise using P1 elements".

Geometry (BASELINE.json configs; SURVEY.md §8 "Geometry"):
  2D  Ω=(0,1)^2, each cell split along its (0,0)->(1,1) diagonal (Freudenthal);
  3D  Ω=(0,1)^3, each cube split into the 6 Kuhn tetrahedra along (0,0,0)->(1,1,1).
  Γ = {x = 0}.  Homogeneous Dirichlet on ∂Ω \\ Γ and on ∂Γ (reading A3 in DESIGN.md).
  Bulk operator is the P1 stiffness only (Eq.(2) is -KΔ with no mass; reading A5).

Everything here is element-by-element assembly (no stencils are typed in), so the
stencil closed forms used elsewhere are *checked* against it, never assumed.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp


def _p1_element(P: np.ndarray):
    """Stiffness and mass of one P1 simplex with vertex coordinates P (d+1, d).

    Barycentric gradients from the inverse of [1 | P]; stiffness = |T| G G^T,
    mass = |T| (1 + δ_ij) / ((d+1)(d+2)).
    """
    d = P.shape[1]
    Mx = np.hstack([np.ones((d + 1, 1)), P])
    C = np.linalg.inv(Mx)
    G = C[1:, :].T                                  # (d+1, d) gradients of barycentric coords
    vol = abs(np.linalg.det(Mx)) / float(np.prod(np.arange(1, d + 1)))
    Ke = vol * G @ G.T
    Me = vol * (np.ones((d + 1, d + 1)) + np.eye(d + 1)) / ((d + 1) * (d + 2))
    return Ke, Me, vol


def _assemble(n_nodes, cells, coords):
    rows, cols, kv, mv = [], [], [], []
    cache = {}
    for cell in cells:
        P = coords[list(cell)]
        key = tuple(np.round((P - P[0]) * 1e9).astype(np.int64).ravel())
        if key not in cache:  # structured mesh: only a handful of distinct element shapes
            cache[key] = _p1_element(P)
        Ke, Me, _ = cache[key]
        idx = np.asarray(cell)
        rows.append(np.repeat(idx, len(idx)))
        cols.append(np.tile(idx, len(idx)))
        kv.append(Ke.ravel())
        mv.append(Me.ravel())
    r = np.concatenate(rows); c = np.concatenate(cols)
    K = sp.csr_matrix((np.concatenate(kv), (r, c)), shape=(n_nodes, n_nodes))
    M = sp.csr_matrix((np.concatenate(mv), (r, c)), shape=(n_nodes, n_nodes))
    K.sum_duplicates(); M.sum_duplicates()
    return K, M


# --------------------------------------------------------------------------- meshes
def square_mesh(N: int):
    """Freudenthal P1 mesh of (0,1)^2: node (i, j) at (i h, j h) has id i*(N+1)+j."""
    if N < 1:
        raise ValueError("N >= 1")
    h = 1.0 / N
    ii, jj = np.meshgrid(np.arange(N + 1), np.arange(N + 1), indexing="ij")
    coords = np.stack([ii.ravel() * h, jj.ravel() * h], axis=1)
    nid = lambda i, j: i * (N + 1) + j
    cells = []
    for i in range(N):
        for j in range(N):
            v00, v10, v11, v01 = nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)
            cells.append((v00, v10, v11))
            cells.append((v00, v11, v01))
    return coords, np.asarray(cells)


def cube_mesh(N: int):
    """Kuhn P1 mesh of (0,1)^3: node (i,j,k) has id (i*(N+1)+j)*(N+1)+k; 6 tets per cube,
    one per monotone lattice path (0,0,0)->(1,1,1)."""
    if N < 1:
        raise ValueError("N >= 1")
    h = 1.0 / N
    g = np.arange(N + 1)
    ii, jj, kk = np.meshgrid(g, g, g, indexing="ij")
    coords = np.stack([ii.ravel() * h, jj.ravel() * h, kk.ravel() * h], axis=1)
    nid = lambda i, j, k: (i * (N + 1) + j) * (N + 1) + k
    E = np.eye(3, dtype=int)
    cells = []
    for i in range(N):
        for j in range(N):
            for k in range(N):
                base = np.array([i, j, k])
                for perm in itertools.permutations(range(3)):
                    v = base.copy(); path = [nid(*v)]
                    for ax in perm:
                        v = v + E[ax]; path.append(nid(*v))
                    cells.append(tuple(path))
    return coords, np.asarray(cells)


# --------------------------------------------------------------------------- problems
class BulkProblem:
    """Assembled bulk stiffness with the DOF partition V = V0 ⊕ VΓ.

    Attributes
    ----------
    A : csr, stiffness on the free (non-Dirichlet) nodes, ordered [Γ nodes, interior nodes]
    n_gamma, n_int : sizes; Γ nodes ordered lexicographically (2D: by j; 3D: j-major)
    layer_of : layer index (x-index i) of every free node in that order (0 = Γ)
    """

    def __init__(self, dim: int, N: int):
        self.dim, self.N = dim, N
        coords, cells = (square_mesh(N) if dim == 2 else cube_mesh(N))
        K, Mfull = _assemble(coords.shape[0], cells, coords)
        idx = np.rint(coords * N).astype(np.int64)          # integer lattice coordinates
        i = idx[:, 0]
        others = idx[:, 1:]
        dirichlet = (i == N) | np.any((others == 0) | (others == N), axis=1)
        gamma = (i == 0) & ~dirichlet
        inner = (i > 0) & ~dirichlet

        def order(mask):
            ids = np.nonzero(mask)[0]
            key = [idx[ids, a] for a in range(dim - 1, -1, -1)]   # sort by (i, j, k) lexicographic
            return ids[np.lexsort(key)]

        g_ids, i_ids = order(gamma), order(inner)
        perm = np.concatenate([g_ids, i_ids])
        self.A = K[perm][:, perm].tocsr()
        self.M = Mfull[perm][:, perm].tocsr()     # consistent P1 mass on the free nodes (same order)
        self.n_gamma, self.n_int = len(g_ids), len(i_ids)
        self.layer_of = idx[perm, 0]
        self.coords = coords[perm]

    def blocks(self):
        """(A^ii, A^i0, A^00) of Eq.(4): Γ-Γ, Γ-interior, interior-interior (sparse)."""
        g = self.n_gamma
        A = self.A
        return A[:g, :g], A[:g, g:], A[g:, g:]


def trace_pair(dim: int, N: int):
    """P1 stiffness/mass pair (A_Γ, M_Γ) on Γ = {x=0} with Dirichlet ∂Γ.

    Assembled on the trace mesh: the facets of the bulk mesh lying on x = 0 (edges in
    2D, Kuhn-face triangles in 3D), in the same Γ ordering as `BulkProblem`.
    Returns dense (A_Γ, M_Γ).
    """
    coords, cells = (square_mesh(N) if dim == 2 else cube_mesh(N))
    on_gamma = np.isclose(coords[:, 0], 0.0)
    facets = set()
    for cell in cells:
        for f in itertools.combinations(sorted(cell), dim):       # facets = d-subsets
            if all(on_gamma[v] for v in f):
                facets.add(f)
    facets = sorted(facets)
    tc = coords[:, 1:]                                            # coordinates within Γ
    K, M = _assemble(coords.shape[0], facets, tc)
    idx = np.rint(coords * N).astype(np.int64)
    others = idx[:, 1:]
    free = on_gamma & ~np.any((others == 0) | (others == N), axis=1)
    ids = np.nonzero(free)[0]
    key = [idx[ids, a] for a in range(dim - 1, 0, -1)]
    ids = ids[np.lexsort(key)]
    return K[ids][:, ids].toarray(), M[ids][:, ids].toarray()


def trace_pair_1d(N: int):
    """1D P1 pair on the trace mesh of Γ = {x=0} of the unit square, assembled directly
    on its N edges (same matrices as `trace_pair(2, N)`, which tests check), returned in
    symmetric tridiagonal form: (a_diag, a_off, m_diag, m_off) arrays of length n / n-1.
    Avoids the O(N^2) bulk mesh walk so the oracle reaches N = 4096."""
    if N < 2:
        raise ValueError("N >= 2")
    n = N - 1
    y = np.arange(N + 1) / N
    a_d = np.zeros(N + 1); a_o = np.zeros(N); m_d = np.zeros(N + 1); m_o = np.zeros(N)
    for e in range(N):                      # element [y_e, y_e+1]
        Ke, Me, _ = _p1_element(y[e:e + 2, None])
        a_d[e] += Ke[0, 0]; a_d[e + 1] += Ke[1, 1]; a_o[e] += Ke[0, 1]
        m_d[e] += Me[0, 0]; m_d[e + 1] += Me[1, 1]; m_o[e] += Me[0, 1]
    # drop the Dirichlet end nodes 0 and N
    return a_d[1:N], a_o[1:N - 1], m_d[1:N], m_o[1:N - 1]


def trace_pair_face(N: int):
    """The 3D trace pair (A_Γ, M_Γ) of `trace_pair(3, N)`, assembled directly on the trace mesh
    of the face Γ = {x=0} — the facets of the Kuhn tetrahedra on x = 0, which are the triangles
    of the (y, z) square split along (0,0)->(1,1) — without walking the 6 N^3 bulk cells, so the
    oracle reaches the config-4 face (N = 128).  Same P1 element integrals (`_p1_element`), same
    Dirichlet ∂Γ and j-major ordering; equality with `trace_pair(3, N)` is pinned in the tests.
    Returns sparse CSR (A_Γ, M_Γ)."""
    if N < 2:
        raise ValueError("N >= 2")
    coords, cells = square_mesh(N)          # node (j, k) at (j h, k h) in the face's (y, z) plane
    K, M = _assemble(coords.shape[0], cells, coords)
    idx = np.rint(coords * N).astype(np.int64)
    free = np.all((idx > 0) & (idx < N), axis=1)
    ids = np.nonzero(free)[0]               # ascending id = j (N+1) + k: j-major
    return K[ids][:, ids].tocsr(), M[ids][:, ids].tocsr()
