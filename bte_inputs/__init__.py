"""Seeded synthetic inputs for the phonon-BTE hot path (arXiv 2305.19400).

This module is the ONE thing the CPU oracle (``oracle/``) and the CUDA path
(``paper_2305_19400_b200``) both consume.  It holds problem DATA only -- mesh
sizes, the direction quadrature, channel/material tables, wall temperatures,
seeds and noise -- and none of the method's arithmetic: no equilibrium
intensity I0(T), no flux, no reduction, no Newton.  Anything that needs I0
(e.g. an initial intensity field) is assembled by the caller from the pieces
returned here with its own implementation.

Citations: P:L<a>-<b> = /root/reference/PAPER.md lines (the paper, arXiv
2305.19400); readings #n = DESIGN.md "Readings of the paper".
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np

# --------------------------------------------------------------------------
# physical constants (CODATA 2018, exact SI values for kB)
HBAR = 1.054571817e-34  # J s
KB = 1.380649e-23  # J / K

BC_ISOTHERMAL = 0
BC_SPECULAR = 1
BC_DIFFUSE = 2
BC_PARTIAL = 3  # partially specular: specularity*specular + (1 - specularity)*diffuse

I0_LINEAR = 0
I0_BOSE_EINSTEIN = 1

REGION_NAMES = ("-x", "+x", "-y", "+y", "-z", "+z")


@dataclasses.dataclass
class Mesh:
    """Uniform structured grid ("a 120x120 grid of uniform cells").

    Canonical cell index c = x + nx*(y + ny*z).  dim=2 means no z faces
    (nz must be 1); dz is then the (unit) depth used only for volumes.
    """

    dim: int
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz

    def n_faces(self, region: int) -> int:
        """Boundary faces on a wall region (0..5 = -x,+x,-y,+y,-z,+z)."""
        ax = region // 2
        if ax == 0:
            return self.ny * self.nz
        if ax == 1:
            return self.nx * self.nz
        return self.nx * self.ny


@dataclasses.dataclass
class UMesh:
    """Unstructured mesh (Eq. 3 P:L176-184 holds for "a
    polygonal/polyhedral cell with m sides"): convex polygons in 2-D (3
    vertices: triangles, 4: quadrilaterals, in boundary order) or tetrahedra
    (dim 3, 4 vertices).  DATA only: vertex coordinates [nverts, 3] (z = 0 in
    2-D) and cell -> vertex lists [ncells, m].  Face k of a cell is the edge
    (v_{k+1}, v_{k+2}) in 2-D (for a triangle: the edge opposite v_k) and the
    face opposite v_k of a tetrahedron.  The domain is the axis-aligned box
    spanned by the vertices; every boundary face must lie on one of its walls
    (region 0..5 = -x,+x,-y,+y,-z,+z, tested in that order).  depth is the z
    extent of a 2-D mesh (volumes = area*depth)."""

    dim: int
    verts: np.ndarray
    cells: np.ndarray
    depth: float = 1.0

    @property
    def ncells(self) -> int:
        return int(self.cells.shape[0])

    @property
    def nverts(self) -> int:
        return int(self.verts.shape[0])


@dataclasses.dataclass
class Directions:
    """Discrete directions s_d (unit vectors, [nd,3]) and weights w_d [nd]."""

    s: np.ndarray
    w: np.ndarray

    @property
    def nd(self) -> int:
        return int(self.s.shape[0])


@dataclasses.dataclass
class Bands:
    """Per-channel tables (readings #1, #5, #6, #15, #16).

    mode I0_LINEAR:        I0_b(T) = I_ref[b] + slope[b]*(T - T_ref)
    mode I0_BOSE_EINSTEIN: band integral over [w_lo, w_hi] with the quadratic
                           dispersion omega = vs*k + c2*k^2 and degeneracy g.
    beta_coef[b] = (p0, p3, p4, pu, theta):
        beta_b(T) = p0 + p3*T^3 + p4*T^4 + pu/sinh(theta/T)   (pu = 0 drops the term)
    """

    v: np.ndarray
    mode: int
    beta_coef: np.ndarray
    I_ref: Optional[np.ndarray] = None
    slope: Optional[np.ndarray] = None
    T_ref: float = 300.0
    w_lo: Optional[np.ndarray] = None
    w_hi: Optional[np.ndarray] = None
    vs: Optional[np.ndarray] = None
    c2: Optional[np.ndarray] = None
    g: Optional[np.ndarray] = None
    polarization: Optional[List[str]] = None

    @property
    def nb(self) -> int:
        return int(self.v.shape[0])


@dataclasses.dataclass
class WallBC:
    kind: int
    T_wall: Optional[np.ndarray] = None  # per boundary face (isothermal only)
    T_uniform: float = 300.0
    specularity: float = 1.0  # BC_PARTIAL only, in [0, 1]


@dataclasses.dataclass
class Problem:
    name: str
    mesh: Mesh
    dirs: Directions
    bands: Bands
    dt: float
    T_init: float
    bcs: List[WallBC]  # 6 entries (-x,+x,-y,+y,-z,+z); z entries ignored for dim 2
    nsteps: int = 100
    seed: int = 0
    tau_mode: int = 0  # 0: lagged tau (reading #15); 1: self-consistent tau(T^{n+1}) (reading R-k)
    semi: int = 0  # 1: semi-implicit step (explicit advection, implicit relaxation; reading R-l)
    implicit: int = 0  # 1: implicit step by source iteration (reading R-n)
    imp_max_iter: int = 0  # R-n: iterations per step (exactly this many when imp_tol == 0)
    imp_tol: float = 0.0  # R-n: stop early when max_c |T^{k+1} - T^k| / T^k <= imp_tol

    @property
    def dof(self) -> int:
        return self.mesh.ncells * self.dirs.nd * self.bands.nb


# --------------------------------------------------------------------------
# direction quadratures (reading #7): generated in the first octant/quadrant
# and sign-flipped, so every axis reflection is bit-exact.

def directions_inplane(n: int) -> Directions:
    """2-D in-plane set theta_d = 2*pi*(d - 1/2)/n, w_d = 2*pi/n.

    Emitted in ascending theta; values of quadrants 2-4 are exact sign flips
    of the first-quadrant values, so reflections are bit-exact.
    """
    if n < 4 or n % 4:
        raise ValueError("in-plane direction count must be a positive multiple of 4")
    q = n // 4
    th = [2.0 * math.pi * (j + 0.5) / n for j in range(q)]
    c = [math.cos(t) for t in th]
    sn = [math.sin(t) for t in th]
    s = []
    for j in range(q):  # quadrant 1: (+,+)
        s.append((c[j], sn[j], 0.0))
    for j in range(q):  # quadrant 2: theta = pi - th[m], m descending
        m = q - 1 - j
        s.append((-c[m], sn[m], 0.0))
    for j in range(q):  # quadrant 3: theta = pi + th[j]
        s.append((-c[j], -sn[j], 0.0))
    for j in range(q):  # quadrant 4: theta = 2 pi - th[m]
        m = q - 1 - j
        s.append((c[m], -sn[m], 0.0))
    w = np.full(n, 2.0 * math.pi / n)
    return Directions(np.asarray(s, dtype=np.float64), w)


def directions_control_angle(n_theta: int = 20, n_phi: int = 20) -> Directions:
    """3-D control-angle set: n_theta uniform polar cells on [0,pi] x n_phi azimuthal
    cells on [0,2pi] ("20x20 = 400"; reading #7/#8).

    s = unit vector at the cell midpoint, w = dphi*(cos th_lo - cos th_hi).
    Octant-major order o = 4*[sx<0] + 2*[sy<0] + [sz<0]; inside an octant the
    first-octant index j (theta-major, phi ascending) -- reflections map j->j.
    """
    if n_theta % 2 or n_phi % 4:
        raise ValueError("need n_theta even and n_phi divisible by 4")
    dth = math.pi / n_theta
    dph = 2.0 * math.pi / n_phi
    first = []
    for i in range(n_theta // 2):
        th_lo, th_hi = i * dth, (i + 1) * dth
        thm = (i + 0.5) * dth
        w = dph * (math.cos(th_lo) - math.cos(th_hi))
        for k in range(n_phi // 4):
            phm = (k + 0.5) * dph
            first.append((math.sin(thm) * math.cos(phm), math.sin(thm) * math.sin(phm), math.cos(thm), w))
    s, ws = [], []
    for o in range(8):
        sx = -1.0 if o & 4 else 1.0
        sy = -1.0 if o & 2 else 1.0
        sz = -1.0 if o & 1 else 1.0
        for (a, b, c, w) in first:
            s.append((sx * a, sy * b, sz * c))
            ws.append(w)
    return Directions(np.asarray(s, dtype=np.float64), np.asarray(ws, dtype=np.float64))


# --------------------------------------------------------------------------
# channel tables

# Pop-type quadratic dispersion and Holland-type relaxation constants for
# silicon: paper-silent material DATA (P:L392-394 defers to Ali2014 and
# mazumder2022); values as recorded in SURVEY.md Appendix A.
SI_LATTICE = 5.43e-10
SI_LA = dict(vs=9.01e3, c2=-2.00e-7, g=1.0)
SI_TA = dict(vs=5.23e3, c2=-2.26e-7, g=2.0)
SI_A_IMP = 1.32e-45  # s^3        beta_I  = A w^4
SI_B_L = 2.0e-24  # s K^-3        beta_L  = B_L w^2 T^3
SI_B_TN = 9.3e-13  # K^-4         beta_TN = B_TN w T^4        (w < w_half)
SI_B_TU = 5.5e-18  # s            beta_TU = B_TU w^2 / sinh(hbar w / kB T)
SI_W_HALF = 2.42e13  # rad/s


def _omega_max(vs: float, c2: float, kmax: float) -> float:
    return vs * kmax + c2 * kmax * kmax


def silicon_bands(n_freq: int) -> Bands:
    """n_freq uniform bands on [0, w_max,LA]; a TA channel for each band lying
    fully below w_max,TA (reading #6).  n_freq=40 -> 40 LA + 15 TA = 55
    channels; n_freq=29 -> 29 + 11 = 40 (reading #5).

    Channel order: all LA bands ascending, then TA bands ascending.
    v_b = d(omega)/dk at the band centre = sqrt(vs^2 + 4*c2*w_c) (reading #16).
    """
    kmax = 2.0 * math.pi / SI_LATTICE
    wmax_la = _omega_max(SI_LA["vs"], SI_LA["c2"], kmax)
    wmax_ta = _omega_max(SI_TA["vs"], SI_TA["c2"], kmax)
    dw = wmax_la / n_freq
    rows = []
    for pol, prm in (("LA", SI_LA), ("TA", SI_TA)):
        for i in range(n_freq):
            lo, hi = i * dw, (i + 1) * dw
            if pol == "TA" and hi > wmax_ta:
                continue
            rows.append((pol, lo, hi, prm))
    nb = len(rows)
    v = np.empty(nb)
    w_lo = np.empty(nb)
    w_hi = np.empty(nb)
    vs = np.empty(nb)
    c2 = np.empty(nb)
    g = np.empty(nb)
    beta = np.zeros((nb, 5))
    pols = []
    for b, (pol, lo, hi, prm) in enumerate(rows):
        wc = 0.5 * (lo + hi)
        w_lo[b], w_hi[b] = lo, hi
        vs[b], c2[b], g[b] = prm["vs"], prm["c2"], prm["g"]
        v[b] = math.sqrt(prm["vs"] ** 2 + 4.0 * prm["c2"] * wc)
        beta[b, 0] = SI_A_IMP * wc ** 4
        if pol == "LA":
            beta[b, 1] = SI_B_L * wc ** 2
        elif wc < SI_W_HALF:
            beta[b, 2] = SI_B_TN * wc
        else:
            beta[b, 3] = SI_B_TU * wc ** 2
            beta[b, 4] = HBAR * wc / KB
        pols.append(pol)
    return Bands(v=v, mode=I0_BOSE_EINSTEIN, beta_coef=beta, w_lo=w_lo, w_hi=w_hi,
                 vs=vs, c2=c2, g=g, polarization=pols)


def gray_linear_bands(C: float = 1.66e6, v: float = 6400.0, tau: float = 40e-12,
                      T_ref: float = 300.0, W: float = 2.0 * math.pi) -> Bands:
    """Single gray channel, LINEAR I0 (SPEC S:L332 linear mode): slope a = C*v/W,
    I_ref = a*T_ref, constant tau (config 1)."""
    a = C * v / W
    beta = np.zeros((1, 5))
    beta[0, 0] = 1.0 / tau
    return Bands(v=np.array([v]), mode=I0_LINEAR, beta_coef=beta,
                 I_ref=np.array([a * T_ref]), slope=np.array([a]), T_ref=T_ref,
                 polarization=["gray"])


def linear_bands(v, tau, slope, I_ref, T_ref=300.0) -> Bands:
    """Generic multi-channel LINEAR table (tests)."""
    v = np.asarray(v, dtype=np.float64)
    beta = np.zeros((v.shape[0], 5))
    beta[:, 0] = 1.0 / np.asarray(tau, dtype=np.float64)
    return Bands(v=v, mode=I0_LINEAR, beta_coef=beta,
                 I_ref=np.asarray(I_ref, dtype=np.float64),
                 slope=np.asarray(slope, dtype=np.float64), T_ref=T_ref,
                 polarization=["lin"] * v.shape[0])


def debye_bands(v: float, kmax: float, nband: int) -> Bands:
    """Debye test table: c2 = 0, one polarization, bands tiling [0, v*kmax]."""
    wmax = v * kmax
    edges = np.linspace(0.0, wmax, nband + 1)
    beta = np.zeros((nband, 5))
    beta[:, 0] = 1e10
    return Bands(v=np.full(nband, v), mode=I0_BOSE_EINSTEIN, beta_coef=beta,
                 w_lo=edges[:-1].copy(), w_hi=edges[1:].copy(), vs=np.full(nband, v),
                 c2=np.zeros(nband), g=np.ones(nband), polarization=["D"] * nband)


def subset_bands(b: Bands, idx) -> Bands:
    idx = np.asarray(idx)
    pick = lambda a: None if a is None else np.ascontiguousarray(a[idx])
    return Bands(v=pick(b.v), mode=b.mode, beta_coef=np.ascontiguousarray(b.beta_coef[idx]),
                 I_ref=pick(b.I_ref), slope=pick(b.slope), T_ref=b.T_ref,
                 w_lo=pick(b.w_lo), w_hi=pick(b.w_hi), vs=pick(b.vs), c2=pick(b.c2),
                 g=pick(b.g), polarization=None if b.polarization is None else [b.polarization[i] for i in idx])


# --------------------------------------------------------------------------
# walls

def face_centre_offsets(n: int, d: float) -> np.ndarray:
    """Face-centre coordinate relative to the wall centre, x = ((2i+1) - n)*d/2,
    so mirrored faces get exactly negated x (reading #13)."""
    i = np.arange(n, dtype=np.float64)
    return ((2.0 * i + 1.0) - n) * d / 2.0


def hotspot_profile(nx: int, dx: float, T_cold: float = 300.0, T_peak: float = 350.0,
                    width: float = 10e-6) -> np.ndarray:
    """T_wall(x) = T_cold + (T_peak - T_cold)*exp(-2x^2/w^2), w = 1/e^2 distance
    10 um (reading #13)."""
    x = face_centre_offsets(nx, dx)
    return T_cold + (T_peak - T_cold) * np.exp(-2.0 * x * x / (width * width))


def uniform_bcs(kind: int, T: float = 300.0) -> List[WallBC]:
    return [WallBC(kind, None, T) for _ in range(6)]


# --------------------------------------------------------------------------
# random start (SURVEY 8(d) "random start")

MASK64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Standard splitmix64 output function applied to state x (uint64 array).
    The CUDA library carries its own copy (counter-based generator, one per side)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
        return z ^ (z >> np.uint64(31))


def uniform_noise(seed: int, n: int, start: int = 0) -> np.ndarray:
    """u_idx = (splitmix64(seed XOR idx) >> 11) * 2^-53 for idx in [start, start+n)."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    z = splitmix64(np.uint64(seed & MASK64) ^ idx)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_phases(seed: int) -> Tuple[float, float, float]:
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.random(3)
    return float(p[0]), float(p[1]), float(p[2])


def random_temperature(mesh: Mesh, seed: int, T_mean: float = 300.0, T_amp: float = 20.0,
                       box=None) -> np.ndarray:
    """T_c = T_mean + T_amp*sin(2pi(x/Lx+p1))*sin(2pi(y/Ly+p2))[*sin(2pi(z/Lz+p3))],
    x = cell centre (i+1/2)*dx with the GLOBAL index i.  Canonical cell order of
    the full mesh, or of the sub-box ((x0,x1),(y0,y1),(z0,z1)) when given."""
    if isinstance(mesh, UMesh):
        return random_temperature_umesh(mesh, seed, T_mean, T_amp)
    p1, p2, p3 = random_phases(seed)
    (x0, x1), (y0, y1), (z0, z1) = box if box is not None else ((0, mesh.nx), (0, mesh.ny), (0, mesh.nz))
    x = (np.arange(x0, x1) + 0.5) * mesh.dx
    y = (np.arange(y0, y1) + 0.5) * mesh.dy
    z = (np.arange(z0, z1) + 0.5) * mesh.dz
    fx = np.sin(2.0 * math.pi * (x / (mesh.nx * mesh.dx) + p1))
    fy = np.sin(2.0 * math.pi * (y / (mesh.ny * mesh.dy) + p2))
    if mesh.dim == 3:
        fz = np.sin(2.0 * math.pi * (z / (mesh.nz * mesh.dz) + p3))
    else:
        fz = np.ones(z1 - z0)
    T = T_mean + T_amp * (fz[:, None, None] * fy[None, :, None] * fx[None, None, :])
    return np.ascontiguousarray(T.reshape(-1))


def intensity_noise_factor(seed: int, ncells: int, nd: int, nb: int, amp: float = 0.05,
                           mesh: Optional[Mesh] = None, box=None) -> np.ndarray:
    """(1 + amp*(2u - 1)) in canonical [cell][d][b] order, u from the GLOBAL
    canonical index (c*nd + d)*nb + b; the caller multiplies by its own
    I0_b(T_c).  With mesh and box, only the sub-box cells (sub-box order)."""
    if box is None:
        u = uniform_noise(seed, ncells * nd * nb)
        return (1.0 + amp * (2.0 * u - 1.0)).reshape(ncells, nd, nb)
    (x0, x1), (y0, y1), (z0, z1) = box
    zz, yy, xx = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    cg = (xx + mesh.nx * (yy + mesh.ny * zz)).reshape(-1).astype(np.uint64)
    idx = (cg[:, None] * np.uint64(nd * nb) + np.arange(nd * nb, dtype=np.uint64)[None, :]).reshape(-1)
    z = splitmix64(np.uint64(seed & MASK64) ^ idx)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (1.0 + amp * (2.0 * u - 1.0)).reshape(cg.size, nd, nb)


def intensity_noise_factor_cells(seed: int, cells, nd: int, nb: int, amp: float = 0.05) -> np.ndarray:
    """intensity_noise_factor for an explicit list of GLOBAL canonical cells
    (e.g. a sub-mesh of an unstructured mesh), in list order."""
    cg = np.asarray(cells, dtype=np.uint64)
    idx = (cg[:, None] * np.uint64(nd * nb) + np.arange(nd * nb, dtype=np.uint64)[None, :]).reshape(-1)
    z = splitmix64(np.uint64(seed & MASK64) ^ idx)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (1.0 + amp * (2.0 * u - 1.0)).reshape(cg.size, nd, nb)


# --------------------------------------------------------------------------
# unstructured simplex meshes: a lattice of squares / cubes,
# each split into 2 triangles / 6 tetrahedra, with seeded vertex jitter.  A
# vertex coordinate along axis a is jittered only when the vertex is not on a
# wall normal to a, so walls stay planar and axis-aligned.

def _lattice_verts(n, h, jitter: float, seed: int) -> np.ndarray:
    dim = len(n)
    grids = np.meshgrid(*[np.arange(k + 1) for k in n[::-1]], indexing="ij")  # slowest axis first
    idx = [g.reshape(-1) for g in grids[::-1]]  # idx[0] = x index (fastest)
    nv = idx[0].size
    X = np.zeros((nv, 3))
    u = uniform_noise(seed, nv * dim).reshape(nv, dim) if jitter > 0 else np.zeros((nv, dim))
    for a in range(dim):
        x = idx[a] * h[a]
        interior = (idx[a] > 0) & (idx[a] < n[a])
        X[:, a] = np.where(interior, x + jitter * h[a] * (2.0 * u[:, a] - 1.0), x)
    return X


def umesh_tri(nx: int, ny: int, Lx: float, Ly: float, jitter: float = 0.2, seed: int = 11,
              shuffle: bool = False, mirror: bool = False, depth: float = 1.0) -> UMesh:
    """2-D triangulation of an nx x ny lattice of squares (2 triangles each, the
    diagonal drawn per square from the seeded noise, or mirror-symmetric about
    x = Lx/2 when mirror=True); square-major cell order unless shuffled."""
    V = _lattice_verts((nx, ny), (Lx / nx, Ly / ny), jitter, seed)
    vid = lambda i, j: i + (nx + 1) * j  # noqa: E731
    flip = uniform_noise(seed + 1, nx * ny) < 0.5
    cells = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            f = (i < nx // 2) if mirror else bool(flip[i + nx * j])
            if f:
                cells += [(a, b, c), (a, c, d)]
            else:
                cells += [(a, b, d), (b, c, d)]
    C = np.array(cells, dtype=np.int64)
    if shuffle:
        C = C[np.random.Generator(np.random.PCG64(seed + 2)).permutation(len(C))]
    return UMesh(2, V, np.ascontiguousarray(C), depth)


def umesh_quad(nx: int, ny: int, Lx: float, Ly: float, jitter: float = 0.2, seed: int = 19,
               shuffle: bool = False, depth: float = 1.0) -> UMesh:
    """2-D quadrilaterals: the nx x ny lattice of squares with jittered
    interior vertices (convex for jitter < 0.25), vertices counter-clockwise
    from the lower-left corner, row-major cell order (the structured grid's
    canonical order when jitter = 0) unless shuffled."""
    V = _lattice_verts((nx, ny), (Lx / nx, Ly / ny), jitter, seed)
    vid = lambda i, j: i + (nx + 1) * j  # noqa: E731
    C = np.array([(vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1))
                  for j in range(ny) for i in range(nx)], dtype=np.int64)
    if shuffle:
        C = C[np.random.Generator(np.random.PCG64(seed + 2)).permutation(len(C))]
    return UMesh(2, V, np.ascontiguousarray(C), depth)


# Kuhn subdivision of a cube into 6 tetrahedra along the main diagonal: for each
# axis order (p, q, r), the path 000 -> e_p -> e_p + e_q -> 111 (conforming
# across cubes because every cube uses the same split)
_KUHN = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def umesh_tet(nx: int, ny: int, nz: int, h: float = 1e-6, jitter: float = 0.1, seed: int = 13,
              shuffle: bool = False) -> UMesh:
    """3-D tetrahedral mesh: nx x ny x nz cubes of side h, 6 Kuhn tetrahedra
    each, jittered vertices; cube-major cell order unless shuffled."""
    V = _lattice_verts((nx, ny, nz), (h, h, h), jitter, seed)
    vid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)  # noqa: E731
    cells = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                for p in _KUHN:
                    o = [0, 0, 0]
                    path = [vid(i, j, k)]
                    for a in p:
                        o[a] = 1
                        path.append(vid(i + o[0], j + o[1], k + o[2]))
                    cells.append(tuple(path))
    C = np.array(cells, dtype=np.int64)
    if shuffle:
        C = C[np.random.Generator(np.random.PCG64(seed + 2)).permutation(len(C))]
    return UMesh(3, V, np.ascontiguousarray(C), 1.0)


def umesh_hex(nx: int, ny: int, nz: int, h: float = 1e-6, jitter: float = 0.1, seed: int = 23,
              shuffle: bool = False) -> UMesh:
    """3-D hexahedral mesh: the nx x ny x nz lattice of cubes of side h with
    jittered interior vertices (faces become bilinear, non-planar), vertices in
    the Gmsh order (bottom 0-1-2-3 counter-clockwise, top 4-5-6-7 above them);
    cube-major cell order unless shuffled.  jitter = 0 gives the structured grid
    in its canonical cell order."""
    V = _lattice_verts((nx, ny, nz), (h, h, h), jitter, seed)
    vid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)  # noqa: E731
    cells = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                cells.append((vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                              vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1), vid(i, j + 1, k + 1)))
    C = np.array(cells, dtype=np.int64)
    if shuffle:
        C = C[np.random.Generator(np.random.PCG64(seed + 2)).permutation(len(C))]
    return UMesh(3, V, np.ascontiguousarray(C), 1.0)


def umesh_tet_subbox(m: UMesh, n, box):
    """The cubes [x0,x1) x [y0,y1) x [z0,z1) of a umesh_tet(n[0], n[1], n[2])
    mesh (unshuffled, cube-major order) as a mesh of its own: returns (sub mesh,
    global cell ids in sub order).  Vertices on a cut plane of the box are
    moved onto the plane (their jitter along that axis dropped), so the sub
    mesh's walls are planar; only the tetrahedra of the box's outer cube layer
    change geometry (a sample k+1 cubes inside the cut is exact for k steps)."""
    nx, ny, nz = n
    (x0, x1), (y0, y1), (z0, z1) = box
    cubes = [i + nx * (j + ny * k) for k in range(z0, z1) for j in range(y0, y1) for i in range(x0, x1)]
    gcells = np.array([6 * c + t for c in cubes for t in range(6)], dtype=np.int64)
    C = m.cells[gcells]
    used, inv = np.unique(C.reshape(-1), return_inverse=True)
    V = m.verts[used].copy()
    vi = used % (nx + 1)
    vj = (used // (nx + 1)) % (ny + 1)
    vk = used // ((nx + 1) * (ny + 1))
    h = (m.verts[:, 0].max() - m.verts[:, 0].min()) / nx
    for a, (idx, lo, hi) in enumerate(((vi, x0, x1), (vj, y0, y1), (vk, z0, z1))):
        on = (idx == lo) | (idx == hi)
        V[on, a] = idx[on] * h
    sub = UMesh(3, V, np.ascontiguousarray(inv.reshape(C.shape).astype(np.int64)), m.depth)
    return sub, gcells


def umesh_centroids(m: UMesh) -> np.ndarray:
    """Cell centroids: vertex coordinates summed in local vertex order, / (dim+1)."""
    X = m.verts[m.cells]  # [nc, m, 3]
    acc = X[:, 0, :].copy()
    for k in range(1, X.shape[1]):
        acc = acc + X[:, k, :]
    return acc / X.shape[1]


def random_temperature_umesh(m: UMesh, seed: int, T_mean: float = 300.0, T_amp: float = 20.0,
                             lo=None, L=None) -> np.ndarray:
    """Random start on an unstructured mesh: the structured recipe with the cell
    centre replaced by the centroid, measured from the box corner, and L the
    box extent (a sub-mesh passes the whole mesh's corner and extent)."""
    p1, p2, p3 = random_phases(seed)
    cen = umesh_centroids(m)
    lo = m.verts.min(axis=0) if lo is None else np.asarray(lo, dtype=np.float64)
    L = (m.verts.max(axis=0) - lo) if L is None else np.asarray(L, dtype=np.float64)
    fx = np.sin(2.0 * math.pi * ((cen[:, 0] - lo[0]) / L[0] + p1))
    fy = np.sin(2.0 * math.pi * ((cen[:, 1] - lo[1]) / L[1] + p2))
    fz = np.sin(2.0 * math.pi * ((cen[:, 2] - lo[2]) / L[2] + p3)) if m.dim == 3 else np.ones(m.ncells)
    return np.ascontiguousarray(T_mean + T_amp * (fz * fy * fx))


def subproblem(problem: "Problem", box, open_kind: int = BC_SPECULAR) -> "Problem":
    """The problem restricted to a sub-box ((x0,x1),(y0,y1),(z0,z1)).  Sides on
    the domain boundary keep their wall (T_wall restricted to the box faces);
    interior ("open") sides get `open_kind` -- cells within k cells of an open
    side are wrong after k steps, all others are exact."""
    m = problem.mesh
    (x0, x1), (y0, y1), (z0, z1) = box
    sub = Mesh(m.dim, x1 - x0, y1 - y0, z1 - z0, m.dx, m.dy, m.dz)
    lo = [x0, y0, z0]
    hi = [x1, y1, z1]
    n = [m.nx, m.ny, m.nz]
    bcs = []
    for r in range(6):
        a = r // 2
        on_wall = (lo[a] == 0) if r % 2 == 0 else (hi[a] == n[a])
        bc = problem.bcs[r]
        if not on_wall:
            bcs.append(WallBC(open_kind, None, 300.0))
            continue
        Tw = None
        if bc.T_wall is not None:
            full = np.asarray(bc.T_wall)
            if a == 0:
                Tw = full.reshape(m.nz, m.ny)[z0:z1, y0:y1].reshape(-1)
            elif a == 1:
                Tw = full.reshape(m.nz, m.nx)[z0:z1, x0:x1].reshape(-1)
            else:
                Tw = full.reshape(m.ny, m.nx)[y0:y1, x0:x1].reshape(-1)
            Tw = np.ascontiguousarray(Tw)
        bcs.append(WallBC(bc.kind, Tw, bc.T_uniform))
    return Problem(problem.name + f"_sub{box}", sub, problem.dirs, problem.bands, problem.dt,
                   problem.T_init, bcs, problem.nsteps, problem.seed, problem.tau_mode, problem.semi,
                   problem.implicit, problem.imp_max_iter, problem.imp_tol)


# --------------------------------------------------------------------------
# the BASELINE.json configs; seeds 2305194000 + k

SEED_BASE = 2305194000


def config1() -> Problem:
    """2-D gray 20x20, 16 in-plane dirs, hot/cold isothermal y-walls, diffuse
    adiabatic x-walls, 100 steps (BJ configs[0])."""
    L = 2e-6
    n = 20
    d = L / n
    mesh = Mesh(2, n, n, 1, d, d, 1.0)
    bcs = [WallBC(BC_DIFFUSE), WallBC(BC_DIFFUSE),
           WallBC(BC_ISOTHERMAL, None, 300.0), WallBC(BC_ISOTHERMAL, None, 310.0),
           WallBC(BC_SPECULAR), WallBC(BC_SPECULAR)]
    return Problem("config1_2d_gray_20x20x16x1", mesh, directions_inplane(16),
                   gray_linear_bands(), dt=5e-12, T_init=300.0, bcs=bcs, nsteps=100,
                   seed=SEED_BASE + 1)


def config2(n: int = 120, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """2-D non-gray silicon 120x120 on a 525 um square, 400 dirs,
    40 channels, Gaussian hot spot on +y, 300 K on -y, specular x-walls
    (P:L413-425), dt = 1e-12 s (reading #9), 100 steps."""
    L = 525e-6
    d = L / n
    mesh = Mesh(2, n, n, 1, d, d, 1.0)
    bcs = [WallBC(BC_SPECULAR), WallBC(BC_SPECULAR),
           WallBC(BC_ISOTHERMAL, None, 300.0),
           WallBC(BC_ISOTHERMAL, hotspot_profile(n, d), 300.0),
           WallBC(BC_SPECULAR), WallBC(BC_SPECULAR)]
    return Problem(f"config2_2d_si_{n}x{n}x{n_theta*n_phi}x{len(silicon_bands(n_freq).v)}", mesh,
                   directions_control_angle(n_theta, n_phi), silicon_bands(n_freq),
                   dt=1e-12, T_init=300.0, bcs=bcs, nsteps=100, seed=SEED_BASE + 2)


def config_demo(n: int = 120, ndirs: int = 20, n_freq: int = 40) -> Problem:
    """The paper's own demonstration: 2-D 525 um square, 120x120
    cells, 20 in-plane directions, 40 frequency bands -> 55 channels (40 LA +
    15 TA), 20 x 55 = 1100 DOF per cell, ~1.6e7 DOF; Gaussian hot
    spot on +y, 300 K on -y, symmetry (specular) sides; dt = 1e-12 s (reading #9);
    100 steps."""
    p = config2(n=n, n_freq=n_freq)
    p.dirs = directions_inplane(ndirs)
    p.name = f"demo_2d_si_{n}x{n}x{ndirs}x{p.bands.nb}"
    p.seed = SEED_BASE + 6
    return p


def config_fig9(nx: int = 40, ny: int = 120, ndirs: int = 20, n_freq: int = 40) -> Problem:
    """The paper's second example (Fig. 9): "a
    smaller-scale, elongated material with a heat source in one corner ...
    symmetry conditions on the left and right, and an isothermal boundary on
    the bottom".  The figure is an image without sizes (reading R-m): 2-D,
    nx x ny cells of 1 um (40 x 120 um), the demo's 20 in-plane directions and
    55 channels, specular x-walls, 300 K on -y, and on +y a Gaussian source
    centred on the left corner, T_wall(x) = 300 + 50 exp(-2 x^2 / w^2) with x
    the face centre's distance from the corner and w = 10 um."""
    d = 1e-6
    mesh = Mesh(2, nx, ny, 1, d, d, 1.0)
    x = (np.arange(nx) + 0.5) * d
    top = 300.0 + 50.0 * np.exp(-2.0 * x * x / (10e-6 * 10e-6))
    bcs = [WallBC(BC_SPECULAR), WallBC(BC_SPECULAR), WallBC(BC_ISOTHERMAL, None, 300.0),
           WallBC(BC_ISOTHERMAL, top, 300.0), WallBC(BC_SPECULAR), WallBC(BC_SPECULAR)]
    b = silicon_bands(n_freq)
    return Problem(f"fig9_2d_si_{nx}x{ny}x{ndirs}x{b.nb}", mesh, directions_inplane(ndirs), b, dt=1e-12,
                   T_init=300.0, bcs=bcs, nsteps=100, seed=SEED_BASE + 10)


def config3(n: int = 64, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """3-D silicon box n^3, 1 um cells, z=0 isothermal 300 K, z=L 310 K, x/y specular."""
    d = 1e-6
    mesh = Mesh(3, n, n, n, d, d, d)
    bcs = [WallBC(BC_SPECULAR), WallBC(BC_SPECULAR), WallBC(BC_SPECULAR), WallBC(BC_SPECULAR),
           WallBC(BC_ISOTHERMAL, None, 300.0), WallBC(BC_ISOTHERMAL, None, 310.0)]
    return Problem(f"config3_3d_si_{n}^3x{n_theta*n_phi}x{len(silicon_bands(n_freq).v)}", mesh,
                   directions_control_angle(n_theta, n_phi), silicon_bands(n_freq),
                   dt=1e-12, T_init=300.0, bcs=bcs, nsteps=100, seed=SEED_BASE + 3)


def config4(n: int = 100) -> Problem:
    p = config3(n)
    p.name = f"config4_3d_si_{n}^3x400x40"
    p.seed = SEED_BASE + 4
    return p


def config5(nranks: int = 1, n: int = 64) -> Problem:
    """64x64x(64*P) closed specular box (weak scaling)."""
    d = 1e-6
    mesh = Mesh(3, n, n, n * nranks, d, d, d)
    return Problem(f"config5_3d_si_{n}x{n}x{n*nranks}x400x40", mesh,
                   directions_control_angle(20, 20), silicon_bands(29), dt=1e-12,
                   T_init=300.0, bcs=uniform_bcs(BC_SPECULAR), nsteps=100, seed=SEED_BASE + 5)


def small_3d(nx=5, ny=4, nz=3, dirs=None, bands=None, bcs=None, dt=1e-12, d=1e-6, seed=7) -> Problem:
    """Small 3-D case for parity tests (several tiles and a ragged tail)."""
    mesh = Mesh(3, nx, ny, nz, d, d, d)
    dirs = dirs if dirs is not None else directions_control_angle(4, 8)
    bands = bands if bands is not None else subset_bands(silicon_bands(29), [0, 5, 17, 28, 30, 39])
    if bcs is None:
        bcs = [WallBC(BC_SPECULAR), WallBC(BC_DIFFUSE), WallBC(BC_ISOTHERMAL, None, 305.0),
               WallBC(BC_SPECULAR), WallBC(BC_ISOTHERMAL, None, 300.0), WallBC(BC_DIFFUSE)]
    return Problem(f"small3d_{nx}x{ny}x{nz}", mesh, dirs, bands, dt=dt, T_init=300.0,
                   bcs=bcs, nsteps=10, seed=seed)


def config_u2(n: int = 120, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """Unstructured analogue of config 2: the 525 um square as 2 n^2
    jittered triangles, 400 directions, 40 channels, +y 310 K / -y 300 K
    isothermal walls, specular x-walls, dt = 1e-12 s."""
    L = 525e-6
    p = config2(n=n, n_freq=n_freq, n_theta=n_theta, n_phi=n_phi)
    p.mesh = umesh_tri(n, n, L, L, jitter=0.2, seed=SEED_BASE + 7)
    p.bcs[3] = WallBC(BC_ISOTHERMAL, None, 310.0)
    p.name = f"u2_tri_{2*n*n}x{n_theta*n_phi}x{p.bands.nb}"
    p.seed = SEED_BASE + 7
    return p


def config_uq(n: int = 120, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """config_u2 on jittered quadrilaterals (n^2 cells)."""
    p = config_u2(n=n, n_freq=n_freq, n_theta=n_theta, n_phi=n_phi)
    L = 525e-6
    p.mesh = umesh_quad(n, n, L, L, jitter=0.2, seed=SEED_BASE + 9)
    p.name = f"uq_quad_{n*n}x{n_theta*n_phi}x{p.bands.nb}"
    p.seed = SEED_BASE + 9
    return p


def config_u3(n: int = 32, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """Unstructured analogue of config 3: n^3 cubes of 1 um as 6 n^3 jittered
    tetrahedra, 400 directions, 40 channels, z walls 300/310 K, x/y specular."""
    p = config3(n=n, n_freq=n_freq, n_theta=n_theta, n_phi=n_phi)
    p.mesh = umesh_tet(n, n, n, 1e-6, jitter=0.1, seed=SEED_BASE + 8)
    p.name = f"u3_tet_{6*n**3}x{n_theta*n_phi}x{p.bands.nb}"
    p.seed = SEED_BASE + 8
    return p


def config_u3h(n: int = 64, n_freq: int = 29, n_theta: int = 20, n_phi: int = 20) -> Problem:
    """config 3 on jittered hexahedra (R-o): n^3 cells of 1 um with bilinear
    faces, 400 directions, 40 channels, z walls 300/310 K, x/y specular."""
    p = config3(n=n, n_freq=n_freq, n_theta=n_theta, n_phi=n_phi)
    p.mesh = umesh_hex(n, n, n, 1e-6, jitter=0.1, seed=SEED_BASE + 11)
    p.name = f"u3h_hex_{n**3}x{n_theta*n_phi}x{p.bands.nb}"
    p.seed = SEED_BASE + 11
    return p


def small_umesh(dim: int = 2, n=(4, 3, 2), dirs=None, bands=None, bcs=None, dt=1e-12, shuffle=False,
                jitter=None, seed=17, quad=False, hexa=False) -> Problem:
    """Small unstructured case for parity tests (hexa: hexahedra in 3-D)."""
    if dim == 3 and hexa:
        mesh = umesh_hex(n[0], n[1], n[2], 1e-6, 0.1 if jitter is None else jitter, seed, shuffle)
    elif dim == 2 and quad:
        mesh = umesh_quad(n[0], n[1], n[0] * 1e-6, n[1] * 1e-6, 0.2 if jitter is None else jitter, seed, shuffle)
    elif dim == 2:
        mesh = umesh_tri(n[0], n[1], n[0] * 1e-6, n[1] * 1e-6, 0.2 if jitter is None else jitter, seed, shuffle)
    elif dim == 3:
        mesh = umesh_tet(n[0], n[1], n[2], 1e-6, 0.1 if jitter is None else jitter, seed, shuffle)
    dirs = dirs if dirs is not None else directions_control_angle(4, 8)
    bands = bands if bands is not None else subset_bands(silicon_bands(29), [0, 5, 17, 28, 30, 39])
    if bcs is None:
        bcs = [WallBC(BC_SPECULAR), WallBC(BC_DIFFUSE), WallBC(BC_ISOTHERMAL, None, 305.0),
               WallBC(BC_SPECULAR), WallBC(BC_ISOTHERMAL, None, 300.0), WallBC(BC_DIFFUSE)]
    return Problem(f"small_umesh{dim}d_{mesh.ncells}", mesh, dirs, bands, dt=dt, T_init=300.0,
                   bcs=bcs, nsteps=10, seed=seed)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5, 6: config_demo, 10: config_fig9}
