"""GPU parity on unstructured simplex meshes: the CUDA path
(bte_create_umesh through the C ABI) against the CPU oracle
(oracle/bte_oracle_umesh.c) on the same seeded inputs.  Tolerances as for the
structured path (BASELINE.json north_star): max relative error 1e-10 on
intensities, 1e-8 K absolute on temperature."""
import numpy as np
import pytest

import bte_inputs as bi
import oracle
from paper_2305_19400_b200.bte import DEBUG_SKIP_EXCHANGE

pytestmark = pytest.mark.gpu

REL_I = 1e-10
ABS_T = 1e-8


@pytest.fixture(scope="module")
def Solver():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_19400_b200 import Solver as S, build
    build.build()
    return S


def _cmp(Ig, Tg, Io, To):
    return float(np.max(np.abs(Ig - Io) / np.abs(Io))), float(np.max(np.abs(Tg - To)))


def _run_both(Solver, p, nsteps, solve_T=False):
    o = oracle.Oracle(p)
    I, T = o.random_state()
    with Solver.from_problem(p) as sv:
        for r in range(2 * p.mesh.dim):
            assert sv.region_faces(r) == o.n_region_faces(r)
        if solve_T:
            sv.set_state(I, None)
            T, I0c, betac = o.solve_T(I, np.full(p.mesh.ncells, p.T_init))
            assert np.max(np.abs(sv.temperature() - T)) <= ABS_T
            Io, To, _, _ = o.run(I, T, nsteps, I0c, betac)
        else:
            sv.set_state(I, T)
            Io, To, _, _ = o.run(I, T, nsteps)
        sv.step(nsteps)
        Ig, Tg = sv.intensity(), sv.temperature()
    return _cmp(Ig, Tg, Io, To)


def _walls(p):
    o = oracle.Oracle(p)
    nf = o.n_region_faces(2)
    return [bi.WallBC(bi.BC_SPECULAR), bi.WallBC(bi.BC_DIFFUSE),
            bi.WallBC(bi.BC_ISOTHERMAL, 300.0 + 10.0 * np.linspace(0, 1, nf)),
            bi.WallBC(bi.BC_PARTIAL, specularity=0.35), bi.WallBC(bi.BC_ISOTHERMAL, None, 298.0),
            bi.WallBC(bi.BC_DIFFUSE)]


@pytest.mark.parametrize("dim,n,shuffle", [(2, (5, 4, 1), False), (2, (7, 3, 1), True), (3, (3, 2, 2), False),
                                           (3, (2, 3, 3), True)])
def test_umesh_parity_all_wall_kinds(Solver, dim, n, shuffle):
    p = bi.small_umesh(dim, n, shuffle=shuffle)
    p.bcs = _walls(p)
    rel, dT = _run_both(Solver, p, 8)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_umesh_parity_set_state_solves_T(Solver):
    p = bi.small_umesh(3, (3, 3, 2))
    rel, dT = _run_both(Solver, p, 4, solve_T=True)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


@pytest.mark.parametrize("case", ["u2", "u3"])
def test_umesh_parity_silicon_400x40_reduced(Solver, case):
    """The bench workloads' directions (400) and channels (40) on reduced meshes."""
    p = bi.config_u2(n=10) if case == "u2" else bi.config_u3(n=3)
    rel, dT = _run_both(Solver, p, 3)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_umesh_full_size_u2(Solver):
    """bench workload u2 at full size (28,800 triangles x 400 x 40), 2 steps, full field."""
    p = bi.config_u2()
    rel, dT = _run_both(Solver, p, 2)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_umesh_init_random_matches_recipe(Solver):
    p = bi.small_umesh(3, (3, 2, 2))
    o = oracle.Oracle(p)
    I, T = o.random_state()
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        Tg, Ig = sv.temperature(), sv.intensity()
    assert np.max(np.abs(Tg - T)) < 1e-10
    assert np.max(np.abs(Ig / I - 1)) < 1e-12


@pytest.mark.parametrize("kind", [bi.BC_SPECULAR, bi.BC_DIFFUSE, bi.BC_PARTIAL])
def test_umesh_closed_box_energy(Solver, kind):
    b = bi.subset_bands(bi.silicon_bands(29), [2, 19, 33])
    p = bi.small_umesh(3, (3, 3, 2), bands=b, bcs=[bi.WallBC(kind, specularity=0.6) for _ in range(6)],
                       dirs=bi.directions_control_angle(2, 8))
    I, _ = oracle.Oracle(p).random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, None)
        E0 = sv.energy()
        sv.step(200)
        E1 = sv.energy()
    assert abs(E1 / E0 - 1) < 1e-12, E1 / E0 - 1
    assert abs(E0 / oracle.Oracle(p).energy(I) - 1) < 1e-13


def test_umesh_full_size_u3_properties(Solver):
    """bench workload u3 at full size (196,608 tetrahedra x 400 x 40): closed
    specular box conserves energy; a uniform equilibrium stays fixed."""
    p = bi.config_u3()
    p.bcs = bi.uniform_bcs(bi.BC_SPECULAR)
    with Solver.from_problem(p) as sv:
        T0 = sv.temperature()
        sv.step(2)
        assert np.max(np.abs(sv.temperature() - T0)) < 1e-10
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        sv.step(1)  # afterwards (I, T) satisfy the Newton balance (conservation holds from here)
        E0 = sv.energy()
        sv.step(3)
        E1 = sv.energy()
    assert abs(E1 / E0 - 1) < 1e-12


def test_umesh_fixed_point_and_errors(Solver):
    from paper_2305_19400_b200 import BteError
    b = bi.subset_bands(bi.silicon_bands(29), [0, 20, 39])
    bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 300.0), bi.WallBC(3, specularity=0.5),
           bi.WallBC(1), bi.WallBC(0, None, 300.0)]
    p = bi.small_umesh(3, (3, 2, 2), bands=b, bcs=bcs)
    with Solver.from_problem(p) as sv:
        I0, T0 = sv.intensity(), sv.temperature()
        sv.step(20)
        assert np.max(np.abs(sv.intensity() / I0 - 1)) < 1e-14
        assert np.max(np.abs(sv.temperature() - T0)) < 1e-10
    q = bi.small_umesh(2, (3, 2, 1))
    q.dt = 1e-9  # violates the positivity bound
    with pytest.raises(BteError) as e:
        Solver.from_problem(q)
    assert e.value.status == 5
    q = bi.small_umesh(2, (3, 2, 1))
    q.mesh.cells = q.mesh.cells.copy()
    q.mesh.cells[0, 1] = q.mesh.cells[0, 0]  # degenerate triangle
    with pytest.raises(BteError) as e:
        Solver.from_problem(q)
    assert e.value.status == 1
    q = bi.small_umesh(2, (3, 2, 1))
    q.mesh.cells = q.mesh.cells[1:].copy()  # a hole: interior faces become boundary faces off the walls
    with pytest.raises(BteError) as e:
        Solver.from_problem(q)
    assert e.value.status == 1
    with pytest.raises(ValueError):  # unstructured meshes partition by cells, not channels
        Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=0, nranks=2, decomp="band")
    with pytest.raises(BteError) as e:  # more parts than cells
        Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=0, nranks=p.mesh.ncells + 1)
    assert e.value.status == 1


@pytest.mark.parametrize("dim", [2, 3])
def test_umesh_kernel_variants_bitwise(Solver, dim, monkeypatch):
    """The pipelined sweep (k_usweep_tma: TMA ring + register prefetch) is
    bitwise identical across chunk sizes and pipeline depths, and agrees with
    the one-CTA-per-cell k_usweep to rounding (the two group the face and
    direction sums differently)."""
    p = bi.config_u2(n=9) if dim == 2 else bi.config_u3(n=3)
    I, T = oracle.Oracle(p).random_state()
    out = []
    for env in ({"BTE_SWEEP": "plain"}, {}, {"BTE_SEGS": "5", "BTE_STAGES": "2"}, {"BTE_SEGS": "1000"},
                {"BTE_UGENERIC": "1"}):
        for k in ("BTE_SWEEP", "BTE_SEGS", "BTE_STAGES", "BTE_UGENERIC"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(3)
            out.append((sv.intensity(), sv.temperature()))
    for Ix, Tx in out[2:]:
        assert np.array_equal(Ix, out[1][0]) and np.array_equal(Tx, out[1][1])
    assert np.max(np.abs(out[1][0] / out[0][0] - 1)) < 1e-13
    assert np.max(np.abs(out[1][1] - out[0][1])) < 1e-10


# ----------------------------------------------------------------- quadrilaterals (Eq. 3 "polygonal cell with m sides")

@pytest.mark.parametrize("shuffle", [False, True])
def test_uquad_parity(Solver, shuffle):
    p = bi.small_umesh(2, (6, 5, 1), shuffle=shuffle, quad=True)
    p.bcs = _walls(p)
    rel, dT = _run_both(Solver, p, 8)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_uquad_silicon_and_structured_equivalence(Solver):
    """Jittered quads with the bench's 400 x 40 against the oracle; an unjittered
    row-major quad mesh on the GPU agrees with the structured GPU path."""
    p = bi.config_uq(n=10)
    rel, dT = _run_both(Solver, p, 3)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    h = 2.0 ** -19
    nx, ny = 7, 6
    b = bi.subset_bands(bi.silicon_bands(29), [1, 18, 34, 39])
    d = bi.directions_control_angle(4, 8)
    bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, 300.0 + np.arange(nx)), bi.WallBC(3, specularity=0.3),
           bi.WallBC(1), bi.WallBC(1)]
    ps = bi.Problem("grid", bi.Mesh(2, nx, ny, 1, h, h, 1.0), d, b, 1e-12, 300.0, bcs, seed=4)
    pu = bi.Problem("quads", bi.umesh_quad(nx, ny, nx * h, ny * h, jitter=0.0), d, b, 1e-12, 300.0, bcs, seed=4)
    I, T = oracle.Oracle(ps).random_state()
    out = []
    for p in (ps, pu):
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(6)
            out.append((sv.intensity(), sv.temperature()))
    assert np.max(np.abs(out[1][0] / out[0][0] - 1)) < 1e-12 and np.max(np.abs(out[1][1] - out[0][1])) < 1e-9


# ----------------------------------------------------------------- partitioned meshes (local groups)

def _part_case(case):
    if case == "tri":
        p = bi.small_umesh(2, (7, 5, 1))
    elif case == "quad":
        p = bi.small_umesh(2, (6, 5, 1), quad=True, shuffle=True)
    elif case == "hex":
        p = bi.small_umesh(3, (4, 3, 3), hexa=True, shuffle=True)
    else:
        p = bi.small_umesh(3, (3, 3, 3))
    p.bcs = _walls(p)
    return p


def _part_group(Solver, p, P, I, T, **kw):
    group = []
    for r in range(P):
        sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=P, **kw)
        group.append(sv)
        for reg in range(2 * p.mesh.dim):
            sv.set_wall(reg, p.bcs[reg])
        if I is not None:
            sv.set_state(I[sv.cell0:sv.cell0 + sv.ncells], T[sv.cell0:sv.cell0 + sv.ncells])
    return group


@pytest.mark.parametrize("case,P", [("tri", 2), ("tri", 3), ("quad", 3), ("tet", 2), ("tet", 4), ("hex", 3)])
def test_umesh_partition_group_bitexact(Solver, case, P):
    """P contexts each owning a contiguous cell range plus halo copies of the
    neighbours owned elsewhere (refreshed after every step) reproduce the
    single-context run bit for bit; the random start draws the same state."""
    p = _part_case(case)
    I, T = oracle.Oracle(p).random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(5)
        I1, T1 = sv.intensity(), sv.temperature()
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        sv.step(2)
        Ir = sv.intensity()
    group = _part_group(Solver, p, P, I, T)
    try:
        assert sum(s.ncells for s in group) == p.mesh.ncells
        Solver.group_step(group, 2)
        Solver.group_step(group, 3)
        Ig = np.concatenate([s.intensity() for s in group])
        Tg = np.concatenate([s.temperature() for s in group])
        for s in group:
            s.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        Solver.group_step(group, 2)
        Igr = np.concatenate([s.intensity() for s in group])
    finally:
        for s in group:
            s.close()
    assert np.array_equal(Ig, I1) and np.array_equal(Tg, T1)
    assert np.array_equal(Igr, Ir)


def test_umesh_partition_semi_and_mutation(Solver, monkeypatch):
    p = _semi_umesh = _part_case("tet")
    p.dt = 8 * p.dt
    p.semi = 1
    I, T = oracle.Oracle(p).random_state()
    Io, To, _, _ = oracle.Oracle(p).run(I, T, 4)
    group = _part_group(Solver, p, 3, I, T, step_mode=1)
    try:
        Solver.group_step(group, 4)
        Ig = np.concatenate([s.intensity() for s in group])
        Tg = np.concatenate([s.temperature() for s in group])
    finally:
        for s in group:
            s.close()
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    group = _part_group(Solver, p, 3, I, T, step_mode=1)
    group[0].set_debug(DEBUG_SKIP_EXCHANGE, 1)  # without the halo refresh the result must differ
    try:
        Solver.group_step(group, 4)
        Ig2 = np.concatenate([s.intensity() for s in group])
    finally:
        for s in group:
            s.close()
    assert np.max(np.abs(Ig2 / Io - 1)) > 1e3 * REL_I


def test_umesh_full_size_u3_sampled(Solver):
    """u3 at full size (196,608 tetrahedra x 400 x 40, the bench workload),
    device random start, 3 steps, against the oracle at sampled cells: each
    sample's 3-step domain of dependence (cubes within 3, plus one layer) is
    cut out as a mesh of its own and run by the oracle with the same global
    random start (centroids from the whole box, noise from global indices)."""
    p = bi.config_u3()
    n = (32, 32, 32)
    k = 3
    samples = [(0, 0, 0, 0), (31, 31, 31, 5), (16, 9, 0, 3), (4, 31, 20, 1), (15, 16, 17, 2), (31, 0, 30, 4),
               (7, 22, 11, 5), (0, 15, 31, 0)]
    gids = [6 * (x + 32 * (y + 32 * z)) + t for (x, y, z, t) in samples]
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        sv.step(k)
        Tg = sv.temperature()
        Is = sv.intensity_cells(gids)
    m = p.mesh
    lo = m.verts.min(axis=0)
    L = m.verts.max(axis=0) - lo
    worst_rel, worst_T = 0.0, 0.0
    for si, (x, y, z, t) in enumerate(samples):
        box = [(max(0, c - k - 1), min(32, c + k + 2)) for c in (x, y, z)]
        sub, gcells = bi.umesh_tet_subbox(m, n, box)
        bcs = []
        for r in range(6):
            a = r // 2
            on_wall = box[a][0] == 0 if r % 2 == 0 else box[a][1] == n[a]
            bcs.append(p.bcs[r] if on_wall else bi.WallBC(bi.BC_SPECULAR))
        sp = bi.Problem(p.name + f"_sub{si}", sub, p.dirs, p.bands, p.dt, p.T_init, bcs, p.nsteps, p.seed)
        o = oracle.Oracle(sp)
        T0 = bi.random_temperature_umesh(sub, p.seed, p.T_init, 20.0, lo=lo, L=L)
        I0 = o.equilibrium(T0) * bi.intensity_noise_factor_cells(p.seed, gcells, p.dirs.nd, p.bands.nb, 0.05)
        Io, To, _, _ = o.run(I0, T0, k)
        lc = int(np.nonzero(gcells == gids[si])[0][0])
        worst_T = max(worst_T, abs(Tg[gids[si]] - To[lc]))
        worst_rel = max(worst_rel, float(np.max(np.abs(Is[si] - Io[lc]) / np.abs(Io[lc]))))
    assert worst_rel <= REL_I and worst_T <= ABS_T, (worst_rel, worst_T)


# ----------------------------------------------------------------- mesh import and RCB partition

@pytest.mark.parametrize("kind", ["tet", "quad", "hex"])
def test_imported_mesh_parity(Solver, tmp_path, kind):
    """A mesh read from a Gmsh file (bte_mesh_read) runs on the GPU
    and matches the oracle run on the generator's arrays."""
    import test_mesh_io as tio
    from paper_2305_19400_b200 import read_mesh
    if kind == "tet":
        p = bi.small_umesh(3, (3, 3, 2), shuffle=True)
    elif kind == "hex":
        p = bi.small_umesh(3, (3, 3, 2), hexa=True, shuffle=True)
    else:
        p = bi.small_umesh(2, (5, 4, 1), quad=True)
    path = str(tmp_path / "m.msh")
    tio._gmsh41(path, p.mesh)
    m = read_mesh(path, depth=p.mesh.depth)
    q = bi.Problem(p.name + "_imported", m, p.dirs, p.bands, p.dt, p.T_init, p.bcs, p.nsteps, p.seed)
    o = oracle.Oracle(p)  # the generator's mesh
    I, T = o.random_state()
    Io, To, _, _ = o.run(I, T, 4)
    with Solver.from_problem(q) as sv:
        sv.set_state(I, T)
        sv.step(4)
        rel, dT = _cmp(sv.intensity(), sv.temperature(), Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


@pytest.mark.parametrize("kind,P", [("tri", 3), ("tet", 4)])
def test_rcb_partitioned_group_parity(Solver, kind, P):
    """A randomly ordered mesh reordered by bte_partition_rcb, then split over
    P contexts (the cell-range partition now follows the RCB parts): the
    gathered result matches the oracle on the reordered mesh."""
    from paper_2305_19400_b200 import partition_rcb
    if kind == "tri":
        p = bi.small_umesh(2, (9, 7, 1), shuffle=True)
    else:
        p = bi.small_umesh(3, (4, 4, 3), shuffle=True)
    perm = partition_rcb(p.mesh, P)
    p.mesh = bi.UMesh(p.mesh.dim, p.mesh.verts, np.ascontiguousarray(p.mesh.cells[perm]), p.mesh.depth)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    Io, To, _, _ = o.run(I, T, 4)
    group = _part_group(Solver, p, P, I, T)
    try:
        Solver.group_step(group, 4)
        Ig = np.concatenate([s.intensity() for s in group])
        Tg = np.concatenate([s.temperature() for s in group])
    finally:
        for s in group:
            s.close()
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


# ----------------------------------------------------------------- hexahedra (Eq. 3 for polyhedra)

@pytest.mark.parametrize("shuffle", [False, True])
def test_hex_parity_all_wall_kinds(Solver, shuffle):
    """Jittered hexahedra (bilinear, non-planar faces) against the oracle, every wall kind."""
    p = bi.small_umesh(3, (4, 3, 3), hexa=True, shuffle=shuffle)
    p.bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(3, specularity=0.4),
             bi.WallBC(0, None, 298.0), bi.WallBC(2)]
    rel, dT = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_hex_silicon_400x40_and_structured_equivalence(Solver):
    """Hexahedra with the BASELINE 400 x 40 tables against the oracle; an
    unjittered hexahedral mesh reproduces the structured-grid GPU run to
    rounding (two different kernels and geometries)."""
    p = bi.config3(n=6)
    p.mesh = bi.umesh_hex(6, 5, 4, 1e-6, jitter=0.1, seed=31, shuffle=True)
    rel, dT = _run_both(Solver, p, 3)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    g = bi.config3(n=6)
    g.mesh = bi.Mesh(3, 6, 5, 4, 1e-6, 1e-6, 1e-6)
    h = bi.config3(n=6)
    h.mesh = bi.umesh_hex(6, 5, 4, 1e-6, jitter=0.0)
    I, T = oracle.Oracle(g).random_state()
    out = []
    for q in (g, h):
        with Solver.from_problem(q) as sv:
            sv.set_state(I, T)
            sv.step(4)
            out.append((sv.intensity(), sv.temperature()))
    assert np.max(np.abs(out[1][0] / out[0][0] - 1)) < 1e-12 and np.max(np.abs(out[1][1] - out[0][1])) < 1e-9
