"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerance (BASELINE.json north_star): max relative error
1e-10 on intensities and 1e-8 K absolute on temperature after the run.

Sizes: small cases span several CTAs per axis and a ragged tail; the full
BASELINE.json sizes (config 2 at 120x120x400x40 and config 3 at 64^3x400x40)
are checked on sampled cells whose k-step domain of dependence the oracle
recomputes exactly on a sub-box (explicit upwind stencil: a cell after k
steps depends only on cells within k of it), plus invariants that hold at any
size (fixed point, energy conservation, mirror symmetry, determinism)."""
import math

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
    rel = float(np.max(np.abs(Ig - Io) / np.abs(Io)))
    dT = float(np.max(np.abs(Tg - To)))
    return rel, dT


def _assert_oracle(p, I, T, nsteps, Ig, Tg):
    """A multi-rank (gathered) result against the oracle's single-domain run
    of the same problem and start (north_star tolerance)."""
    Io, To, _, _ = oracle.Oracle(p).run(I, T, nsteps)
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def _run_both(Solver, p, nsteps, start="random", solve_T=False):
    o = oracle.Oracle(p)
    if start == "random":
        I, T = o.random_state()
    else:
        T = np.full(p.mesh.ncells, p.T_init)
        I = o.equilibrium(T)
    with Solver.from_problem(p) as sv:
        if solve_T:
            sv.set_state(I, None)
            T, I0c, betac = o.solve_T(I, np.full(p.mesh.ncells, p.T_init))
            Tg0 = sv.temperature()
            assert np.max(np.abs(Tg0 - T)) <= ABS_T
            Io, To, _, _ = o.run(I, T, nsteps, I0c, betac)
        else:
            sv.set_state(I, T)
            Io, To, _, _ = o.run(I, T, nsteps)
        sv.step(nsteps)
        Ig, Tg = sv.intensity(), sv.temperature()
    return _cmp(Ig, Tg, Io, To), (Ig, Tg, Io, To)


# ----------------------------------------------------------------- small full-field parity

@pytest.mark.parametrize("shape", [(5, 4, 3), (7, 3, 6), (1, 1, 5), (9, 8, 2)])
def test_parity_small_3d_all_bc_kinds(Solver, shape):
    p = bi.small_3d(*shape)
    (rel, dT), _ = _run_both(Solver, p, 10)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_config1_full(Solver):
    """BASELINE configs[0]: 2-D gray 20x20x16x1, hot/cold walls, diffuse sides, 100 steps."""
    p = bi.config1()
    (rel, dT), (Ig, Tg, Io, To) = _run_both(Solver, p, p.nsteps, start="physical")
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    assert To.max() > 300.5  # heat entered from the 310 K wall


def test_parity_config2_reduced_physical(Solver):
    """Config 2 geometry (hot spot, specular sides) on 24x24 with the full 400 x 40 tables."""
    p = bi.config2(n=24)
    p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(24, p.mesh.dx, width=40e-6), 300.0)
    (rel, dT), (Ig, Tg, Io, To) = _run_both(Solver, p, 100, start="physical")
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    assert To.max() > 300.0


def test_parity_config2_reduced_random(Solver):
    p = bi.config2(n=16)
    (rel, dT), _ = _run_both(Solver, p, 20)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_config3_reduced(Solver):
    p = bi.config3(n=8)
    p.mesh = bi.Mesh(3, 9, 7, 6, 1e-6, 1e-6, 1e-6)
    (rel, dT), _ = _run_both(Solver, p, 5)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_inplane_3d_mesh_55_channels(Solver):
    """In-plane direction set on a 3-D mesh (4 populated octants), 55 channels (n_freq = 40)."""
    p = bi.small_3d(6, 5, 3, dirs=bi.directions_inplane(20), bands=bi.silicon_bands(40),
                    bcs=[bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 303.0), bi.WallBC(1),
                         bi.WallBC(1), bi.WallBC(1)])
    (rel, dT), _ = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_set_state_solves_T(Solver):
    p = bi.small_3d(5, 4, 3)
    (rel, dT), _ = _run_both(Solver, p, 4, solve_T=True)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_linear_multichannel(Solver):
    rng = np.random.default_rng(3)
    nb = 3
    bands = bi.linear_bands(rng.uniform(2e3, 8e3, nb), rng.uniform(2e-11, 8e-11, nb),
                            rng.uniform(1e2, 1e3, nb), rng.uniform(1e4, 1e5, nb))
    p = bi.small_3d(6, 5, 4, bands=bands, dirs=bi.directions_control_angle(4, 8), dt=2e-12, d=1e-7)
    (rel, dT), _ = _run_both(Solver, p, 30)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


# ----------------------------------------------------------------- kernel units (sub-steps)

def test_substep_sweep_and_reduce(Solver):
    p = bi.small_3d(7, 5, 4)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    I0c, betac = o.refresh(T)
    J = o.sweep(I, I0c, betac)
    D = o.reduce(J, I0c)
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        I0g, bg = sv.debug_substep(2), sv.debug_substep(3)
        assert np.max(np.abs(I0g / I0c - 1)) < 1e-13
        assert np.max(np.abs(bg / betac - 1)) < 1e-14
        Jg = sv.debug_substep(0)
        Dg = sv.debug_substep(1)
        # state unchanged by the sub-step calls
        assert np.array_equal(sv.intensity(), I)
    assert np.max(np.abs(Jg / J - 1)) < 1e-13
    scale = np.abs(p.dirs.w[None, :, None] * (I0c[:, None, :] - J)).sum(1)
    assert np.max(np.abs(Dg - D) / scale) < 1e-13


def test_init_random_matches_recipe(Solver):
    p = bi.small_3d(6, 5, 4)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        Ig, Tg = sv.intensity(), sv.temperature()
    assert np.max(np.abs(Tg - T)) < 1e-11
    assert np.max(np.abs(Ig / I - 1)) < 1e-13


# ----------------------------------------------------------------- full BASELINE sizes, sampled

def _sampled_full_size(Solver, p, nsteps, samples):
    """Run the full problem on the GPU (device-generated random start); for each
    sample cell recompute its nsteps-step dependence box with the oracle."""
    m = p.mesh
    gcs = [x + m.nx * (y + m.ny * z) for (x, y, z) in samples]
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        sv.step(nsteps)
        Tg = sv.temperature()
        Is = sv.intensity_cells(gcs)  # sampled rows (the full state may not fit the host)
        rotated = sv.rotate
    worst_rel, worst_T = 0.0, 0.0
    k = nsteps
    for (x, y, z) in samples:
        box = [(max(0, x - k), min(m.nx, x + k + 1)), (max(0, y - k), min(m.ny, y + k + 1)),
               (max(0, z - k), min(m.nz, z + k + 1))]
        sp = bi.subproblem(p, box)
        o = oracle.Oracle(sp)
        T0 = bi.random_temperature(m, p.seed, p.T_init, 20.0, box=box)
        I0 = o.equilibrium(T0) * bi.intensity_noise_factor(p.seed, 0, p.dirs.nd, p.bands.nb, 0.05, mesh=m,
                                                           box=box)
        Io, To, _, _ = o.run(I0, T0, nsteps)
        sm = sp.mesh
        lc = (x - box[0][0]) + sm.nx * ((y - box[1][0]) + sm.ny * (z - box[2][0]))
        gc = x + m.nx * (y + m.ny * z)
        worst_T = max(worst_T, abs(Tg[gc] - To[lc]))
        worst_rel = max(worst_rel, float(np.max(np.abs(Is[gcs.index(gc)] - Io[lc]) / np.abs(Io[lc]))))
    _sampled_full_size.rotated = rotated
    return worst_rel, worst_T


def test_full_size_config2_sampled(Solver):
    """BASELINE configs[1] at full size (the bench workload), 3 steps, sampled cells incl. walls."""
    p = bi.config2()
    n = p.mesh.nx
    samples = [(0, 0, 0), (n - 1, n - 1, 0), (n // 2, n - 1, 0), (n // 2 - 1, n - 2, 0), (37, 61, 0),
               (n - 1, 5, 0), (0, n // 2, 0)]
    rel, dT = _sampled_full_size(Solver, p, 3, samples)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_full_size_config3_sampled(Solver):
    """BASELINE configs[2] at full size (64^3 x 400 x 40, 33.6 GB/buffer), 2 steps, sampled T."""
    p = bi.config3()
    n = p.mesh.nx
    samples = [(0, 0, 0), (n - 1, n - 1, n - 1), (31, 17, 0), (5, n - 1, 40), (32, 32, 32), (n - 1, 0, n - 2)]
    rel, dT = _sampled_full_size(Solver, p, 2, samples)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_full_size_config3_sampled_5_steps(Solver):
    """BASELINE configs[2] at full size, 5 steps, 36 sampled cells (I and T):
    every wall and edge, and the planes on both sides of each z-segment
    boundary of the sweep (segments restart their march-axis upwind value)."""
    p = bi.config3()
    n = p.mesh.nx
    rng = np.random.Generator(np.random.PCG64(2305194003))
    zs = [0, 1, 15, 16, 17, 31, 32, 33, 47, 48, 62, 63]
    samples = []
    for i, z in enumerate(zs):
        samples.append((int(rng.integers(0, n)), int(rng.integers(0, n)), z))
        edge = [(0, int(rng.integers(0, n))), (n - 1, int(rng.integers(0, n))), (int(rng.integers(0, n)), 0),
                (int(rng.integers(0, n)), n - 1)][i % 4]
        samples.append((edge[0], edge[1], z))
        samples.append(((0, n - 1)[i % 2], (n - 1, 0)[(i // 2) % 2], z))  # x/y corners (two walls)
    assert len(samples) >= 32
    rel, dT = _sampled_full_size(Solver, p, 5, samples)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_full_size_config4_sampled(Solver):
    """BASELINE configs[3] (100^3 x 400 x 40, 128 GB per state) on one GPU as
    bench.py runs it (octant-slot rotation), 2 steps, sampled cells incl. corners
    and walls: intensities and temperature."""
    import torch
    torch.cuda.empty_cache()
    p = bi.config4()
    n = p.mesh.nx
    samples = [(0, 0, 0), (n - 1, n - 1, n - 1), (50, 17, 0), (3, n - 1, 61), (49, 50, 51), (n - 1, 0, n - 2)]
    rel, dT = _sampled_full_size(Solver, p, 2, samples)
    assert _sampled_full_size.rotated
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_full_size_config5_sampled(Solver):
    """BASELINE configs[4] at one GPU (64^3 closed specular box), 2 steps, sampled cells."""
    import torch
    torch.cuda.empty_cache()
    p = bi.config5(1)
    n = p.mesh.nx
    samples = [(0, 0, 0), (n - 1, n - 1, n - 1), (0, 33, n - 1), (40, 0, 7)]
    rel, dT = _sampled_full_size(Solver, p, 2, samples)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


# ----------------------------------------------------------------- invariants

def test_fixed_point_bitexact(Solver):
    b = bi.subset_bands(bi.silicon_bands(29), [0, 10, 20, 30, 39])
    bcs = [bi.WallBC(1), bi.WallBC(1), bi.WallBC(0, None, 300.0), bi.WallBC(1), bi.WallBC(0, None, 300.0),
           bi.WallBC(1)]
    p = bi.small_3d(8, 6, 5, bands=b, bcs=bcs)
    with Solver.from_problem(p) as sv:
        I0 = sv.intensity()
        T0 = sv.temperature()
        sv.step(50)
        assert np.array_equal(sv.intensity(), I0)
        assert np.array_equal(sv.temperature(), T0)


@pytest.mark.parametrize("kind", [bi.BC_SPECULAR, bi.BC_DIFFUSE])
def test_energy_conservation_closed_box(Solver, kind):
    b = bi.subset_bands(bi.silicon_bands(29), [2, 19, 33])
    p = bi.small_3d(6, 5, 4, bands=b, bcs=bi.uniform_bcs(kind), dirs=bi.directions_control_angle(4, 16))
    o = oracle.Oracle(p)
    I, _ = o.random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, None)  # consistent T from the Newton
        E0 = sv.energy()
        sv.step(300)
        E1 = sv.energy()
    assert abs(E1 / E0 - 1) < 1e-12, E1 / E0 - 1


def test_mirror_symmetry_bitexact(Solver):
    b = bi.subset_bands(bi.silicon_bands(29), [0, 15, 35])
    p = bi.config2(n=12)
    p.bands = b
    p.mesh = bi.Mesh(2, 12, 12, 1, 2e-6, 2e-6, 1.0)
    p.dirs = bi.directions_control_angle(4, 8)
    p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, 2e-6, width=4e-6), 300.0)
    with Solver.from_problem(p) as sv:
        sv.step(40)
        I, T = sv.intensity(), sv.temperature()
    r = oracle.Oracle(p).reflection(0)
    A = I.reshape(12, 12, p.dirs.nd, b.nb)
    assert np.array_equal(A, A[:, ::-1][:, :, r, :])
    assert np.array_equal(T.reshape(12, 12), T.reshape(12, 12)[:, ::-1])
    assert T.max() > 300.0


def test_determinism(Solver):
    p = bi.small_3d(8, 7, 6)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    out = []
    for _ in range(2):
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(7)
            out.append((sv.intensity(), sv.temperature()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


# ----------------------------------------------------------------- error paths

def test_errors(Solver):
    from paper_2305_19400_b200 import BteError
    p = bi.small_3d()
    p.dt = 1e-10  # violates the positivity bound
    with pytest.raises(BteError) as e:
        Solver.from_problem(p)
    assert e.value.status == 5
    p = bi.small_3d()
    with Solver.from_problem(p) as sv:
        I = sv.intensity()
        I[3, 2, 1] = np.nan
        T = sv.temperature()
        sv.set_state(I, T)
        with pytest.raises(BteError) as e:
            sv.step(2)
        assert e.value.status == 8 and "step 0" in str(e.value)
        with pytest.raises(ValueError):
            sv.set_state(I[:-1], T)
        with pytest.raises(BteError) as e:
            sv.set_bc(7, 0)
        assert e.value.status == 1
    # specular wall with a direction set not closed under the reflection
    d = bi.directions_control_angle(4, 8)
    d.s = d.s.copy()
    d.s[0, 0] += 1e-9
    p = bi.small_3d(dirs=d, bcs=bi.uniform_bcs(bi.BC_DIFFUSE))
    with Solver.from_problem(p) as sv:
        with pytest.raises(BteError) as e:
            sv.set_bc(0, bi.BC_SPECULAR)
        assert e.value.status == 6


def test_full_size_config2_physical_100_steps(Solver):
    """The paper's own scenario at BASELINE.json configs[1] size: equilibrium at
    300 K, Gaussian hot spot on +y, cold -y wall, specular sides, 100 steps
    (P:L413-436); full-field comparison against the oracle (~1.5 min on 16 cores)."""
    p = bi.config2()
    o = oracle.Oracle(p)
    T = np.full(p.mesh.ncells, p.T_init)
    I = o.equilibrium(T)
    Io, To, _, _ = o.run(I, T, p.nsteps)
    with Solver.from_problem(p) as sv:
        sv.step(p.nsteps)
        Ig, Tg = sv.intensity(), sv.temperature()
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    assert To.max() > 300.0 and To.min() == 300.0
    # heat enters only from the hot +y wall: the excess decays away from it
    dT_rows = np.abs(To.reshape(p.mesh.ny, p.mesh.nx) - 300.0).max(axis=1)
    assert dT_rows.argmax() == p.mesh.ny - 1
    assert np.all(np.diff(dT_rows[-20:]) >= 0)


@pytest.mark.parametrize("seed", range(10))
def test_parity_randomized_problems(Solver, seed):
    """Seeded random small problems: dimension, extents (incl. 1-cell axes),
    per-wall BC kinds, direction set, channel table and step count."""
    rng = np.random.default_rng(1000 + seed)
    dim = int(rng.choice([2, 3]))
    nx, ny = int(rng.integers(1, 8)), int(rng.integers(1, 8))
    nz = int(rng.integers(1, 6)) if dim == 3 else 1
    d = float(rng.choice([1e-6, 2e-6]))
    dirs = [bi.directions_control_angle(2, 4), bi.directions_control_angle(4, 8), bi.directions_inplane(8),
            bi.directions_inplane(12)][int(rng.integers(0, 4))]
    if rng.random() < 0.7:
        si = bi.silicon_bands(29)
        bands = bi.subset_bands(si, np.sort(rng.choice(si.nb, int(rng.integers(1, 7)), replace=False)))
    else:
        nb = int(rng.integers(1, 4))
        bands = bi.linear_bands(rng.uniform(2e3, 8e3, nb), rng.uniform(2e-11, 8e-11, nb),
                                rng.uniform(1e2, 1e3, nb), rng.uniform(1e4, 1e5, nb))
    bcs = []
    for r in range(6):
        k = int(rng.integers(0, 3))
        if k == 0:
            bcs.append(bi.WallBC(0, None, float(rng.uniform(295, 310))))
        else:
            bcs.append(bi.WallBC(k))
    p = bi.small_3d(nx, ny, nz, dirs=dirs, bands=bands, bcs=bcs, d=d, dt=1e-12 if d == 1e-6 else 2e-12,
                    seed=seed)
    if dim == 2:
        p.mesh = bi.Mesh(2, nx, ny, 1, d, d, 1.0)
    (rel, dT), _ = _run_both(Solver, p, int(rng.integers(2, 9)))
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_step_splitting_and_energy(Solver):
    """bte_step(3)+bte_step(4) == bte_step(7) bit-for-bit; the energy diagnostic
    matches the oracle's sum_c V sum_b (1/v_b) sum_d w_d I."""
    p = bi.small_3d(7, 6, 5)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(3)
        sv.step(4)
        a = (sv.intensity(), sv.temperature())
        E = sv.energy()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(7)
        b = (sv.intensity(), sv.temperature())
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert abs(E / o.energy(a[0]) - 1) < 1e-13


def test_newton_failure_is_reported(Solver):
    """No root in the [1, 5000] K bracket -> BTE_ENEWTON with the step index (the oracle agrees)."""
    from paper_2305_19400_b200 import BteError
    p = bi.small_3d(3, 2, 2, bcs=bi.uniform_bcs(bi.BC_SPECULAR))
    o = oracle.Oracle(p)
    T = np.full(p.mesh.ncells, 300.0)
    I = o.equilibrium(T) * 1e8
    with pytest.raises(oracle.OracleError) as eo:
        o.run(I, T, 1)
    assert eo.value.code == 7
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        with pytest.raises(BteError) as e:
            sv.step(1)
        assert e.value.status == 7 and "step 0" in str(e.value)


def _group_case(case):
    if case == "3d":
        b = bi.subset_bands(bi.silicon_bands(29), [0, 17, 33, 39])
        bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(1), bi.WallBC(2),
               bi.WallBC(0, None, 302.0)]
        return bi.small_3d(6, 5, 9, bands=b, bcs=bcs)
    p = bi.config2(n=10)
    p.mesh = bi.Mesh(2, 10, 13, 1, 2e-6, 2e-6, 1.0)
    p.bands = bi.subset_bands(bi.silicon_bands(29), [3, 22, 30])
    p.dirs = bi.directions_control_angle(4, 8)
    p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(10, 2e-6, width=4e-6), 300.0)
    return p


@pytest.mark.parametrize("case", ["3d", "2d"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("overlap", ["1", "0"])
def test_local_slab_group_matches_single_domain(Solver, case, P, overlap, monkeypatch):
    """Multi-rank data path on one GPU: P slab contexts (halo planes, walls only
    on the end ranks, bte_plan_slab exchange by device copies) reproduce the
    single-context run bit-for-bit (per-DOF arithmetic is partition-free)."""
    monkeypatch.setenv("BTE_OVERLAP", overlap)  # boundary planes first + exchange on the comm stream
    p = _group_case(case)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    nsteps = 7
    Io, To, _, _ = o.run(I, T, nsteps)
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(nsteps)
        I1, T1 = sv.intensity(), sv.temperature()
    group = []
    try:
        for r in range(P):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=P)
            for reg in range(6 if p.mesh.dim == 3 else 4):
                bc = p.bcs[reg]
                sv.set_wall(reg, bc)
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
            group.append(sv)
        Solver.group_step(group, 3)
        Solver.group_step(group, nsteps - 3)
        Ig = np.concatenate([sv.intensity() for sv in group])
        Tg = np.concatenate([sv.temperature() for sv in group])
    finally:
        for sv in group:
            sv.close()
    rel, dT = _cmp(Ig, Tg, Io, To)  # the multi-rank result against the oracle (north_star tolerance)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    assert np.array_equal(Ig, I1) and np.array_equal(Tg, T1)


def test_local_slab_group_mutation_skip_halo(Solver, monkeypatch):
    """Mutation: without the halo copies the slab group must differ."""
    p = _group_case("3d")
    o = oracle.Oracle(p)
    I, T = o.random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(4)
        I1 = sv.intensity()
    group = []
    try:
        for r in range(2):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=2)
            sv.set_debug(DEBUG_SKIP_EXCHANGE, 1)
            for reg in range(6):
                bc = p.bcs[reg]
                sv.set_wall(reg, bc)
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
            group.append(sv)
        Solver.group_step(group, 4)
        Ig = np.concatenate([sv.intensity() for sv in group])
    finally:
        for sv in group:
            sv.close()
    assert not np.array_equal(Ig, I1)


@pytest.mark.parametrize("start,nsteps", [("physical", 100), ("random", 20)])
def test_demo_workload_full_size(Solver, start, nsteps):
    """The paper's own demo at full size: 120x120 cells,
    20 in-plane directions, 55 channels (odd (cell, quadrant) block: 5 x 55
    doubles -> padded even stride), full-field parity."""
    p = bi.config_demo()
    (rel, dT), (Ig, Tg, Io, To) = _run_both(Solver, p, nsteps, start=start)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_parity_nonuniform_band_grid(Solver):
    """Channels whose edges are not on one uniform grid take the direct expm1
    Newton path (reading R-d); also a Debye (c2 = 0) table."""
    si = bi.subset_bands(bi.silicon_bands(29), [0, 9, 20, 31])
    si.w_hi = si.w_hi * (1.0 + 1e-3 * np.arange(1, si.nb + 1))  # break the uniform grid
    p = bi.small_3d(6, 5, 4, bands=si)
    (rel, dT), _ = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    deb = bi.debye_bands(6000.0, 2 * math.pi / 5.43e-10, 5)
    p = bi.small_3d(5, 4, 3, bands=deb, dt=1e-12)
    (rel, dT), _ = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


@pytest.mark.parametrize("variant", ["BTE_SWEEP_PLAIN", "BTE_SPARE"])
def test_parity_kernel_variants(Solver, variant, monkeypatch):
    """The A/B kernel variants (direct-load sweep for large blocks, side jobs
    on the compute threads) reach the same results."""
    if variant == "BTE_SWEEP_PLAIN":
        monkeypatch.setenv("BTE_SWEEP", "plain")
    else:
        monkeypatch.setenv("BTE_SPARE", "0")
    for p, n in ((bi.config2(n=16), 8), (bi.config3(n=8), 4)):
        if p.mesh.dim == 3:
            p.mesh = bi.Mesh(3, 9, 7, 6, 1e-6, 1e-6, 1e-6)
        (rel, dT), _ = _run_both(Solver, p, n)
        assert rel <= REL_I and dT <= ABS_T, (variant, p.name, rel, dT)


# ----------------------------------------------------------------- band partition

def _band_group(Solver, p, P, I, T):
    """P band contexts (bte_create_band, local mode) of problem p holding the
    channel slices of the state (I, T)."""
    group = []
    for r in range(P):
        sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=P, decomp="band")
        group.append(sv)
        for reg in range(6 if p.mesh.dim == 3 else 4):
            bc = p.bcs[reg]
            sv.set_wall(reg, bc)
        sv.set_state(np.ascontiguousarray(I[:, :, sv.b0:sv.b1]), T)
    return group


def _band_cases():
    si = bi.config2(n=12)
    si.mesh = bi.Mesh(2, 12, 11, 1, 2e-6, 2e-6, 1.0)
    si.dirs = bi.directions_control_angle(4, 8)
    si.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, 2e-6, width=4e-6), 300.0)
    return {"3d": _group_case("3d"), "2d": _group_case("2d"), "si40": si}


@pytest.mark.parametrize("case,P", [("3d", 2), ("3d", 3), ("2d", 3), ("si40", 3), ("si40", 8), ("si40", 1)])
def test_band_group_matches_oracle(Solver, case, P):
    """Band partition on one GPU: P contexts each sweep their channels [b0, b1),
    exchange one partial per cell, and run the same Newton over all channels.
    Union of slices and T match the oracle; T is bitwise identical on every
    part; the result matches the single-context GPU run to rounding."""
    p = _band_cases()[case]
    o = oracle.Oracle(p)
    I, T = o.random_state()
    nsteps = 6
    Io, To, _, _ = o.run(I, T, nsteps)
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(nsteps)
        I1, T1 = sv.intensity(), sv.temperature()
    group = _band_group(Solver, p, P, I, T)
    try:
        assert [(sv.b0, sv.b1) for sv in group][-1][1] == p.bands.nb
        Solver.group_step(group, 2)
        Solver.group_step(group, nsteps - 2)
        Ig = np.concatenate([sv.intensity() for sv in group], axis=2)
        Ts = [sv.temperature() for sv in group]
    finally:
        for sv in group:
            sv.close()
    assert all(np.array_equal(t, Ts[0]) for t in Ts)
    rel, dT = _cmp(Ig, Ts[0], Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    assert np.max(np.abs(Ts[0] - T1)) <= 1e-10 and np.max(np.abs(Ig / I1 - 1)) <= 1e-12


def test_band_group_mutation_skip_exchange(Solver, monkeypatch):
    """Mutation: without the partial exchange each part's Newton sees
    only its own channels' reduction, and T leaves the oracle's tolerance."""
    p = _band_cases()["si40"]
    o = oracle.Oracle(p)
    I, T = o.random_state()
    Io, To, _, _ = o.run(I, T, 3)
    group = _band_group(Solver, p, 2, I, T)
    group[0].set_debug(DEBUG_SKIP_EXCHANGE, 1)
    try:
        Solver.group_step(group, 3)
        Tg = group[0].temperature()
    finally:
        for sv in group:
            sv.close()
    assert np.max(np.abs(Tg - To)) > 1e3 * ABS_T


def test_band_init_random_and_tables(Solver):
    """Band contexts draw the single-domain random start (global channel index
    in the counter) and hold all channels' I0c / beta rows."""
    p = _band_cases()["si40"]
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        I1, T1 = sv.intensity(), sv.temperature()
        I0c1, b1 = sv.debug_substep(2), sv.debug_substep(3)
    group = []
    try:
        for r in range(3):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=3, decomp="band")
            group.append(sv)
            sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
            assert np.array_equal(sv.intensity(), I1[:, :, sv.b0:sv.b1])
            assert np.array_equal(sv.temperature(), T1)
            assert np.array_equal(sv.debug_substep(2), I0c1) and np.array_equal(sv.debug_substep(3), b1)
        with pytest.raises(Exception):
            group[0].set_state(I1[:, :, group[0].b0:group[0].b1], None)  # band contexts need T
        with pytest.raises(Exception):
            group[0].step(1)  # local-mode parts advance only through group_step
    finally:
        for sv in group:
            sv.close()


# ----------------------------------------------------------------- octant-slot rotation

@pytest.mark.parametrize("case", ["small3d", "3d", "2d"])
def test_slot_rotation_bit_exact(Solver, case, monkeypatch):
    """One buffer of nslot + 1 regions (each octant swept into the spare region,
    specular ghosts snapshotted first) gives the two-buffer result bit for bit;
    state I/O, energy and the random start go through the slot map."""
    p = bi.small_3d(7, 5, 6) if case == "small3d" else _group_case(case)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    res = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("BTE_ROTATE", rot)
        with Solver.from_problem(p) as sv:
            assert sv.rotate == (rot == "1")
            sv.set_state(I, T)
            sv.step(3)
            sv.step(4)
            E = sv.energy()
            Ig, Tg = sv.intensity(), sv.temperature()
            sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
            sv.step(2)
            Ir = sv.intensity()
        res[rot] = (Ig, Tg, E, Ir)
    a, b = res["0"], res["1"]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert np.array_equal(a[3], b[3])
    Io, To, _, _ = o.run(I, T, 7)
    rel, dT = _cmp(b[0], b[1], Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_slot_rotation_groups(Solver, monkeypatch):
    """Rotation under the slab group (halo planes follow the slot map) and the
    band group: bit-exact against the same groups without rotation."""
    p = _group_case("3d")
    o = oracle.Oracle(p)
    I, T = o.random_state()
    out = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("BTE_ROTATE", rot)
        group = []
        try:
            for r in range(2):
                sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=2)
                group.append(sv)
                for reg in range(6):
                    bc = p.bcs[reg]
                    sv.set_wall(reg, bc)
                ncross = sv.ncells // sv.nz_local
                c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
                sv.set_state(I[c0:c1], T[c0:c1])
            Solver.group_step(group, 5)
            slab = (np.concatenate([sv.intensity() for sv in group]),
                    np.concatenate([sv.temperature() for sv in group]))
        finally:
            for sv in group:
                sv.close()
        bgroup = _band_group(Solver, p, 2, I, T)
        try:
            Solver.group_step(bgroup, 5)
            band = (np.concatenate([sv.intensity() for sv in bgroup], axis=2), bgroup[0].temperature())
        finally:
            for sv in bgroup:
                sv.close()
        out[rot] = slab + band
    for x, y in zip(out["0"], out["1"]):
        assert np.array_equal(x, y)
    _assert_oracle(p, I, T, 5, out["1"][0], out["1"][1])  # rotated slab group
    _assert_oracle(p, I, T, 5, out["1"][2], out["1"][3])  # rotated band group


# ----------------------------------------------------------------- partially specular walls (reading R-i)

def _partial_problem(case, spec):
    if case == "3d":
        b = bi.subset_bands(bi.silicon_bands(29), [1, 18, 34, 39])
        bcs = [bi.WallBC(bi.BC_PARTIAL, specularity=spec), bi.WallBC(bi.BC_PARTIAL, specularity=1.0 - spec),
               bi.WallBC(bi.BC_ISOTHERMAL, None, 305.0), bi.WallBC(bi.BC_PARTIAL, specularity=spec),
               bi.WallBC(bi.BC_PARTIAL, specularity=spec), bi.WallBC(bi.BC_ISOTHERMAL, None, 298.0)]
        return bi.small_3d(7, 5, 6, bands=b, bcs=bcs)
    p = _group_case("2d")
    p.bcs[0] = bi.WallBC(bi.BC_PARTIAL, specularity=spec)
    p.bcs[1] = bi.WallBC(bi.BC_PARTIAL, specularity=spec)
    return p


@pytest.mark.parametrize("case", ["3d", "2d"])
@pytest.mark.parametrize("spec", [0.37, 0.9])
def test_partial_wall_parity(Solver, case, spec):
    """Partially specular walls (ghost = p I_r + (1-p) g_diffuse) against the oracle."""
    p = _partial_problem(case, spec)
    (rel, dT), _ = _run_both(Solver, p, 9)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


@pytest.mark.parametrize("spec,kind", [(1.0, bi.BC_SPECULAR), (0.0, bi.BC_DIFFUSE)])
def test_partial_wall_limits_bitexact_gpu(Solver, spec, kind):
    """p = 1 is the specular wall and p = 0 the diffuse wall, bit for bit."""
    p = _partial_problem("3d", spec)
    p.bcs[1] = bi.WallBC(bi.BC_PARTIAL, specularity=spec)
    q = _partial_problem("3d", spec)
    q.bcs = [bi.WallBC(kind) if bc.kind == bi.BC_PARTIAL else bc for bc in q.bcs]
    I, T = oracle.Oracle(p).random_state()
    out = []
    for prob in (p, q):
        with Solver.from_problem(prob) as sv:
            sv.set_state(I, T)
            sv.step(6)
            out.append((sv.intensity(), sv.temperature()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_partial_wall_closed_box_energy(Solver):
    b = bi.subset_bands(bi.silicon_bands(29), [2, 19, 33])
    bcs = [bi.WallBC(bi.BC_PARTIAL, specularity=0.4) for _ in range(6)]
    p = bi.small_3d(6, 5, 4, bands=b, bcs=bcs, dirs=bi.directions_control_angle(4, 16))
    I, _ = oracle.Oracle(p).random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, None)
        E0 = sv.energy()
        sv.step(300)
        E1 = sv.energy()
    assert abs(E1 / E0 - 1) < 1e-12, E1 / E0 - 1


def test_partial_wall_rotation_and_groups(Solver, monkeypatch):
    """Partial walls under octant-slot rotation (snapshot + diffuse table), the
    slab group and the band group: bit-exact against one plain context."""
    p = _partial_problem("3d", 0.37)
    I, T = oracle.Oracle(p).random_state()
    res = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("BTE_ROTATE", rot)
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(5)
            res[rot] = (sv.intensity(), sv.temperature())
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][1], res["1"][1])
    monkeypatch.setenv("BTE_ROTATE", "0")
    group = []
    try:
        for r in range(3):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=3)
            group.append(sv)
            for reg in range(6):
                sv.set_wall(reg, p.bcs[reg])
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
        Solver.group_step(group, 5)
        Ig = np.concatenate([sv.intensity() for sv in group])
        Tg = np.concatenate([sv.temperature() for sv in group])
    finally:
        for sv in group:
            sv.close()
    _assert_oracle(p, I, T, 5, Ig, Tg)
    assert np.array_equal(Ig, res["0"][0]) and np.array_equal(Tg, res["0"][1])
    bgroup = _band_group(Solver, p, 2, I, T)
    try:
        Solver.group_step(bgroup, 5)
        Ib = np.concatenate([sv.intensity() for sv in bgroup], axis=2)
        Tb = bgroup[0].temperature()
    finally:
        for sv in bgroup:
            sv.close()
    _assert_oracle(p, I, T, 5, Ib, Tb)
    assert np.max(np.abs(Tb - res["0"][1])) <= 1e-10 and np.max(np.abs(Ib / res["0"][0] - 1)) <= 1e-12


def test_partial_wall_errors(Solver):
    from paper_2305_19400_b200 import BteError
    p = _partial_problem("3d", 0.5)
    with Solver.from_problem(p) as sv:
        for bad in (-0.1, 1.5, float("nan")):
            with pytest.raises(BteError) as e:
                sv.set_bc(0, bi.BC_PARTIAL, specularity=bad)
            assert e.value.status == 1
        with pytest.raises(BteError) as e:  # the plain entry point refuses kind 3
            sv._check(sv._lib.bte_set_bc(sv._h, 0, bi.BC_PARTIAL, None, 300.0))
        assert e.value.status == 1
    d = bi.directions_control_angle(4, 8)
    d.s = d.s.copy()
    d.s[0, 0] += 1e-9
    q = bi.small_3d(dirs=d, bcs=bi.uniform_bcs(bi.BC_DIFFUSE))
    with Solver.from_problem(q) as sv:
        with pytest.raises(BteError) as e:
            sv.set_bc(0, bi.BC_PARTIAL, specularity=0.5)
        assert e.value.status == 6


# ----------------------------------------------------------------- self-consistent tau (reading R-k)

@pytest.mark.parametrize("case", ["small3d", "config2_reduced", "umesh3d"])
def test_sc_tau_parity(Solver, case):
    if case == "small3d":
        p = bi.small_3d(7, 5, 4)
    elif case == "config2_reduced":
        p = bi.config2(n=12)
        p.mesh = bi.Mesh(2, 12, 12, 1, p.mesh.dx, p.mesh.dy, 1.0)
        p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, p.mesh.dx), 300.0)
    else:
        p = bi.small_umesh(3, (3, 2, 2))
    p.tau_mode = 1
    (rel, dT), _ = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
    (rel, dT), _ = _run_both(Solver, p, 3, solve_T=True)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_sc_tau_slab_group_and_errors(Solver):
    from paper_2305_19400_b200 import BteError
    p = _group_case("3d")
    p.tau_mode = 1
    I, T = oracle.Oracle(p).random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(5)
        I1, T1 = sv.intensity(), sv.temperature()
    group = []
    try:
        for r in range(2):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=2)
            group.append(sv)
            for reg in range(6):
                sv.set_wall(reg, p.bcs[reg])
            sv.set_tau_mode(1)
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
        Solver.group_step(group, 5)
        Ig = np.concatenate([s.intensity() for s in group])
        Tg = np.concatenate([s.temperature() for s in group])
    finally:
        for sv in group:
            sv.close()
    _assert_oracle(p, I, T, 5, Ig, Tg)
    assert np.array_equal(Ig, I1) and np.array_equal(Tg, T1)
    bg = _band_group(Solver, p, 2, I, T)
    try:
        with pytest.raises(BteError) as e:
            bg[0].set_tau_mode(1)
        assert e.value.status == 1
    finally:
        for sv in bg:
            sv.close()
    with Solver.from_problem(p) as sv:
        with pytest.raises(BteError):
            sv.set_tau_mode(2)


# ----------------------------------------------------------------- semi-implicit step (reading R-l)

def _semi(p, factor=20.0):
    p.dt = factor * p.dt  # beyond the explicit bound: only the semi-implicit step is stable
    p.semi = 1
    return p


@pytest.mark.parametrize("case", ["small3d", "config2_reduced", "umesh3d"])
def test_semi_parity(Solver, case):
    if case == "small3d":
        p = bi.small_3d(7, 5, 4)
    elif case == "config2_reduced":
        p = bi.config2(n=12)
        p.mesh = bi.Mesh(2, 12, 12, 1, p.mesh.dx, p.mesh.dy, 1.0)
        p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, p.mesh.dx), 300.0)
    else:
        p = bi.small_umesh(3, (3, 2, 2))
        p.bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(3, specularity=0.4),
                 bi.WallBC(0, None, 298.0), bi.WallBC(1)]
    p = _semi(p, 10.0 if case == "umesh3d" else 20.0)  # (the simplices' advection bound is tighter)
    (rel, dT), _ = _run_both(Solver, p, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_semi_groups_rotation_energy_errors(Solver, monkeypatch):
    from paper_2305_19400_b200 import BteError
    p = _semi(_group_case("3d"))
    I, T = oracle.Oracle(p).random_state()
    res = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("BTE_ROTATE", rot)
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(5)
            res[rot] = (sv.intensity(), sv.temperature())
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][1], res["1"][1])
    monkeypatch.setenv("BTE_ROTATE", "0")
    group = []
    try:
        for r in range(3):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=3, step_mode=1)
            group.append(sv)
            for reg in range(6):
                sv.set_wall(reg, p.bcs[reg])
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
        Solver.group_step(group, 5)
        Ig = np.concatenate([s.intensity() for s in group])
        Tg = np.concatenate([s.temperature() for s in group])
    finally:
        for sv in group:
            sv.close()
    _assert_oracle(p, I, T, 5, Ig, Tg)
    assert np.array_equal(Ig, res["0"][0]) and np.array_equal(Tg, res["0"][1])
    # closed box at 40x the explicit bound: conservative and positive
    b = bi.subset_bands(bi.silicon_bands(29), [2, 19, 33])
    q = _semi(bi.small_3d(6, 5, 4, bands=b, bcs=bi.uniform_bcs(bi.BC_SPECULAR)), 40.0)
    Iq, _ = oracle.Oracle(q).random_state()
    with Solver.from_problem(q) as sv:
        sv.set_state(Iq, None)
        E0 = sv.energy()
        sv.step(100)
        E1 = sv.energy()
        assert sv.intensity().min() > 0
        with pytest.raises(BteError) as e:
            sv.set_step_mode(0)  # explicit at this dt: unstable
        assert e.value.status == 5
        with pytest.raises(BteError):
            sv.set_tau_mode(1)
    assert abs(E1 / E0 - 1) < 1e-12
    with pytest.raises(BteError) as e:
        Solver(q.mesh, q.dirs, q.bands, q.dt, q.T_init)  # explicit creation at this dt
    assert e.value.status == 5
    with pytest.raises(BteError) as e:
        Solver(q.mesh, q.dirs, q.bands, q.dt, q.T_init, rank=0, nranks=2, decomp="band", step_mode=1)
    assert e.value.status == 1


def test_sc_tau_rotation_bitexact(Solver, monkeypatch):
    """Self-consistent tau under octant-slot rotation equals two buffers bit for bit."""
    p = _group_case("3d")
    p.tau_mode = 1
    I, T = oracle.Oracle(p).random_state()
    res = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("BTE_ROTATE", rot)
        with Solver.from_problem(p) as sv:
            sv.set_state(I, T)
            sv.step(4)
            res[rot] = (sv.intensity(), sv.temperature())
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][1], res["1"][1])


@pytest.mark.parametrize("direct", ["0", "1"])
def test_sc_tau_fixed_point_and_kernels(Solver, direct, monkeypatch):
    """Self-consistent tau: a uniform equilibrium stays exactly fixed, and both
    Newton kernels (uniform-grid band integrals / direct integrals) match the oracle."""
    monkeypatch.setenv("BTE_SC_DIRECT", direct)
    b = bi.subset_bands(bi.silicon_bands(29), [0, 10, 20, 30, 39])
    bcs = [bi.WallBC(1), bi.WallBC(1), bi.WallBC(0, None, 300.0), bi.WallBC(1), bi.WallBC(0, None, 300.0),
           bi.WallBC(1)]
    p = bi.small_3d(8, 6, 5, bands=b, bcs=bcs)
    p.tau_mode = 1
    with Solver.from_problem(p) as sv:
        I0, T0 = sv.intensity(), sv.temperature()
        sv.step(20)
        assert np.array_equal(sv.intensity(), I0) and np.array_equal(sv.temperature(), T0)
    q = bi.config2(n=12)
    q.mesh = bi.Mesh(2, 12, 12, 1, q.mesh.dx, q.mesh.dy, 1.0)
    q.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, q.mesh.dx), 300.0)
    q.tau_mode = 1
    (rel, dT), _ = _run_both(Solver, q, 6)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_fig9_workload_full_size(Solver):
    """The paper's second example (Fig. 9 shape, bench --config 10) at full size."""
    p = bi.config_fig9()
    (rel, dT), (Ig, Tg, Io, To) = _run_both(Solver, p, 5)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_demo_20000_steps_long_run(Solver):
    """The paper's long demo run (20,000 steps = 20 ns at dt = 1 ps)
    from the 300 K equilibrium: finite throughout, inside the walls'
    temperature range (maximum principle of the positive explicit update),
    mirror-symmetric about x = L/2 bit for bit after 20,000 steps, and still
    heating (the first 100 steps are checked against the oracle in
    test_demo_workload_full_size)."""
    p = bi.config_demo()
    n = p.mesh.nx
    with Solver.from_problem(p) as sv:
        sv.step(10000)
        T1 = sv.temperature()
        sv.step(10000)
        T2 = sv.temperature()
        E = sv.energy()
    assert np.all(np.isfinite(T2)) and np.isfinite(E)
    assert T2.min() >= 300.0 - 1e-9 and T2.max() <= 350.0 + 1e-9
    F = T2.reshape(n, n)
    assert np.array_equal(F, F[:, ::-1])
    assert T2.mean() > T1.mean() > 300.0


# ----------------------------------------------------------------- implicit step by source iteration (reading R-n)

def _implicit(p, iters, tol=0.0, dt_factor=1.0):
    p.dt = dt_factor * p.dt
    p.implicit = 1
    p.imp_max_iter = iters
    p.imp_tol = tol
    return p


def _imp_cases():
    c2 = bi.config2(n=12)
    c2.mesh = bi.Mesh(2, 12, 10, 1, c2.mesh.dx, c2.mesh.dy, 1.0)
    c2.bcs[3] = bi.WallBC(0, bi.hotspot_profile(12, c2.mesh.dx), 300.0)
    c3 = bi.config3()
    c3.mesh = bi.Mesh(3, 7, 6, 5, c3.mesh.dx, c3.mesh.dy, c3.mesh.dz)  # the 400 x 40 tables: TMA-ring blocks
    return {"small3d": bi.small_3d(7, 5, 4), "config2_reduced": c2, "config3_tables": c3,
            "inplane_55": bi.Problem("demo_small", bi.Mesh(2, 9, 7, 1, 4.375e-6, 4.375e-6, 1.0),
                                     bi.directions_inplane(20), bi.silicon_bands(40), 1e-12, 300.0,
                                     [bi.WallBC(1), bi.WallBC(1), bi.WallBC(0, None, 300.0),
                                      bi.WallBC(0, bi.hotspot_profile(9, 4.375e-6), 300.0), bi.WallBC(1),
                                      bi.WallBC(1)], seed=3),
            "all_kinds_3d": bi.small_3d(6, 5, 4, bcs=[bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0),
                                                      bi.WallBC(3, specularity=0.4), bi.WallBC(2),
                                                      bi.WallBC(0, None, 298.0)])}


@pytest.mark.parametrize("case", ["small3d", "config2_reduced", "config3_tables", "inplane_55", "all_kinds_3d"])
def test_implicit_parity_fixed_iterations(Solver, case):
    """Implicit step (wavefront transport sweeps + lagged Newton per source
    iteration) against the oracle: 3 steps x 5 iterations at 8x the explicit dt."""
    p = _implicit(_imp_cases()[case], 5, 0.0, 8.0)
    (rel, dT), _ = _run_both(Solver, p, 3)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_implicit_parity_tolerance_and_iteration_counts(Solver):
    """Early stop at a tolerance: the GPU takes the oracle's iteration counts."""
    p = _implicit(_imp_cases()["all_kinds_3d"], 60, 1e-9, 4.0)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    Io, To, _, _ = o.run(I, T, 3)
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(3)
        Ig, Tg = sv.intensity(), sv.temperature()
        its = sv.iterations()
    assert list(its) == list(o.last_iters) and its.max() < 60, (its, o.last_iters)
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_implicit_fixed_point_and_closed_box(Solver):
    b = bi.subset_bands(bi.silicon_bands(29), [0, 10, 20, 30, 39])
    bcs = [bi.WallBC(1), bi.WallBC(1), bi.WallBC(0, None, 300.0), bi.WallBC(1), bi.WallBC(0, None, 300.0),
           bi.WallBC(1)]
    p = _implicit(bi.small_3d(6, 5, 4, bands=b, bcs=bcs), 4, 0.0, 20.0)
    with Solver.from_problem(p) as sv:
        T0, I0 = sv.temperature(), sv.intensity()
        sv.step(5)
        assert np.array_equal(sv.intensity(), I0) and np.array_equal(sv.temperature(), T0)
    b = bi.subset_bands(bi.silicon_bands(29), [2, 19, 33])
    q = _implicit(bi.small_3d(6, 5, 4, bands=b, bcs=bi.uniform_bcs(bi.BC_DIFFUSE)), 200, 1e-14, 10.0)
    I, _ = oracle.Oracle(q).random_state()
    with Solver.from_problem(q) as sv:
        sv.set_state(I, None)
        E0 = sv.energy()
        sv.step(3)
        E1 = sv.energy()
        assert sv.intensity().min() > 0 and sv.iterations().max() < 200
    assert abs(E1 / E0 - 1) < 1e-12


def test_implicit_errors(Solver, monkeypatch):
    from paper_2305_19400_b200 import BteError
    p = _group_case("3d")
    with Solver.from_problem(p) as sv:
        with pytest.raises(BteError):
            sv.set_implicit(0, 1e-9)
        with pytest.raises(BteError):
            sv.set_implicit(5, -1.0)
        sv.set_step_mode(2)
        with pytest.raises(BteError):
            sv.set_tau_mode(1)
        assert sv._lib.bte_set_step_mode(sv._h, 3) == 1
    sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=0, nranks=2)
    try:
        with pytest.raises(BteError):
            sv.set_step_mode(2)  # multi-rank: no wavefront across slabs
    finally:
        sv.close()
    monkeypatch.setenv("BTE_ROTATE", "1")
    with Solver.from_problem(p) as sv:
        with pytest.raises(BteError):
            sv.set_step_mode(2)  # every iteration re-reads I^n: two buffers needed


# ----------------------------------------------------------------- degenerate sizes and edge cases

@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 1, 5), (7, 1, 1), (1, 6, 1), (2, 2, 1)])
def test_degenerate_3d_boxes_400x40(Solver, shape):
    """The BASELINE 400 x 40 tables (the TMA sweep) on boxes whose every column
    is a wall column in x and/or y, single-plane columns and a single cell;
    every wall kind."""
    p = bi.config3()
    p.mesh = bi.Mesh(3, *shape, p.mesh.dx, p.mesh.dy, p.mesh.dz)
    p.bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(3, specularity=0.3),
             bi.WallBC(0, None, 298.0), bi.WallBC(1)]
    (rel, dT), _ = _run_both(Solver, p, 4)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


@pytest.mark.parametrize("shape", [(1, 1), (9, 1), (1, 9)])
def test_degenerate_2d_strips(Solver, shape):
    p = bi.config2(n=4)
    p.mesh = bi.Mesh(2, shape[0], shape[1], 1, p.mesh.dx, p.mesh.dy, 1.0)
    p.bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 300.0), bi.WallBC(0, None, 310.0),
             bi.WallBC(1), bi.WallBC(1)]
    (rel, dT), _ = _run_both(Solver, p, 5)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)


def test_zero_steps_and_repeated_calls(Solver):
    """step(0) changes nothing; many step(1) calls equal one step(n) call (the
    graph-replayed path) bit for bit; the step counter in error messages follows."""
    p = bi.small_3d(6, 5, 4)
    I, T = oracle.Oracle(p).random_state()
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(0)
        assert np.array_equal(sv.intensity(), I) and np.array_equal(sv.temperature(), T)
        for _ in range(6):
            sv.step(1)
        a = (sv.intensity(), sv.temperature())
    with Solver.from_problem(p) as sv:
        sv.set_state(I, T)
        sv.step(6)
        b = (sv.intensity(), sv.temperature())
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_slab_group_one_plane_slabs(Solver):
    """As many slabs as planes (every rank owns one plane: both halo planes are
    live, walls only on the end ranks) against the oracle."""
    p = _group_case("3d")
    p.mesh = bi.Mesh(3, 4, 3, 5, p.mesh.dx, p.mesh.dy, p.mesh.dz)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    group = []
    try:
        for r in range(5):
            sv = Solver(p.mesh, p.dirs, p.bands, p.dt, p.T_init, rank=r, nranks=5)
            group.append(sv)
            for reg in range(6):
                sv.set_wall(reg, p.bcs[reg])
            ncross = sv.ncells // sv.nz_local
            c0, c1 = sv.z0 * ncross, (sv.z0 + sv.nz_local) * ncross
            sv.set_state(I[c0:c1], T[c0:c1])
        assert all(sv.nz_local == 1 for sv in group)
        Solver.group_step(group, 4)
        Ig = np.concatenate([sv.intensity() for sv in group])
        Tg = np.concatenate([sv.temperature() for sv in group])
    finally:
        for sv in group:
            sv.close()
    _assert_oracle(p, I, T, 4, Ig, Tg)


@pytest.mark.parametrize("case", ["config3_tables", "rotated", "inplane55"])
def test_set_state_temperature_only(Solver, monkeypatch, case):
    """bte_set_state(NULL, T) -- the e2e job's input path: I = I0(T) built on the
    device (k_fill_eq) must equal the oracle's equilibrium of that T field, and
    the steps that follow must match the oracle from (I0(T), T).  Covers the
    40-channel 3-D tables, the octant-slot rotated layout and an in-plane set
    with 55 channels (E not a multiple of the 256-thread block)."""
    if case == "rotated":
        monkeypatch.setenv("BTE_ROTATE", "1")
    if case == "inplane55":
        p = bi.small_3d(6, 5, 3, dirs=bi.directions_inplane(20), bands=bi.silicon_bands(40),
                        bcs=[bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 303.0), bi.WallBC(1),
                             bi.WallBC(1), bi.WallBC(1)])
    else:
        p = bi.config3(n=8)
        p.mesh = bi.Mesh(3, 7, 6, 5, 1e-6, 1e-6, 1e-6)
    o = oracle.Oracle(p)
    _, T = o.random_state()
    I = o.equilibrium(T)
    with Solver.from_problem(p) as sv:
        sv.set_state(None, T)
        Ig0 = sv.intensity()
        assert np.array_equal(sv.temperature(), T)
        assert np.max(np.abs(Ig0 - I) / np.abs(I)) <= REL_I
        sv.step(3)
        Ig, Tg = sv.intensity(), sv.temperature()
    Io, To, _, _ = o.run(I, T, 3)
    rel, dT = _cmp(Ig, Tg, Io, To)
    assert rel <= REL_I and dT <= ABS_T, (rel, dT)
