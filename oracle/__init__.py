"""CPU ORACLE for the BTE explicit step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It wraps
``oracle/bte_oracle.c`` (plain fp64, cell -> direction -> band loops, built
with ``gcc -O2 -ffp-contract=off -fopenmp``) through ctypes and shares no code
with the CUDA path.  Every function cites the passage it follows in the C
source; the readings it relies on are listed in DESIGN.md.

``exact.py`` holds the pure-Python ``fractions`` twin used to pin the C sweep.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bte_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "bte_oracle_umesh.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

ORA_OK = 0
ORA_ERRORS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 6: "ENOTCLOSED", 7: "ENEWTON", 8: "ENONFINITE"}


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(f)
                                                      for f in _SRCS):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-std=c11", "-D_GNU_SOURCE", "-o", _LIB_PATH, *_SRCS, "-lm"]
        subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


class _UMesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("nverts", C.c_long), ("verts", C.c_void_p), ("ncells", C.c_long),
                ("cells", C.c_void_p), ("depth", C.c_double), ("nvc", C.c_int)]


class _Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("nx", C.c_long), ("ny", C.c_long), ("nz", C.c_long),
        ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
        ("nd", C.c_int), ("s", C.c_void_p), ("w", C.c_void_p),
        ("nb", C.c_int), ("v", C.c_void_p), ("mode", C.c_int),
        ("I_ref", C.c_void_p), ("slope", C.c_void_p), ("T_ref", C.c_double),
        ("w_lo", C.c_void_p), ("w_hi", C.c_void_p), ("vs", C.c_void_p), ("c2", C.c_void_p),
        ("g", C.c_void_p), ("beta_coef", C.c_void_p),
        ("dt", C.c_double),
        ("bc_kind", C.c_int * 6), ("T_wall", C.c_void_p * 6), ("T_uniform", C.c_double * 6),
        ("nthreads", C.c_int),
        ("specularity", C.c_double * 6),
        ("tau_mode", C.c_int),
        ("semi", C.c_int),
        ("implicit", C.c_int),
        ("imp_max_iter", C.c_int),
        ("imp_tol", C.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        P = C.POINTER(_Problem)
        _lib.ora_I0.restype = C.c_double
        _lib.ora_I0.argtypes = [P, C.c_int, C.c_double, dp]
        _lib.ora_beta.restype = C.c_double
        _lib.ora_beta.argtypes = [P, C.c_int, C.c_double]
        _lib.ora_dbeta.restype = C.c_double
        _lib.ora_dbeta.argtypes = [P, C.c_int, C.c_double]
        _lib.ora_newton_sc.argtypes = [P, C.c_double, C.c_void_p, C.c_void_p, dp, C.POINTER(C.c_int)]
        _lib.ora_energy.restype = C.c_double
        _lib.ora_energy.argtypes = [P, C.c_void_p]
        _lib.ora_dt_margin.restype = C.c_double
        _lib.ora_dt_margin.argtypes = [P, C.c_double]
        _lib.ora_gauss_legendre.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        _lib.ora_reflection.argtypes = [P, C.c_int, C.c_void_p]
        _lib.ora_equilibrium.argtypes = [P, C.c_void_p, C.c_void_p]
        _lib.ora_refresh.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_sweep.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_reduce.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_ghost_table.argtypes = [P, C.c_int, C.c_void_p, C.c_void_p]
        _lib.ora_newton.argtypes = [P, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, dp,
                                    C.POINTER(C.c_int)]
        _lib.ora_temperature_update.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.POINTER(C.c_long), C.POINTER(C.c_int)]
        _lib.ora_run.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long,
                                 C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_int)]
        _lib.ora_run_implicit.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long,
                                          C.c_void_p, C.POINTER(C.c_long), C.POINTER(C.c_long)]
        _lib.ora_solve_T.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_n_faces.restype = C.c_long
        _lib.ora_n_faces.argtypes = [P, C.c_int]
        U = C.POINTER(_UMesh)
        _lib.ora_ugeom_build.argtypes = [U, C.POINTER(C.c_void_p)]
        _lib.ora_ugeom_free.argtypes = [C.c_void_p]
        _lib.ora_ugeom_nfaces.restype = C.c_long
        _lib.ora_ugeom_nfaces.argtypes = [C.c_void_p, C.c_int]
        _lib.ora_ugeom_export.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        _lib.ora_usweep.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_urun.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long,
                                  C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_int)]
        _lib.ora_uenergy.restype = C.c_double
        _lib.ora_uenergy.argtypes = [P, C.c_void_p, C.c_void_p]
        _lib.ora_udt_margin.restype = C.c_double
        _lib.ora_udt_margin.argtypes = [P, C.c_void_p, C.c_double, C.c_int]
        assert _lib.ora_sizeof_problem() == C.sizeof(_Problem)
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {ORA_ERRORS.get(code, code)} {msg}")
        self.code = code


class Oracle:
    """Oracle bound to one ``bte_inputs.Problem``; state arrays are canonical
    numpy arrays: I[ncells, nd, nb], T[ncells], I0c[ncells, nb], betac[ncells, nb]."""

    def __init__(self, problem, nthreads: Optional[int] = None):
        self.problem = problem
        m, d, b = problem.mesh, problem.dirs, problem.bands
        self._keep = []

        def keep(a):
            a = _f64(a)
            if a is not None:
                self._keep.append(a)
            return a

        st = _Problem()
        self.umesh = hasattr(m, "cells")
        if self.umesh:  # unstructured (bte_oracle_umesh.c): per-cell pieces see nx = ncells
            st.dim, st.nx, st.ny, st.nz = m.dim, m.ncells, 1, 1
            st.dx = st.dy = st.dz = 1.0
        else:
            st.dim, st.nx, st.ny, st.nz = m.dim, m.nx, m.ny, m.nz
            st.dx, st.dy, st.dz = m.dx, m.dy, m.dz
        st.nd = d.nd
        st.s = _ptr(keep(d.s))
        st.w = _ptr(keep(d.w))
        st.nb = b.nb
        st.v = _ptr(keep(b.v))
        st.mode = b.mode
        st.I_ref = _ptr(keep(b.I_ref))
        st.slope = _ptr(keep(b.slope))
        st.T_ref = b.T_ref
        for name in ("w_lo", "w_hi", "vs", "c2", "g"):
            setattr(st, name, _ptr(keep(getattr(b, name))))
        st.beta_coef = _ptr(keep(b.beta_coef))
        st.dt = problem.dt
        for r in range(6):
            bc = problem.bcs[r]
            st.bc_kind[r] = bc.kind
            st.T_wall[r] = _ptr(keep(bc.T_wall)) if bc.T_wall is not None else None
            st.T_uniform[r] = bc.T_uniform
            st.specularity[r] = getattr(bc, "specularity", 1.0)
        st.nthreads = nthreads if nthreads else (os.cpu_count() or 1)
        st.tau_mode = int(getattr(problem, "tau_mode", 0))
        st.semi = int(getattr(problem, "semi", 0))
        st.implicit = int(getattr(problem, "implicit", 0))
        st.imp_max_iter = int(getattr(problem, "imp_max_iter", 0))
        st.imp_tol = float(getattr(problem, "imp_tol", 0.0))
        self._st = st
        self.nc, self.nd, self.nb = m.ncells, d.nd, b.nb
        lib()
        self._ug = None
        if self.umesh:
            self._verts = np.ascontiguousarray(m.verts, dtype=np.float64)
            self._cells = np.ascontiguousarray(m.cells, dtype=np.int64)
            um = _UMesh(m.dim, self._verts.shape[0], self._verts.ctypes.data, self._cells.shape[0],
                        self._cells.ctypes.data, float(m.depth), int(self._cells.shape[1]))
            h = C.c_void_p()
            rc = lib().ora_ugeom_build(C.byref(um), C.byref(h))
            if rc:
                raise OracleError(rc, "unstructured geometry")
            self._ug = h

    def __del__(self):
        if getattr(self, "_ug", None):
            lib().ora_ugeom_free(self._ug)
            self._ug = None

    # -- unstructured geometry (tests)
    def geometry(self):
        """(vol[nc], area[nc,K], normal[nc,K,3], nbr[nc,K], region[nc,K]) of an unstructured mesh."""
        m = self.problem.mesh
        K = 6 if (m.dim == 3 and m.cells.shape[1] == 8) else int(m.cells.shape[1])  # faces per cell
        vol = np.empty(self.nc)
        area = np.empty((self.nc, K))
        nrm = np.empty((self.nc, K, 3))
        nbr = np.empty((self.nc, K), dtype=np.int64)
        reg = np.empty((self.nc, K), dtype=np.int32)
        lib().ora_ugeom_export(self._ug, vol.ctypes.data, area.ctypes.data, nrm.ctypes.data, nbr.ctypes.data,
                               reg.ctypes.data)
        return vol, area, nrm, nbr, reg

    def n_region_faces(self, region: int) -> int:
        if self.umesh:
            return int(lib().ora_ugeom_nfaces(self._ug, region))
        return int(lib().ora_n_faces(C.byref(self._st), region))

    def udt_margin(self, beta_max: float, b: int) -> float:
        return lib().ora_udt_margin(C.byref(self._st), self._ug, beta_max, b)

    # -- material functions
    def I0(self, b: int, T: float) -> Tuple[float, float]:
        dI = C.c_double()
        v = lib().ora_I0(C.byref(self._st), b, T, C.byref(dI))
        return v, dI.value

    def beta(self, b: int, T: float) -> float:
        return lib().ora_beta(C.byref(self._st), b, T)

    def dbeta(self, b: int, T: float) -> float:
        return lib().ora_dbeta(C.byref(self._st), b, T)

    def newton_sc(self, Tn: float, D, I0c):
        """Self-consistent-tau Newton of one cell (reading R-k)."""
        D, I0c = _f64(D), _f64(I0c)
        T = C.c_double()
        it = C.c_int()
        st = lib().ora_newton_sc(C.byref(self._st), Tn, _ptr(D), _ptr(I0c), C.byref(T), C.byref(it))
        if st:
            raise OracleError(st, "newton_sc")
        return T.value, it.value

    def I0_vec(self, T: np.ndarray) -> np.ndarray:
        T = np.asarray(T, dtype=np.float64).reshape(-1)
        out = np.empty((T.size, self.nb))
        for i, t in enumerate(T):
            for b in range(self.nb):
                out[i, b] = self.I0(b, float(t))[0]
        return out

    def reflection(self, axis: int) -> np.ndarray:
        r = np.empty(self.nd, dtype=np.int32)
        st = lib().ora_reflection(C.byref(self._st), axis, r.ctypes.data)
        if st:
            raise OracleError(st, f"reflection axis {axis}")
        return r

    def dt_margin(self, Tmax: float) -> float:
        return lib().ora_dt_margin(C.byref(self._st), Tmax)

    # -- state
    def equilibrium(self, T: np.ndarray) -> np.ndarray:
        T = _f64(T)
        I = np.empty((self.nc, self.nd, self.nb))
        lib().ora_equilibrium(C.byref(self._st), _ptr(T), _ptr(I))
        return I

    def refresh(self, T: np.ndarray):
        T = _f64(T)
        I0c = np.empty((self.nc, self.nb))
        betac = np.empty((self.nc, self.nb))
        lib().ora_refresh(C.byref(self._st), _ptr(T), _ptr(I0c), _ptr(betac))
        return I0c, betac

    def random_state(self, seed: Optional[int] = None, T_amp: float = 20.0, I_amp: float = 0.05):
        """Random start: T_c from bte_inputs, I = I0_b(T_c)*(1 + amp(2u-1))."""
        import bte_inputs as bi
        p = self.problem
        seed = p.seed if seed is None else seed
        T = bi.random_temperature(p.mesh, seed, p.T_init, T_amp)
        I = self.equilibrium(T)
        I *= bi.intensity_noise_factor(seed, self.nc, self.nd, self.nb, I_amp)
        return I, T

    # -- step pieces
    def sweep(self, I, I0c, betac) -> np.ndarray:
        I, I0c, betac = _f64(I), _f64(I0c), _f64(betac)
        out = np.empty_like(I)
        if self.umesh:
            st = lib().ora_usweep(C.byref(self._st), self._ug, _ptr(I), _ptr(I0c), _ptr(betac), _ptr(out))
        else:
            st = lib().ora_sweep(C.byref(self._st), _ptr(I), _ptr(I0c), _ptr(betac), _ptr(out))
        if st:
            raise OracleError(st, "sweep")
        return out

    def reduce(self, I, I0c) -> np.ndarray:
        I, I0c = _f64(I), _f64(I0c)
        D = np.empty((self.nc, self.nb))
        lib().ora_reduce(C.byref(self._st), _ptr(I), _ptr(I0c), _ptr(D))
        return D

    def ghost_table(self, region: int, I) -> np.ndarray:
        I = _f64(I)
        n = lib().ora_n_faces(C.byref(self._st), region)
        g = np.empty((n, self.nb))
        st = lib().ora_ghost_table(C.byref(self._st), region, _ptr(I), _ptr(g))
        if st:
            raise OracleError(st, "ghost_table")
        return g

    def newton(self, Tn: float, D, I0c, bnext):
        D, I0c, bnext = _f64(D), _f64(I0c), _f64(bnext)
        T = C.c_double()
        it = C.c_int()
        st = lib().ora_newton(C.byref(self._st), Tn, _ptr(D), _ptr(I0c), _ptr(bnext), C.byref(T), C.byref(it))
        if st:
            raise OracleError(st, "newton")
        return T.value, it.value

    def temperature_update(self, D, T, I0c, betac):
        D = _f64(D)
        T, I0c, betac = _f64(T).copy(), _f64(I0c).copy(), _f64(betac).copy()
        bad = C.c_long()
        it = C.c_int()
        st = lib().ora_temperature_update(C.byref(self._st), _ptr(D), _ptr(T), _ptr(I0c), _ptr(betac),
                                          C.byref(bad), C.byref(it))
        if st:
            raise OracleError(st, f"cell {bad.value}")
        return T, I0c, betac

    def run(self, I, T, nsteps: int, I0c=None, betac=None):
        """nsteps explicit steps from (I, T); I0c/betac default to I0(T), beta(T)."""
        I = _f64(I).copy()
        T = _f64(T).copy()
        if I0c is None or betac is None:
            I0c, betac = self.refresh(T)
        else:
            I0c, betac = _f64(I0c).copy(), _f64(betac).copy()
        es, ec = C.c_long(), C.c_long()
        it = C.c_int()
        if self._st.implicit:  # reading R-n: implicit step by source iteration
            if self.umesh:
                raise OracleError(1, "implicit step: structured grids only")
            iters = np.zeros(max(1, nsteps), dtype=np.int64)
            st = lib().ora_run_implicit(C.byref(self._st), _ptr(I), _ptr(T), _ptr(I0c), _ptr(betac), nsteps,
                                        iters.ctypes.data, C.byref(es), C.byref(ec))
            if st:
                raise OracleError(st, f"step {es.value} cell {ec.value}")
            self.last_iters = iters[:nsteps].copy()
            return I, T, I0c, betac
        if self.umesh:
            st = lib().ora_urun(C.byref(self._st), self._ug, _ptr(I), _ptr(T), _ptr(I0c), _ptr(betac), nsteps,
                                C.byref(es), C.byref(ec), C.byref(it))
        else:
            st = lib().ora_run(C.byref(self._st), _ptr(I), _ptr(T), _ptr(I0c), _ptr(betac), nsteps,
                               C.byref(es), C.byref(ec), C.byref(it))
        if st:
            raise OracleError(st, f"step {es.value} cell {ec.value}")
        self.last_max_iters = it.value
        return I, T, I0c, betac

    def solve_T(self, I, T_guess):
        I, T_guess = _f64(I), _f64(T_guess)
        T = np.empty(self.nc)
        I0c = np.empty((self.nc, self.nb))
        betac = np.empty((self.nc, self.nb))
        st = lib().ora_solve_T(C.byref(self._st), _ptr(I), _ptr(T_guess), _ptr(T), _ptr(I0c), _ptr(betac))
        if st:
            raise OracleError(st, "solve_T")
        return T, I0c, betac

    def energy(self, I) -> float:
        I = _f64(I)
        if self.umesh:
            return lib().ora_uenergy(C.byref(self._st), self._ug, _ptr(I))
        return lib().ora_energy(C.byref(self._st), _ptr(I))


def gauss_legendre(n: int):
    x = np.empty(n)
    w = np.empty(n)
    lib().ora_gauss_legendre(n, x.ctypes.data, w.ctypes.data)
    return x, w
