"""Thin ctypes binding of libbte.so (include/bte.h).  Argument marshalling only:
every step of the BTE hot path runs in the library's CUDA kernels.  PyTorch
supplies device memory (caching allocator), the CUDA stream and, for several
GPUs, the NCCL unique-id broadcast over torch.distributed.

Names follow include/bte.h.  There is no CPU fallback: if libbte.so is
missing or no CUDA device is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BTE_LIB") or os.path.join(_HERE, "libbte.so")  # BTE_LIB: A/B builds

BTE_OK = 0
STATUS = {0: "BTE_OK", 1: "BTE_EINVAL", 2: "BTE_ENOMEM", 3: "BTE_ECUDA", 4: "BTE_ENCCL",
          5: "BTE_EUNSTABLE", 6: "BTE_ENOTCLOSED", 7: "BTE_ENEWTON", 8: "BTE_ENONFINITE"}
BC_ISOTHERMAL, BC_SPECULAR, BC_DIFFUSE, BC_PARTIAL = 0, 1, 2, 3
I0_LINEAR, I0_BOSE_EINSTEIN = 0, 1

EXPORTS = ("bte_group_step", "bte_plan_slab", "bte_plan_band", "bte_create", "bte_create_band", "bte_create_umesh", "bte_get_region_faces", "bte_plan_umesh", "bte_set_tau_mode", "bte_set_step_mode", "bte_set_bc", "bte_set_bc_partial", "bte_set_state", "bte_init_random", "bte_step",
           "bte_get_intensity", "bte_get_intensity_cells", "bte_get_temperature", "bte_get_energy", "bte_debug_substep",
           "bte_timing_enable", "bte_timing_read", "bte_get_info", "bte_last_error", "bte_destroy",
           "bte_version", "bte_set_debug", "bte_set_implicit", "bte_get_iterations", "bte_mesh_read",
           "bte_mesh_free", "bte_mesh_error", "bte_partition_rcb")
DEBUG_SKIP_EXCHANGE = 1


class BteError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double)]


class UMeshC(C.Structure):
    _fields_ = [("dim", C.c_int), ("nverts", C.c_int64), ("verts", C.c_void_p), ("ncells", C.c_int64),
                ("cells", C.c_void_p), ("depth", C.c_double), ("nvc", C.c_int)]


class UPeerC(C.Structure):
    _fields_ = [("peer", C.c_int), ("recv_off", C.c_int64), ("recv_cnt", C.c_int64), ("send_off", C.c_int64),
                ("send_cnt", C.c_int64)]


class UPlanC(C.Structure):
    _fields_ = [("cell0", C.c_int64), ("n_own", C.c_int64), ("n_halo", C.c_int64), ("n_peers", C.c_int),
                ("peer", UPeerC * 32)]


class MeshDataC(C.Structure):
    _fields_ = [("dim", C.c_int), ("nvc", C.c_int), ("nverts", C.c_int64), ("ncells", C.c_int64),
                ("verts", C.POINTER(C.c_double)), ("cells", C.POINTER(C.c_int64))]


class Dirs(C.Structure):
    _fields_ = [("nd", C.c_int), ("s", C.c_void_p), ("w", C.c_void_p)]


class Bands(C.Structure):
    _fields_ = [("nb", C.c_int), ("v", C.c_void_p), ("mode", C.c_int), ("I_ref", C.c_void_p),
                ("slope", C.c_void_p), ("T_ref", C.c_double), ("w_lo", C.c_void_p),
                ("w_hi", C.c_void_p), ("vs", C.c_void_p), ("c2", C.c_void_p), ("g", C.c_void_p),
                ("beta_coef", C.c_void_p)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
DEALLOC_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class Run(C.Structure):
    _fields_ = [("dt", C.c_double), ("T_init", C.c_double), ("device", C.c_int),
                ("stream", C.c_void_p), ("rank", C.c_int), ("nranks", C.c_int),
                ("nccl_id", C.c_void_p), ("alloc", ALLOC_FN), ("dealloc", DEALLOC_FN),
                ("alloc_ctx", C.c_void_p), ("step_mode", C.c_int)]


class Timing(C.Structure):
    _fields_ = [("steps", C.c_int64), ("launches", C.c_int64), ("sweep_ms", C.c_double),
                ("newton_ms", C.c_double), ("boundary_ms", C.c_double), ("halo_ms", C.c_double),
                ("sweep_launches", C.c_int64), ("newton_launches", C.c_int64),
                ("boundary_launches", C.c_int64), ("truncated", C.c_int64)]


class Msg(C.Structure):
    _fields_ = [("send", C.c_int), ("peer", C.c_int), ("octant", C.c_int), ("slot", C.c_int),
                ("plane", C.c_int64), ("count", C.c_int64)]


class SlabPlan(C.Structure):
    _fields_ = [("axis", C.c_int), ("m0", C.c_int64), ("n_local", C.c_int64), ("n_msgs", C.c_int),
                ("msg", Msg * 32)]


class Info(C.Structure):
    _fields_ = [("ncells_local", C.c_int64), ("ncells_global", C.c_int64), ("z0", C.c_int64),
                ("nz_local", C.c_int64), ("nd", C.c_int), ("nb", C.c_int), ("n_octants", C.c_int),
                ("nj", C.c_int), ("bytes_state", C.c_int64), ("b0", C.c_int), ("b1", C.c_int),
                ("nb_total", C.c_int), ("band", C.c_int), ("rotate", C.c_int), ("cell0", C.c_int64),
                ("sweep_kernel", C.c_char_p), ("step_mode", C.c_int),
                ("newton_kernel", C.c_char_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libbte.so; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    P = C.c_void_p
    dp = C.c_void_p
    lib.bte_create.argtypes = [C.POINTER(Mesh), C.POINTER(Dirs), C.POINTER(Bands), C.POINTER(Run),
                               C.POINTER(C.c_void_p)]
    if hasattr(lib, "bte_create_band"):  # (older A/B builds via BTE_LIB lack the band entry points)
        lib.bte_create_band.argtypes = lib.bte_create.argtypes
        lib.bte_plan_band.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    if hasattr(lib, "bte_create_umesh"):
        lib.bte_create_umesh.argtypes = [C.POINTER(UMeshC), C.POINTER(Dirs), C.POINTER(Bands), C.POINTER(Run),
                                         C.POINTER(C.c_void_p)]
        lib.bte_get_region_faces.argtypes = [P, C.c_int, C.POINTER(C.c_int64)]
    if hasattr(lib, "bte_plan_umesh"):
        lib.bte_plan_umesh.argtypes = [C.POINTER(UMeshC), C.c_int, C.c_int, C.POINTER(UPlanC), dp, C.c_int64, dp,
                                       C.c_int64]
    if hasattr(lib, "bte_get_intensity_cells"):
        lib.bte_get_intensity_cells.argtypes = [P, dp, C.c_int64, dp]
    if hasattr(lib, "bte_set_tau_mode"):
        lib.bte_set_tau_mode.argtypes = [P, C.c_int]
    if hasattr(lib, "bte_set_step_mode"):
        lib.bte_set_step_mode.argtypes = [P, C.c_int]
    lib.bte_set_bc.argtypes = [P, C.c_int, C.c_int, dp, C.c_double]
    if hasattr(lib, "bte_set_bc_partial"):
        lib.bte_set_bc_partial.argtypes = [P, C.c_int, C.c_double]
    lib.bte_set_state.argtypes = [P, dp, dp]
    lib.bte_init_random.argtypes = [P, C.c_uint64, dp, C.c_double, C.c_double, C.c_double]
    lib.bte_step.argtypes = [P, C.c_int64]
    lib.bte_group_step.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int64]
    lib.bte_get_intensity.argtypes = [P, dp, C.c_size_t]
    lib.bte_get_temperature.argtypes = [P, dp, C.c_size_t]
    lib.bte_get_energy.argtypes = [P, C.POINTER(C.c_double)]
    lib.bte_debug_substep.argtypes = [P, C.c_int, dp, C.c_size_t]
    lib.bte_set_debug.argtypes = [P, C.c_int, C.c_int]
    lib.bte_set_implicit.argtypes = [P, C.c_int, C.c_double]
    lib.bte_mesh_read.argtypes = [C.c_char_p, C.POINTER(C.POINTER(MeshDataC))]
    lib.bte_mesh_free.argtypes = [C.POINTER(MeshDataC)]
    lib.bte_mesh_free.restype = None
    lib.bte_mesh_error.restype = C.c_char_p
    lib.bte_partition_rcb.argtypes = [C.POINTER(UMeshC), C.c_int, C.c_void_p]
    lib.bte_get_iterations.argtypes = [P, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    lib.bte_timing_enable.argtypes = [P, C.c_int, C.c_int64]
    lib.bte_timing_read.argtypes = [P, C.POINTER(Timing)]
    lib.bte_get_info.argtypes = [P, C.POINTER(Info)]
    lib.bte_plan_slab.argtypes = [C.POINTER(Mesh), C.POINTER(Dirs), C.c_int, C.c_int, C.c_int, C.POINTER(SlabPlan)]
    lib.bte_last_error.argtypes = [P]
    lib.bte_last_error.restype = C.c_char_p
    lib.bte_destroy.argtypes = [P]
    lib.bte_destroy.restype = None
    lib.bte_version.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("bte_last_error", "bte_destroy", "bte_version", "bte_mesh_free", "bte_mesh_error") and \
                hasattr(lib, name):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _f64(a) -> Optional[np.ndarray]:
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class Solver:
    """One BTE context on one GPU: the whole problem, one slab of the mesh
    (decomp="slab", nranks > 1) or one band of channels (decomp="band",
    bte_create_band: rank = band part, nranks = parts)."""

    def __init__(self, mesh, dirs, bands, dt: float, T_init: float, device: int = 0, stream=None,
                 rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 torch_alloc: bool = True, decomp: str = "slab", step_mode: int = 0):
        if decomp not in ("slab", "band"):
            raise ValueError("decomp must be 'slab' or 'band'")
        import torch  # plumbing: device memory and streams
        if not torch.cuda.is_available():
            raise RuntimeError("libbte needs a CUDA device (no CPU fallback)")
        self._lib = load_library()
        self._torch = torch
        self.device = device
        torch.cuda.set_device(device)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._keep = []
        k = self._keep.append

        self.umesh = hasattr(mesh, "cells")
        if self.umesh:  # unstructured simplex mesh (bte_create_umesh)
            if decomp != "slab":
                raise ValueError("unstructured meshes partition by cells (decomp='slab')")
            verts = np.ascontiguousarray(mesh.verts, dtype=np.float64)
            cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
            k(verts), k(cells)
            m = UMeshC(int(mesh.dim), verts.shape[0], _p(verts), cells.shape[0], _p(cells), float(mesh.depth),
                       int(cells.shape[1]))
        else:
            m = Mesh(mesh.dim, mesh.nx, mesh.ny, mesh.nz, mesh.dx, mesh.dy, mesh.dz)
        s, w = _f64(dirs.s), _f64(dirs.w)
        k(s), k(w)
        d = Dirs(int(w.shape[0]), _p(s), _p(w))
        arrs = {}
        for name in ("v", "I_ref", "slope", "w_lo", "w_hi", "vs", "c2", "g", "beta_coef"):
            a = _f64(getattr(bands, name, None))
            arrs[name] = a
            if a is not None:
                k(a)
        b = Bands(int(arrs["v"].shape[0]), _p(arrs["v"]), int(bands.mode), _p(arrs["I_ref"]),
                  _p(arrs["slope"]), float(getattr(bands, "T_ref", 300.0)), _p(arrs["w_lo"]),
                  _p(arrs["w_hi"]), _p(arrs["vs"]), _p(arrs["c2"]), _p(arrs["g"]), _p(arrs["beta_coef"]))
        if torch_alloc:
            def _alloc(nbytes, _ctx):
                return torch.cuda.caching_allocator_alloc(int(nbytes), device, self.stream)

            def _free(ptr, _ctx):
                torch.cuda.caching_allocator_delete(ptr)

            self._alloc_cb, self._free_cb = ALLOC_FN(_alloc), DEALLOC_FN(_free)
        else:
            self._alloc_cb, self._free_cb = ALLOC_FN(), DEALLOC_FN()
        idbuf = None
        if nranks > 1 and nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be the 128-byte ncclUniqueId")
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            k(idbuf)
        run = Run(float(dt), float(T_init), int(device), C.c_void_p(self.stream.cuda_stream), int(rank),
                  int(nranks), C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                  self._alloc_cb, self._free_cb, None, int(step_mode))
        h = C.c_void_p()
        create = self._lib.bte_create_band if decomp == "band" else self._lib.bte_create
        if self.umesh:
            create = self._lib.bte_create_umesh
        st = create(C.byref(m), C.byref(d), C.byref(b), C.byref(run), C.byref(h))
        self._h = h
        if st != BTE_OK:
            msg = self._err()
            self.close()
            raise BteError(st, msg)
        info = Info()
        self._check(self._lib.bte_get_info(self._h, C.byref(info)))
        self.ncells = int(info.ncells_local)
        self.ncells_global = int(info.ncells_global)
        self.z0 = int(info.z0)
        self.nz_local = int(info.nz_local)
        self.nd, self.nb = int(info.nd), int(info.nb)
        self.n_octants, self.nj = int(info.n_octants), int(info.nj)
        self.bytes_state = int(info.bytes_state)
        self.b0, self.b1, self.nb_total = int(info.b0), int(info.b1), int(info.nb_total)
        self.band = bool(info.band)
        self.rotate = bool(info.rotate)
        self.cell0 = int(info.cell0)
        self.sweep_kernel = (info.sweep_kernel or b"").decode()
        self.newton_kernel = (info.newton_kernel or b"").decode()
        if self.nb_total == 0:  # older A/B build without the band fields
            self.b0, self.b1, self.nb_total = 0, self.nb, self.nb

    # ---------------------------------------------------------------- helpers
    @classmethod
    def from_problem(cls, problem, **kw) -> "Solver":
        """Build from a problem description (mesh/dirs/bands/dt/T_init/bcs)."""
        kw.setdefault("step_mode", 2 if getattr(problem, "implicit", 0) else int(getattr(problem, "semi", 0)))
        sv = cls(problem.mesh, problem.dirs, problem.bands, problem.dt, problem.T_init, **kw)
        if getattr(problem, "implicit", 0):
            sv.set_implicit(int(problem.imp_max_iter), float(problem.imp_tol))
        nreg = 6 if problem.mesh.dim == 3 else 4
        for r in range(nreg):
            sv.set_wall(r, problem.bcs[r])
        if getattr(problem, "tau_mode", 0):
            sv.set_tau_mode(problem.tau_mode)
        return sv

    def _err(self) -> str:
        if not self._h:
            return "no context"
        return self._lib.bte_last_error(self._h).decode(errors="replace")

    def _check(self, st: int):
        if st != BTE_OK:
            raise BteError(st, self._err())

    # ---------------------------------------------------------------- API
    def set_bc(self, region: int, kind: int, T_wall=None, T_uniform: float = 300.0, specularity: float = 1.0):
        if int(kind) == BC_PARTIAL:
            self._check(self._lib.bte_set_bc_partial(self._h, int(region), float(specularity)))
            return
        Tw = _f64(T_wall)
        if Tw is not None and Tw.size != self.region_faces(region):
            raise ValueError(f"T_wall has {Tw.size} values, region {region} has {self.region_faces(region)} faces")
        self._check(self._lib.bte_set_bc(self._h, int(region), int(kind), _p(Tw), float(T_uniform)))

    def set_step_mode(self, mode: int) -> None:
        """0: explicit step; 1: semi-implicit (explicit advection, implicit relaxation; reading R-l)."""
        self._check(self._lib.bte_set_step_mode(self._h, int(mode)))

    def set_implicit(self, max_iter: int, tol: float) -> None:
        """Source iterations per implicit step (reading R-n): at most max_iter, early stop at tol (0: exactly max_iter)."""
        self._check(self._lib.bte_set_implicit(self._h, int(max_iter), float(tol)))

    def iterations(self) -> np.ndarray:
        """Iterations of each step of the last step() call in implicit mode."""
        n = C.c_int64()
        self._check(self._lib.bte_get_iterations(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int64)
        if n.value:
            self._check(self._lib.bte_get_iterations(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def set_tau_mode(self, mode: int) -> None:
        """0: lagged tau (default); 1: self-consistent tau(T^{n+1}) (reading R-k)."""
        self._check(self._lib.bte_set_tau_mode(self._h, int(mode)))

    def intensity_cells(self, cells) -> np.ndarray:
        """Intensities [len(cells), nd, nb] of selected local cells (canonical order)."""
        idx = np.ascontiguousarray(cells, dtype=np.int64)
        out = np.empty((idx.size, self.nd, self.nb))
        self._check(self._lib.bte_get_intensity_cells(self._h, _p(idx), idx.size, _p(out)))
        return out

    def region_faces(self, region: int) -> int:
        """Boundary faces of wall region 0..5 (the T_wall length of set_bc)."""
        n = C.c_int64()
        self._check(self._lib.bte_get_region_faces(self._h, int(region), C.byref(n)))
        return int(n.value)

    def set_wall(self, region: int, bc) -> None:
        """Apply a wall description (kind, T_wall, T_uniform[, specularity])."""
        self.set_bc(region, bc.kind, bc.T_wall, bc.T_uniform, getattr(bc, "specularity", 1.0))

    def set_state(self, I=None, T=None):
        I, T = _f64(I), _f64(T)
        if I is not None and I.size != self.ncells * self.nd * self.nb:
            raise ValueError("I has the wrong size")
        if T is not None and T.size != self.ncells:
            raise ValueError("T has the wrong size")
        self._check(self._lib.bte_set_state(self._h, _p(I), _p(T)))

    def init_random(self, seed: int, phase: Sequence[float], T_mean: float, T_amp: float, I_amp: float):
        ph = _f64(list(phase) + [0.0] * (3 - len(phase)))
        self._check(self._lib.bte_init_random(self._h, C.c_uint64(seed & (2 ** 64 - 1)), _p(ph), T_mean,
                                              T_amp, I_amp))

    def step(self, n: int = 1):
        self._check(self._lib.bte_step(self._h, int(n)))

    @staticmethod
    def group_step(solvers, n: int = 1):
        """Advance an in-process slab or band group (contexts built with nranks =
        len(solvers), rank = index, no nccl_id) by n steps; halos (slab) or the
        per-cell band partials (band) move by device-to-device copies."""
        lib = load_library()
        arr = (C.c_void_p * len(solvers))(*[sv._h.value for sv in solvers])
        st = lib.bte_group_step(arr, len(solvers), int(n))
        if st != BTE_OK:
            msgs = "; ".join(sv._err() for sv in solvers if sv._err())
            raise BteError(st, msgs)

    @staticmethod
    def _out(out: Optional[np.ndarray], shape) -> np.ndarray:
        """Caller buffers must be C-contiguous float64 of the exact size (the
        library writes 8*size bytes into them)."""
        if out is None:
            return np.empty(shape)
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != int(np.prod(shape)):
            raise ValueError(f"out must be a C-contiguous float64 array of {int(np.prod(shape))} elements")
        return out

    def intensity(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = self._out(out, (self.ncells, self.nd, self.nb))
        self._check(self._lib.bte_get_intensity(self._h, out.ctypes.data, out.size))
        return out

    def temperature(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = self._out(out, (self.ncells,))
        self._check(self._lib.bte_get_temperature(self._h, out.ctypes.data, out.size))
        return out

    def set_debug(self, what: int, value: int) -> None:
        """Mutation-test switches (bte_set_debug); never on a production run."""
        self._check(self._lib.bte_set_debug(self._h, int(what), int(value)))

    def energy(self) -> float:
        e = C.c_double()
        self._check(self._lib.bte_get_energy(self._h, C.byref(e)))
        return e.value

    def debug_substep(self, which: int) -> np.ndarray:
        shape = {0: (self.ncells, self.nd, self.nb), 1: (self.ncells, self.nb), 2: (self.ncells, self.nb_total),
                 3: (self.ncells, self.nb_total)}[which]
        out = np.empty(shape)
        self._check(self._lib.bte_debug_substep(self._h, which, out.ctypes.data, out.size))
        return out

    def timing_enable(self, enable: bool = True, max_steps: int = 4096):
        self._check(self._lib.bte_timing_enable(self._h, int(enable), int(max_steps)))

    def timing_read(self) -> dict:
        t = Timing()
        self._check(self._lib.bte_timing_read(self._h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in Timing._fields_}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.bte_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def plan_slab(mesh, dirs, nb: int, nranks: int, rank: int) -> dict:
    """The library's slab decomposition + halo plan for one rank (host-only call;
    the same list bte_step executes with NCCL)."""
    lib = load_library()
    m = Mesh(mesh.dim, mesh.nx, mesh.ny, mesh.nz, mesh.dx, mesh.dy, mesh.dz)
    s, w = _f64(dirs.s), _f64(dirs.w)
    d = Dirs(int(w.shape[0]), _p(s), _p(w))
    out = SlabPlan()
    st = lib.bte_plan_slab(C.byref(m), C.byref(d), int(nb), int(nranks), int(rank), C.byref(out))
    if st != BTE_OK:
        raise BteError(st, "bte_plan_slab")
    msgs = [{f: getattr(out.msg[k], f) for f, _ in Msg._fields_} for k in range(out.n_msgs)]
    return {"axis": out.axis, "m0": out.m0, "n_local": out.n_local, "msgs": msgs}


def plan_band(nb: int, nparts: int, part: int) -> tuple:
    """The library's band partition: channels [b0, b1) of part `part` (host-only)."""
    lib = load_library()
    b0, b1 = C.c_int(), C.c_int()
    st = lib.bte_plan_band(int(nb), int(nparts), int(part), C.byref(b0), C.byref(b1))
    if st != BTE_OK:
        raise BteError(st, "bte_plan_band")
    return b0.value, b1.value


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (rank 0), via the NCCL library PyTorch ships."""
    import torch  # noqa: F401  (loads libnccl.so.2)
    nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    buf = C.create_string_buffer(128)
    st = nccl.ncclGetUniqueId(buf)
    if st != 0:
        raise RuntimeError(f"ncclGetUniqueId failed ({st})")
    return buf.raw


def loopback_unique_id() -> bytes:
    """A fresh id for the in-process loopback transport (include/bte.h, bte_run):
    ranks as threads of one process, exchanges as device copies -- the
    multi-rank code path on one GPU (test infrastructure)."""
    return b"BTELOOP\0" + os.urandom(16) + bytes(104)


def plan_umesh(mesh, nranks: int, rank: int) -> dict:
    """bte_plan_umesh (host only): the cell partition libbte uses for an
    unstructured mesh -- owned range, halo cells (canonical), per-peer lists."""
    lib = load_library()
    verts = np.ascontiguousarray(mesh.verts, dtype=np.float64)
    cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
    m = UMeshC(int(mesh.dim), verts.shape[0], _p(verts), cells.shape[0], _p(cells), float(mesh.depth),
               int(cells.shape[1]))
    out = UPlanC()
    cap = int(cells.shape[0]) * int(cells.shape[1])
    halo = np.empty(cap, dtype=np.int64)
    send = np.empty(cap, dtype=np.int64)
    st = lib.bte_plan_umesh(C.byref(m), int(nranks), int(rank), C.byref(out), _p(halo), cap, _p(send), cap)
    if st != BTE_OK:
        raise BteError(st, "bte_plan_umesh")
    peers = [dict(peer=out.peer[k].peer, recv_off=out.peer[k].recv_off, recv_cnt=out.peer[k].recv_cnt,
                  send=send[out.peer[k].send_off:out.peer[k].send_off + out.peer[k].send_cnt].copy())
             for k in range(out.n_peers)]
    return dict(cell0=out.cell0, n_own=out.n_own, n_halo=out.n_halo, halo=halo[:out.n_halo].copy(), peers=peers)


def read_mesh(path: str, depth: float = 1.0):
    """bte_mesh_read (host only): a Gmsh (ASCII 2.2 / 4.1) or MEDIT .mesh file as
    a bte_inputs.UMesh (vertex coordinates [n, 3], cells [nc, m] 0-based)."""
    import bte_inputs as bi
    lib = load_library()
    out = C.POINTER(MeshDataC)()
    st = lib.bte_mesh_read(os.fsencode(path), C.byref(out))
    if st != BTE_OK:
        raise BteError(st, lib.bte_mesh_error().decode(errors="replace"))
    try:
        m = out.contents
        verts = np.ctypeslib.as_array(m.verts, shape=(m.nverts, 3)).copy()
        cells = np.ctypeslib.as_array(m.cells, shape=(m.ncells, m.nvc)).copy()
        return bi.UMesh(int(m.dim), verts, cells, float(depth))
    finally:
        lib.bte_mesh_free(out)


def partition_rcb(mesh, nparts: int) -> np.ndarray:
    """bte_partition_rcb (host only): a cell permutation whose ranges
    [r N/P, (r+1) N/P) are compact parts (recursive coordinate bisection)."""
    lib = load_library()
    verts = np.ascontiguousarray(mesh.verts, dtype=np.float64)
    cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
    m = UMeshC(int(mesh.dim), verts.shape[0], _p(verts), cells.shape[0], _p(cells), float(mesh.depth),
               int(cells.shape[1]))
    perm = np.empty(cells.shape[0], dtype=np.int64)
    st = lib.bte_partition_rcb(C.byref(m), int(nparts), _p(perm))
    if st != BTE_OK:
        raise BteError(st, lib.bte_mesh_error().decode(errors="replace"))
    return perm
