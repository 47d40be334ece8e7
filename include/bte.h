/*
 * bte.h -- C ABI of the B200-native explicit phonon-BTE time step
 * (arXiv 2305.19400, "Automating GPU Scalability for Complex Scientific
 * Models: Phonon Boltzmann Transport Equation").
 *
 * One step (all on the GPU, no host callbacks):
 *   a1  boundary pass: ghost intensities from I^n           (Eq. 6)
 *   a2  fused upwind-flux + relaxation sweep -> I^{n+1}      (Eq. 5, P:L378-387,
 *       forward Euler Eqs. 2-3; upwind P:L150-157)
 *       with the per-(cell, octant, band) partial sum of w_d (I0c - I^{n+1})
 *   a3  per-cell reduction over directions and bands
 *   a4  per-cell Newton for T^{n+1} against I0_b(T); refresh I0c, beta
 *
 *   a5  (nranks > 1) slab halo exchange of boundary planes
 * "P:L<a>-<b>" = lines of /root/reference/PAPER.md; readings #n = DESIGN.md.
 *
 * Units: SI (m, s, K, rad/s); intensities in W m^-2 sr^-1 per channel.
 * Precision: IEEE fp64 throughout (fp32 "did not provide adequate
 * precision").
 *
 * Conventions (all functions):
 *  - Every pointer argument documented "host" is caller-owned and only read
 *    (or written, for outputs) during the call; the library copies what it
 *    needs.  Device memory is owned by the context, obtained through
 *    run->alloc/dealloc when given (PyTorch's caching allocator from Python),
 *    else cudaMalloc/cudaFree, and released by bte_destroy.
 *  - Canonical external orders: cell c = x + nx*(y + ny*z); intensity
 *    arrays are [cell][d][b] (d = index into the caller's direction table,
 *    b = channel), row-major, fp64.
 *  - Errors: a bte_status is returned; nothing throws across the ABI.  A
 *    human-readable message is available from bte_last_error(ctx).  Device-side
 *    failures (Newton non-convergence, non-finite values) are latched in a
 *    device word and reported by the bte_step call that observed them, with
 *    the step and cell index in the message; the state is then undefined.
 *  - Threading: one context per device per process; calls on one context are
 *    not thread-safe.  All work is ordered on run->stream (a cudaStream_t, or
 *    NULL for the legacy default stream).
 */
#ifndef BTE_H
#define BTE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BTE_API __attribute__((visibility("default")))
#else
#define BTE_API
#endif

typedef struct bte_ctx bte_ctx;

typedef enum {
  BTE_OK = 0,
  BTE_EINVAL = 1,      /* invalid argument / size / table                         */
  BTE_ENOMEM = 2,      /* device allocation failed                                */
  BTE_ECUDA = 3,       /* CUDA runtime error (message has cudaGetErrorString)     */
  BTE_ENCCL = 4,       /* NCCL error (multi-rank)                                 */
  BTE_EUNSTABLE = 5,   /* dt violates 1 - dt*beta_max - dt*v_b*sum|s_a|/D_a >= 0  */
  BTE_ENOTCLOSED = 6,  /* specular wall: reflected direction not in the set      */
  BTE_ENEWTON = 7,     /* temperature Newton did not converge in 50 iterations   */
  BTE_ENONFINITE = 8   /* NaN/Inf reached the temperature update                 */
} bte_status;

typedef enum {
  BTE_BC_ISOTHERMAL = 0, /* ghost = I0_b(T_wall(face)) for incoming d (Eq. 6 case 1) */
  BTE_BC_SPECULAR = 1,   /* ghost = I_{r(d),b} of the boundary cell (Eq. 6 case 2;  */
                         /* "symmetry" walls of the paper)                          */
  BTE_BC_DIFFUSE = 2,    /* adiabatic diffuse wall: ghost_b = sum_out w|s_a| I /     */
                         /* sum_in w|s_a|, same for every incoming d (reading #11)  */
  BTE_BC_PARTIAL = 3     /* partially specular adiabatic wall (SURVEY 8(f) f4,      */
                         /* DESIGN reading R-i): ghost = p*I_{r(d),b} + (1-p)*the   */
                         /* diffuse ghost; set with bte_set_bc_partial              */
} bte_bc_kind;

typedef enum {
  BTE_I0_LINEAR = 0,        /* I0_b(T) = I_ref[b] + slope[b]*(T - T_ref)   */
  BTE_I0_BOSE_EINSTEIN = 1  /* g hbar/(8 pi^3) int w k(w)^2/(exp(hbar w/kB T)-1) dw,      */
                            /* 16-point Gauss-Legendre per channel (reading #1)         */
} bte_i0_mode;

/* Uniform structured mesh.  dim = 2 or 3; for dim 2,
 * nz must be 1 and dz is the (unit) depth used for cell volumes only.
 * Wall regions: 0..5 = -x, +x, -y, +y, -z, +z (4, 5 unused for dim 2). */
typedef struct {
  int dim;
  int64_t nx, ny, nz;
  double dx, dy, dz;
} bte_mesh;

/* Discrete directions.  s: host [nd][3] unit vectors,
 * w: host [nd] weights.  Directions are grouped by octant (sign pattern of s;
 * a zero component counts as +); every non-empty octant must hold the same
 * number of directions.  Reflection maps are derived by bit-exact matching. */
typedef struct {
  int nd;
  const double *s;
  const double *w;
} bte_dirs;

/* Channels ("bands").  All arrays host, length nb, except
 * beta_coef [nb][5] = {p0, p3, p4, pu, theta}:
 *   beta_b(T) = 1/tau_b(T) = p0 + p3*T^3 + p4*T^4 + pu/sinh(theta/T)  (pu = 0 drops
 *   the term), all coefficients >= 0 (readings #3, #15).
 * LINEAR mode uses I_ref, slope, T_ref; BOSE_EINSTEIN uses w_lo, w_hi (band
 * edges, rad/s), vs, c2 (dispersion w = vs*k + c2*k^2), g (degeneracy). */
typedef struct {
  int nb;
  const double *v; /* group speed |v_g|_b, m/s (> 0) */
  int mode;        /* bte_i0_mode */
  const double *I_ref, *slope;
  double T_ref;
  const double *w_lo, *w_hi, *vs, *c2, *g;
  const double *beta_coef;
} bte_bands;

/* Run parameters.  stream: cudaStream_t (NULL = legacy default stream).
 * alloc/dealloc: optional device allocator (bytes, alloc_ctx) -> 256-B aligned
 * pointer / (ptr, alloc_ctx); NULL -> cudaMalloc/cudaFree.
 * rank/nranks/nccl_id: multi-GPU slab decomposition along the slowest axis
 * (z for dim 3, y for dim 2); nccl_id = 128-byte ncclUniqueId broadcast by the
 * caller (e.g. through torch.distributed), ignored when nranks == 1.
 * An nccl_id whose first 7 bytes are "BTELOOP" selects the in-process loopback
 * transport instead of NCCL (test infrastructure): the ranks are threads of one
 * process sharing that id, every send/recv/AllGather is matched across them at
 * group end and executed as stream-ordered device copies, so the multi-rank
 * code path runs on one GPU; a rank that never reaches an exchange makes its
 * peers fail with BTE_ENCCL after 120 s. */
typedef struct {
  double dt;
  double T_init;
  int device;
  void *stream;
  int rank, nranks;
  const void *nccl_id;
  void *(*alloc)(size_t bytes, void *alloc_ctx);
  void (*dealloc)(void *ptr, void *alloc_ctx);
  void *alloc_ctx;
  int step_mode;  /* 0: explicit step (Eq. 5 + forward Euler); 1: semi-implicit (reading
                     R-l: explicit advection, implicit relaxation); 2: implicit step by
                     source iteration (reading R-n); see bte_set_step_mode */
} bte_run;

/* Create a context: validates tables (positive sizes/speeds, equal octant
 * populations, W > 0), precomputes geometry and coefficient tables, allocates
 * the state and initialises it to equilibrium at T_init (I = I0_b(T_init)).
 * All walls start SPECULAR; call bte_set_bc to change them.
 * Intensity storage: two full buffers (I^n, I^{n+1}) when they fit in free
 * device memory next to ~2 GB of tables, else octant-slot rotation (SURVEY
 * 7.3 #1): one buffer of (octants + 1) slot regions, each octant swept from
 * its region into the spare one, specular ghosts snapshotted first -- e.g.
 * 144 GB instead of 256 GB for 10^6 cells x 400 directions x 40 channels.
 * Same results bit for bit; env BTE_ROTATE=0/1 overrides the choice;
 * bte_info.rotate reports it.  bte_debug_substep 0/1 are unavailable then.
 * Errors: BTE_EINVAL, BTE_ENOMEM, BTE_ECUDA, BTE_EUNSTABLE, BTE_ENCCL. */
BTE_API bte_status bte_create(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                      const bte_run *run, bte_ctx **out);

/* Create a band-partitioned context.
 * Arguments as bte_create with the FULL channel table; run->rank and
 * run->nranks are this context's band part and the number of parts.  Every
 * part holds the whole mesh (no halo planes) and sweeps only its channels
 * [b0, b1) (bte_plan_band).  Per step the parts exchange ONE scalar per cell,
 * S_r(c) = sum_{b in part r} c_b D_{c,b} (c_b = beta_b(T^n)/v_b, Eq. 8's
 * weights): ncclAllGather of [nranks][ncells] when run->nccl_id is set, device
 * copies inside bte_group_step when it is NULL ("local" mode, as for slabs).
 * Every part then sums the gathered partials in rank order and runs the same
 * temperature Newton over all channels, so T is bitwise identical on all
 * parts.  State: I holds this part's channels, canonical [cell][d][b - b0]
 * (nd*(b1-b0) doubles per cell); T is the whole field; bte_set_state needs
 * T; bte_get_energy sums this part's channels only; bte_debug_substep
 * which = 2/3 return all nb_total channels.  Errors as bte_create. */
BTE_API bte_status bte_create_band(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                                   const bte_run *run, bte_ctx **out);

/* Unstructured mesh.  The finite-volume step is
 * Eq. 3 for m-sided cells with the upwind face value of
 * I' = I + dt*(beta (I0c - I) - v_b sum_f (A_f/V_c)(s_d.n_f) I_up).
 *   dim 2: triangles (nvc 3) or convex quadrilaterals (nvc 4), verts z
 *          ignored, depth = z extent; face k = edge (v_{k+1}, v_{k+2})
 *          (for a triangle: the edge opposite v_k);
 *   dim 3: tetrahedra, cells[c][0..3]; face k = the face opposite v_k;
 *          or hexahedra (nvc 8, Gmsh order: bottom 0-1-2-3, top 4-5-6-7),
 *          faces (0,1,2,3) (4,5,6,7) (0,1,5,4) (1,2,6,5) (2,3,7,6) (3,0,4,7),
 *          each the bilinear patch through its corners: A_f n_f =
 *          (q2 - q0) x (q3 - q1)/2 away from the vertex mean, V_c from the
 *          divergence theorem (exact for such faces).  The domain is
 * the axis-aligned bounding box of the vertices; every face without a
 * neighbour must lie on one of its walls (all face vertices at x = xmin ->
 * region 0, x = xmax -> 1, y -> 2/3, z -> 4/5, tested in that order).  Wall
 * faces are numbered per region in (cell, local face) ascending order: that
 * is the order of bte_set_bc's T_wall array (bte_get_region_faces gives the
 * count).  Arrays are host memory, read during the call only. */
typedef struct {
  int dim;               /* 2 or 3 */
  int64_t nverts;
  const double *verts;   /* [nverts][3], metres */
  int64_t ncells;
  const int64_t *cells;  /* [ncells][nvc] vertex indices */
  double depth;          /* dim 2: z extent (volumes and face areas scale with it) */
  int nvc;               /* vertices per cell: 0 -> dim + 1 (simplices); dim 2 also 4
                            (convex quadrilaterals, vertices in boundary order:
                            Eq. 3's "polygonal cell with m sides");
                            dim 3 also 8 (hexahedra) */
} bte_umesh;

/* Create a single-GPU context on an unstructured mesh.  Geometry precompute
 * (a0) on the host: A_f n_f / V_c per (cell, face) without square roots
 * (triangle: 2 perp(edge)/|cross|; tetrahedron: 3 cross/|det|, oriented away
 * from the opposite vertex), face matching by vertex sets, wall regions.
 * State layout, set_state/get_* orders, the temperature update and the wall
 * kinds are as for bte_create (canonical cell index = position in cells).
 * run->nranks > 1 partitions the mesh: rank r owns the
 * contiguous canonical cell range [r*nc/P, (r+1)*nc/P) (bte_info.cell0 /
 * ncells_local; state I/O covers those cells) and keeps read-only halo copies
 * of the face neighbours owned elsewhere, refreshed after every step by NCCL
 * send/recv (run->nccl_id) or device copies inside bte_group_step (local
 * mode).  Every rank must pass the whole mesh.  Octant-slot rotation is not
 * used.  The dt check is the general positivity
 * bound 1 - dt beta_b - dt v_b max_c sum_{f: s.n>0} (A_f/V_c) s.n >= 0.
 * Errors: BTE_EINVAL (degenerate cell, bad vertex index, a face shared by more
 * than two cells, a boundary face off the box walls, nranks != 1, or as
 * bte_create), BTE_EUNSTABLE, BTE_ENOMEM, BTE_ECUDA. */
BTE_API bte_status bte_create_umesh(const bte_umesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                                    const bte_run *run, bte_ctx **out);

/* Mesh import ("A mesh must either be imported
 * from a Gmsh or MEDIT formatted mesh file, or generated internally").
 * Host only, no GPU.  Reads an ASCII Gmsh file (format 2.2 or 4.1: $Nodes,
 * $Elements; element types 2 triangle, 3 quadrangle, 4 tetrahedron, 5
 * hexahedron; points and lines are boundary tags and skipped; other sections
 * ignored) or a MEDIT .mesh file (Dimension, Vertices, Triangles /
 * Quadrilaterals / Tetrahedra / Hexahedra, 1-based, with references; Edges /
 * Corners skipped).  The cells are the 3-D elements when present (tetrahedra
 * or hexahedra, not both; triangles / quadrilaterals are then boundary
 * faces), else the triangles or the quadrilaterals (not both).  Node order of the file is kept
 * (Gmsh node tags are mapped to their position).  *out is allocated by the
 * library: verts [nverts][3] (z = 0 for 2-D files), cells [ncells][nvc]
 * 0-based; free it with bte_mesh_free.  The arrays plug into bte_umesh
 * (depth is the caller's).  Errors: BTE_EINVAL (unreadable file, malformed
 * record, binary Gmsh, prisms / pyramids, mixed cell kinds, index out of
 * range) with the reason in bte_mesh_error(). */
typedef struct {
  int dim, nvc;
  int64_t nverts, ncells;
  double *verts;
  int64_t *cells;
} bte_mesh_data;
BTE_API bte_status bte_mesh_read(const char *path, bte_mesh_data **out);
BTE_API void bte_mesh_free(bte_mesh_data *mesh);
BTE_API const char *bte_mesh_error(void); /* thread-local text of the last mesh-call failure */

/* Recursive coordinate bisection of an unstructured mesh into nparts
 * (host only): perm[0..ncells) receives a cell order in which part r is the
 * range [r ncells/nparts, (r+1) ncells/nparts) -- exactly the ranges
 * bte_create_umesh gives rank r of nparts -- and each part is a compact box
 * of cell centroids (the centroid set is split at the median of its longest
 * extent, recursively, parts sized as those ranges; ties by cell index; the
 * input order is kept inside a part).  Apply it as cells' = cells[perm] (and
 * state rows likewise) before bte_create_umesh.  The paper partitions with
 * Metis; any partition works with the halo exchange, this one
 * keeps halos small for meshes given in arbitrary order.  Errors: BTE_EINVAL
 * (nparts outside [1, ncells], bad mesh) with the reason in bte_mesh_error(). */
BTE_API bte_status bte_partition_rcb(const bte_umesh *mesh, int nparts, int64_t *perm);

/* Temperature-update rule for tau(T).
 *   mode 0 (default, reading #15): lagged, beta_next = beta_b(T^n) weights the
 *          Newton for T^{n+1} and the next sweep;
 *   mode 1 (reading R-k): self-consistent, the Newton solves
 *          sum_b (beta_b(T)/v_b) [W (I0_b(T) - I0c_b) + D_b] = 0 (beta' in F')
 *          and the next sweep uses beta_b(T^{n+1}).
 * Switching to mode 1 refreshes I0c and beta from the current T.  Identical
 * results in both modes when beta does not depend on T.
 * Errors: BTE_EINVAL (mode, band contexts, the fused-Newton variant). */
BTE_API bte_status bte_set_tau_mode(bte_ctx *ctx, int mode);

/* Time integrator (SURVEY 8(f) f4 "implicit per-step solvers").
 *   mode 0 (default): explicit forward-Euler step of Eq. 5;
 *   mode 1: semi-implicit step -- J = I^n - dt v_b sum_f (A_f/V)(s.n) I_up
 *           (explicit upwind advection), T^{n+1} from the energy balance with
 *           weights beta_b/(v_b (1 + dt beta_b)) on the reduction of J, then
 *           I^{n+1} = (J + dt beta_b I0_b(T^{n+1})) / (1 + dt beta_b).
 *           The dt bound keeps only the advection term (1 - dt v_b
 *           sum_a |s_a|/D_a >= 0), so stiff scattering no longer limits dt.
 *   mode 2: implicit step (reading R-n; "solvers take 10-20 iterations
 *           ... within each time step"): backward Euler for every term of
 *           Eq. 4/5, I' - I^n = dt[beta (I0(T') - I') - v_b sum_f (A_f/V)(s.n) I'_up],
 *           beta = beta(T^n), wall ghosts of I', T' from the scattering
 *           balance of I'; solved by source iteration -- per iteration k:
 *           wall data from I^k; a wavefront transport sweep per octant
 *           (every cell after its upwind neighbours, exact inversion of the
 *           upwind operator):
 *             I^{k+1} = I^n + [dt beta (I0c^k - I^n) + sum_a kk_a (I^{k+1}_up - I^n)]
 *                             / (1 + dt beta + sum_a kk_a),  kk_a = dt v_b |s_a|/D_a;
 *           then the lagged Newton (#18) for T^{k+1} with weights beta(T^n)/v_b
 *           and I0c^{k+1} = I0(T^{k+1}).  bte_set_implicit sets the iteration
 *           count and tolerance.  No dt bound (positive for every dt).  One
 *           structured context only (no band / unstructured / multi-rank /
 *           octant-slot rotation: every iteration re-reads I^n).
 * Also settable at creation through bte_run.step_mode (needed when dt
 * exceeds the explicit bound).  Errors: BTE_EINVAL (mode, band contexts,
 * self-consistent tau, the context kinds above), BTE_EUNSTABLE (switching to
 * the explicit step at a dt beyond its bound). */
BTE_API bte_status bte_set_step_mode(bte_ctx *ctx, int mode);

/* Source iterations of the implicit step (step mode 2): at most max_iter per
 * step (default 20); with tol > 0 (default 1e-10) a step stops early once both
 * inputs of its last sweep had settled -- max_c |T^{k+1} - T^k| / T^k <= tol
 * and the wall data (outgoing intensities of specular / partial wall cells,
 * diffuse ghost tables) changed by at most tol relative since the previous
 * iterate (the first iteration never stops while such walls exist).  tol = 0:
 * exactly max_iter iterations, no host synchronisation inside the step.
 * Errors: BTE_EINVAL (max_iter outside [1, 100000], tol < 0 or not finite). */
BTE_API bte_status bte_set_implicit(bte_ctx *ctx, int max_iter, double tol);

/* Iterations taken by each step of the last bte_step call in implicit mode:
 * *count = number of steps recorded, out[0 .. min(n, count)) their iteration
 * counts.  Errors: BTE_EINVAL. */
BTE_API bte_status bte_get_iterations(const bte_ctx *ctx, int64_t *out, int64_t n, int64_t *count);

/* Number of boundary faces of wall region 0..5 (the T_wall length of
 * bte_set_bc) for structured and unstructured contexts.  Errors: BTE_EINVAL. */
BTE_API bte_status bte_get_region_faces(const bte_ctx *ctx, int region, int64_t *nfaces);

/* Boundary condition of one wall region (0..5 = -x,+x,-y,+y,-z,+z).
 * T_wall: host array with one temperature per boundary face of that wall,
 * row-major over the two in-plane axes in (x,y,z) order ((y,z) for x-walls,
 * (x,z) for y-walls, (x,y) for z-walls), or NULL to use T_uniform.  Ignored
 * unless kind == BTE_BC_ISOTHERMAL.  Isothermal ghosts I0_b(T_wall) are
 * tabulated on the device once here.
 * Errors: BTE_EINVAL (region/kind), BTE_ENOTCLOSED (specular wall whose
 * reflections are not in the set), BTE_EUNSTABLE (T_wall raises beta_max past
 * the dt bound). */
BTE_API bte_status bte_set_bc(bte_ctx *ctx, int region, int kind, const double *T_wall, double T_uniform);

/* Partially specular adiabatic wall on region 0..5 (the
 * paper has only isothermal and symmetry walls, Eq. 6, so this is
 * reading R-i of DESIGN.md): for each incoming direction d and channel b
 *   ghost = p * I^n_{r(d),b} + (1 - p) * [sum_out w|s_a| I^n_b / sum_in w|s_a|]
 * (products rounded separately, then added: no FMA), i.e. the Ziman/Soffer
 * specularity-weighted mix of BTE_BC_SPECULAR and BTE_BC_DIFFUSE.  Zero net
 * energy flux per channel for any p.  p = 1 and p = 0 reproduce the specular
 * and diffuse walls bit for bit.
 * Errors: BTE_EINVAL (region, p outside [0, 1] or NaN, no direction crosses
 * the wall), BTE_ENOTCLOSED (reflections of the set not in the set). */
BTE_API bte_status bte_set_bc_partial(bte_ctx *ctx, int region, double specularity);

/* Replace the state from host arrays (canonical orders, this rank's slab).
 *  I != NULL, T != NULL : I and T as given; I0c = I0(T), beta = beta(T).
 *  I == NULL, T != NULL : equilibrium I_{c,d,b} = I0_b(T_c).
 *  I != NULL, T == NULL : T from one reduction + Newton solve starting at
 *                         T_init with beta_next = beta(T_init).
 * Sizes: I has ncells_local*nd*nb doubles, T has ncells_local doubles. */
BTE_API bte_status bte_set_state(bte_ctx *ctx, const double *I, const double *T);

/* Device-generated random start:
 *   T_c = T_mean + T_amp*sin(2pi(x/Lx+phase[0]))*sin(2pi(y/Ly+phase[1]))[*sin(2pi(z/Lz+phase[2]))]
 *   I_{c,d,b} = I0_b(T_c) * (1 + I_amp*(2u-1)),
 *   u = (splitmix64(seed ^ idx) >> 11) * 2^-53, idx = (c_global*nd + d)*nb + b.
 * x = (i+1/2)*dx is the cell centre (global coordinates under slab decomposition). */
BTE_API bte_status bte_init_random(bte_ctx *ctx, uint64_t seed, const double phase[3], double T_mean,
                           double T_amp, double I_amp);

/* Advance nsteps explicit steps on the context stream, then synchronise once
 * and check the device error word.  Errors: BTE_ENEWTON, BTE_ENONFINITE
 * (with step/cell in bte_last_error), BTE_ECUDA, BTE_ENCCL. */
BTE_API bte_status bte_step(bte_ctx *ctx, int64_t nsteps);

/* In-process slab group.  Contexts created in one process with nranks = n,
 * rank = 0..n-1 and nccl_id == NULL ("local" mode) form one slab-decomposed
 * problem whose halo planes are moved with device-to-device copies (same GPU,
 * or peers) instead of NCCL, following exactly the bte_plan_slab list.
 * bte_group_step advances all n contexts by nsteps (ctxs[r] must be rank r);
 * bte_step on a local-mode context returns BTE_EINVAL.  Errors as bte_step. */
BTE_API bte_status bte_group_step(bte_ctx **ctxs, int n, int64_t nsteps);

/* Copy state to caller-allocated host buffers (canonical order, this rank's
 * slab).  count must equal the exact element count: ncells_local*nd*nb for
 * the intensity, ncells_local for the temperature; else BTE_EINVAL. */
BTE_API bte_status bte_get_intensity(bte_ctx *ctx, double *out, size_t count);
/* Intensities of selected cells (this rank's local canonical indices, host
 * array of n), in canonical [i][d][b] order into host out (n*nd*nb doubles).
 * For sampled checks of states too large to copy whole.  Errors: BTE_EINVAL. */
BTE_API bte_status bte_get_intensity_cells(bte_ctx *ctx, const int64_t *cells, int64_t n, double *out);
BTE_API bte_status bte_get_temperature(bte_ctx *ctx, double *out, size_t count);

/* Diagnostic total energy E = sum_c V_c sum_b (1/v_b) sum_d w_d I_{c,d,b}
 * (SURVEY 8(b) "allreduced").  With an NCCL communicator
 * (nranks > 1, nccl_id given) E is the whole problem's: every rank sums its
 * own cells (or, for band contexts, its own channels), the per-rank sums are
 * all-gathered and added in rank order, so all ranks return the same bits.
 * Collective: every rank must call it.  Without a communicator (one context,
 * or an in-process local group) E covers this context only.  Not on the hot
 * path.  Errors: BTE_EINVAL, BTE_ENOMEM, BTE_ECUDA, BTE_ENCCL. */
BTE_API bte_status bte_get_energy(bte_ctx *ctx, double *E);

/* Debug switches for the mutation tests ("skipping the exchange must
 * break it").  BTE_DEBUG_SKIP_EXCHANGE: value 1 makes the halo / band-partial
 * exchange of this context's group a no-op (checked on the group's first
 * context).  Never set on a production run.  Errors: BTE_EINVAL (unknown what). */
#define BTE_DEBUG_SKIP_EXCHANGE 1
BTE_API bte_status bte_set_debug(bte_ctx *ctx, int what, int value);

/* Sub-step access for kernel unit tests (state unchanged):
 *   which = 0: I after one boundary pass + sweep from the current state, [cell][d][b]
 *   which = 1: the reduced deviation D_{c,b} = sum_d w_d (I0c - I^{n+1}), [cell][b]
 *   which = 2: current I0c [cell][b];  which = 3: current beta [cell][b]. */
BTE_API bte_status bte_debug_substep(bte_ctx *ctx, int which, double *out, size_t count);

/* Per-kernel device timing (CUDA events recorded on the context stream around
 * every launch while enabled; read out after the next bte_step). */
typedef struct {
  int64_t steps;           /* steps timed                                    */
  int64_t launches;        /* kernels launched by the library in those steps */
  double sweep_ms;         /* summed device time of the a1+a2 sweep launches  */
  double newton_ms;        /* summed device time of the a3+a4 launches        */
  double boundary_ms;      /* summed device time of the diffuse-ghost launches */
  double halo_ms;          /* summed time of the halo exchange (nranks > 1)   */
  int64_t sweep_launches;
  int64_t newton_launches;
  int64_t boundary_launches;
  int64_t truncated;       /* 1: the event pool (max_steps of bte_timing_enable) ran out; the
                              *_ms sums then miss launches the *_launches counts include */
} bte_timing;
BTE_API bte_status bte_timing_enable(bte_ctx *ctx, int enable, int64_t max_steps);
BTE_API bte_status bte_timing_read(bte_ctx *ctx, bte_timing *out);

/* Slab decomposition and halo plan for P ranks (P:L552-560 cell
 * partitioning).  Host-only (no CUDA call): the library's own halo exchange
 * (a5) executes exactly this list every step, after the sweep.  Planes are
 * split along the slowest axis (z for dim 3, y for dim 2): rank r owns
 * [m0, m0 + n_local) with the first (n mod P) ranks taking one extra plane.
 * For each octant whose slab-axis component points up (s >= 0), rank r sends
 * its last owned plane to r+1 and receives plane m0-1 from r-1; octants
 * pointing down do the mirror exchange.  msg[] lists this rank's messages in
 * execution order; `plane` is the global plane index sent or received. */
#define BTE_MAX_MSGS 32
typedef struct {
  int send;      /* 1 = send an owned plane, 0 = receive into a halo plane */
  int peer;      /* the other rank                                        */
  int octant;    /* sign pattern (4*[sx<0] + 2*[sy<0] + [sz<0]) moved     */
  int slot;      /* index of that octant among the non-empty ones         */
  int64_t plane; /* global plane index                                    */
  int64_t count; /* doubles in the message: cells per plane * Es, where   */
                 /* Es = nj*nb rounded up to even (device block stride)  */
} bte_msg;
typedef struct {
  int axis;        /* slab axis: 2 (z) for dim 3, 1 (y) for dim 2 */
  int64_t m0, n_local;
  int n_msgs;
  bte_msg msg[BTE_MAX_MSGS];
} bte_slab_plan;
BTE_API bte_status bte_plan_slab(const bte_mesh *mesh, const bte_dirs *dirs, int nb, int nranks, int rank,
                                 bte_slab_plan *out);

/* Band (channel) partition -- the paper's own multi-process decomposition
 * ("equation"/band partitioning): part `part` of
 * `nparts` owns the contiguous channels [*b0, *b1) of every cell,
 * b0 = floor(part*nb/nparts).  Host-only.  Errors: BTE_EINVAL unless
 * 1 <= nparts <= nb and 0 <= part < nparts. */
/* Partition plan of an unstructured mesh (host only, no GPU; what
 * bte_create_umesh builds for rank `rank` of `nranks`).  halo_cells (optional,
 * capacity halo_cap) receives the canonical indices of the halo copies in
 * halo order; send_cells (optional, capacity send_cap) the local indices of
 * the owned cells each peer holds, concatenated in peer order (peer[k].send_off).
 * Errors: BTE_EINVAL (mesh as bte_create_umesh, ranks, more than
 * BTE_MAX_MSGS peers, capacities too small). */
typedef struct {
  int peer;
  int64_t recv_off, recv_cnt; /* its cells in my halo: halo positions [off, off + cnt) */
  int64_t send_off, send_cnt; /* my cells in its halo: send_cells[off, off + cnt)       */
} bte_upeer;
typedef struct {
  int64_t cell0, n_own, n_halo;
  int n_peers;
  bte_upeer peer[BTE_MAX_MSGS];
} bte_umesh_plan;
BTE_API bte_status bte_plan_umesh(const bte_umesh *mesh, int nranks, int rank, bte_umesh_plan *out,
                                  int64_t *halo_cells, int64_t halo_cap, int64_t *send_cells, int64_t send_cap);

BTE_API bte_status bte_plan_band(int nb, int nparts, int part, int *b0, int *b1);

/* Sizes of this rank's slab and the layout.  nb is the channel count this
 * context sweeps (its band [b0, b1) of nb_total for a band context, else
 * b0 = 0 and nb = nb_total). */
typedef struct {
  int64_t ncells_local, ncells_global, z0, nz_local; /* slab along the slowest axis */
  int nd, nb, n_octants, nj;                         /* nj = directions per octant  */
  int64_t bytes_state;                               /* device bytes held by ctx    */
  int b0, b1, nb_total, band;                        /* channel band; band = 1 for bte_create_band */
  int rotate;                                        /* 1: octant-slot rotation (see bte_create)  */
  int64_t cell0;                                     /* canonical index of the first owned cell   */
  const char *sweep_kernel;                          /* the a1+a2 kernel bte_step launches (static) */
  int step_mode;                                     /* 0 explicit, 1 semi-implicit, 2 implicit     */
  const char *newton_kernel;                         /* the a3+a4 kernel of an explicit step (static) */
} bte_info;
BTE_API bte_status bte_get_info(const bte_ctx *ctx, bte_info *out);

BTE_API const char *bte_last_error(const bte_ctx *ctx);
BTE_API void bte_destroy(bte_ctx *ctx);

/* Library build identification (for the tests' symbol/ABI check). */
BTE_API const char *bte_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BTE_H */
