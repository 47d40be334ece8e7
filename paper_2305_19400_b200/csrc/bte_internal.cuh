// bte_internal.cuh -- device-side data layout and kernel interfaces of the
// B200 BTE step.  See DESIGN.md "Data layout in HBM" and include/bte.h.
//
// Layout (octant-major, band-innermost):
//   I[slot][plane][cross cell][j][b]   fp64
//     slot  = index of a non-empty octant (sign pattern of s_d), 0..nslot-1
//     plane = position along the slowest ("march") axis: z for dim 3, y for dim 2;
//             when nranks > 1 each slot holds nplanes+2 planes (one halo plane
//             on each side), else nplanes
//     cross = x + nx*y (dim 3) or x (dim 2)
//     j     = direction index inside the octant, b = channel
//   E = nj*nb doubles (16 KB at 50 x 40) are contiguous per (slot, cell).
//   I0c[c][b], beta[c][b], T[c], Dpart[c][slot][b] over the rank's own cells.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bte {

constexpr int kNGL = 16;        // Gauss-Legendre nodes per channel (reading #1)
constexpr int kMaxBands = 128;  // channels per context
constexpr int kMaxSlots = 8;
constexpr double kTlo = 1.0, kThi = 5000.0;  // Newton bracket (reading #18)
constexpr int kNewtonMaxIt = 50;
constexpr double kNewtonRtol = 1e-13;

enum { BC_ISO = 0, BC_SPEC = 1, BC_DIFF = 2, BC_PART = 3 };
enum { ERR_NONE = 0, ERR_NEWTON = 7, ERR_NONFINITE = 8 };

// Channel model tables (device pointers).
struct Material {
  int nb;
  int mode;               // 0 linear, 1 Bose-Einstein
  const double *v;        // [nb]
  const double *bcoef;    // [nb][5]
  const double *I_ref, *slope;
  double T_ref;
  const double *A;        // [nb][16] g hbar/(8pi^3) * half * wgl_j * w_j * k_j^2
  const double *X;        // [nb][16] hbar w_j / kB
  // uniform band grid (every channel spans [i*dw, (i+1)*dw], detected exactly):
  // exp(hbar w_ij / kB T) = exp(a u_j) r^i, a = Xd/T, r = exp(a), u_j = (1 + x_j)/2
  int uniform;
  int imax;
  double Xd;              // hbar dw / kB
  const double *U;        // [16] u_j
  const int *ichan;       // [imax+1][4] channels with band index i (-1 padded)
  int maxcnt;             // max channels sharing one band index
  const int *ib;          // [nb] band index i of each channel
  const double *rv;       // [nb] 1 / v_b
};

struct Geometry {
  int dim;
  int nx, ny;             // cross extents (dim 2: ny = 1 in the cross sense)
  int ncross;             // cells per plane
  int nplanes;            // owned planes along the march axis
  int64_t m0;             // global index of the first owned plane
  int64_t cell0;          // canonical index of the first owned cell (random start, errors)
  int64_t nplanes_global;
  int plane_off;          // 1 when halo planes are stored, else 0
  int64_t plane_stride;   // doubles per plane (ncross * E)
  int64_t slot_stride;    // doubles per slot
  int nslot, nj, nb, E;   // nb: channels this context sweeps
  int nbT, b0;            // band partition (bte_create_band): channels [b0, b0+nb) of nbT
                          // (else nbT = nb, b0 = 0); only the random-start counter uses them
  int Es;                 // (cell, octant) block stride in doubles: E rounded up to even (16-B TMA)
  int slot_oct[kMaxSlots];
  int oct_slot[8];        // inverse: slot of octant o, or -1
  int has_lo_wall, has_hi_wall;  // march-axis walls exist on this rank
  // per-(slot, j) coefficient table [nslot*nj][4]: dt|s_x|/dx, dt|s_y|/dy, dt|s_z|/dz, w
  const double *coef;
  // reflected element offset for specular ghosts: [3][nslot*nj] -> slot_r*slot_stride + jr*nb
  const int64_t *refl_off;
  // per-(slot, j) weight times |s_a| for the diffuse numerator: [3][nslot*nj]
  const double *ws;
  int kind[6];
  const double *gtab[6];  // iso / diffuse ghost tables [face][nb] (global face index)
  // where each octant slot of the CURRENT intensity buffer starts (doubles):
  // slot * slot_stride, or a rotated region under octant-slot rotation
  int64_t slot_off[kMaxSlots];
  int rot;                // octant-slot rotation: specular ghosts come from gspec snapshots
  const double *gspec[6]; // rot: [face][slot][j][nb] snapshot of the reflected I^n (specular walls)
  double diff_den[6];
  double spec_p[6], spec_q[6];  // BC_PART: specularity p and 1 - p (rounded on the host)
};

struct NewtonArgs {
  Material m;
  const double *Dpart;
  double *T, *I0c, *dI0c, *beta_next;
  int nslot, nb;
  int slot_oct[kMaxSlots];
  int oct_slot[8];        // slot of octant o, or -1 (register-indexed octant tree)
  double W;
  int64_t ncells, cell0_global;
  unsigned long long *err;
  int64_t step;           // step index for error reporting
  int col0, ncols;        // column (cross-cell) range of this launch
  int ncross, nplanes;
  const double *Sall;     // band partition: [nparts][ncells] gathered partials (else null)
  int nparts;
  double *I0s, *betas;    // band partition: the sweep's rows [c][nbs] = channels [b0s, b0s+nbs)
  int b0s, nbs;
  int predict;            // quadratic-convergence acceptance (reading R-f)
  int minb;               // k_newton occupancy variant (0 = default)
  double semi_dt;         // > 0: semi-implicit step weights beta/(v(1 + semi_dt beta)) (reading R-l)
  unsigned long long *stats;  // debug counters: [evaluations, final re-evaluations, cells solved] or null
  int sc_direct;          // self-consistent tau: direct band integrals even on uniform grids (A/B)
  int beta_fixed;         // implicit step (R-n): weights from the stored beta_next, not beta(T)
  unsigned long long *dTmax;  // implicit step: max_c |T^{k+1} - T^k| / T^k (double bits), or null
  const unsigned long long *step_ctr;  // graph replay: device step index for the error key (else `step`)
  int lpc;                // eval_channels: lane per channel (A/B)
};

struct SweepArgs {
  Geometry g;
  const double *Iin;
  double *Iout;
  const double *I0c, *beta;
  double *Dpart;
  const double *v;
  double dt;
  int seg_len;            // cells per CTA along the march axis
  int jpt;                // directions per thread (set by launch_sweep)
  int jg;                 // thread groups (set by launch_sweep)
  int use_tma;            // cp.async.bulk pipeline (k_sweep_tma) when the layout allows
  int stages;             // pipeline depth (set by launch_sweep)
  int stages_override;    // 0 = automatic
  int target_threads;     // CTA size target (0 = 448)
  int smem_budget_kb;     // per-CTA shared memory budget for the stage ring (0 = 113 KB)
  int64_t stage_doubles;  // doubles per stage (set by launch_sweep)
  int col0, ncols;        // column range of this launch (ncols = 0: all)
  int slot0, nslots;      // octant slots of this launch (nslots = 0: all)
  int64_t out_off[kMaxSlots];  // where slot s of I^{n+1} goes in Iout
  int p_lo, p_hi;         // owned-plane range of this launch (p_hi <= p_lo: all)
  int no_spare;           // 1: side jobs on compute threads (A/B switch read at create)
  int pf;                 // k_sweep: L2 prefetch distance in cells (0: off)
  int raster;             // 3-D column order: strips of `raster` columns along x (0: row-major)
};

// Unstructured simplex mesh, device view.  The state layout
// is the structured one with one "plane" of ncells cross cells:
// I[slot][cell][j][b], (cell, slot) blocks of Es doubles.
struct UMeshDev {
  int K;                  // faces per cell (triangle 3, tetrahedron / quadrilateral 4, hexahedron 6)
  int KP;                 // face slots per device row: 4 (K <= 4) or 8 (hexahedra)
  int64_t ncells;
  const int64_t *nbr;     // [nc][KP] (faces >= K unused): neighbour >= 0, or -1 - (face_in_region * 8 + region)
  const double *an;       // [nc][KP][3] (faces >= K unused): (A_f / V_c) n_f
  const double *sw;       // [nslot * nj][4]: s_x, s_y, s_z, w of direction (slot, j)
  const int64_t *rcell[6];  // owned wall faces: local cell
  const int64_t *rface[6];  // ... and their global face index (ghost-table row)
  int64_t rn[6];          // owned wall faces per region
};

struct USweepArgs {
  Geometry g;
  UMeshDev u;
  const double *Iin;
  double *Iout;
  const double *I0c, *beta;
  double *Dpart;
  const double *v;
  double dt;
  int jpt, jg;
  int target_threads;
  int pipelined;          // k_usweep_tma (default) vs the one-CTA-per-cell k_usweep
  int stages, chunk;      // pipeline depth and cells per CTA (0 = automatic)
  int generic;            // 1: skip the 40-channel x 50-direction specialisation (A/B)
  int single_buf;         // 1: one neighbour buffer, 2-deep ring, 2 CTAs/SM on triangles (A/B)
};

// kernels / launchers (kernels.cu)
cudaError_t launch_sweep(const SweepArgs &a, cudaStream_t s);
const char *sweep_kernel_name(const SweepArgs &a);
cudaError_t launch_newton(const NewtonArgs &a, cudaStream_t s);
cudaError_t launch_newton_sc(const NewtonArgs &a, cudaStream_t s);
cudaError_t launch_diffuse(const Geometry &g, const double *I, int region, double *gtab,
                           cudaStream_t s, unsigned long long *chg = nullptr);
cudaError_t launch_spec_snapshot(const Geometry &g, const double *I, int region, double *out, cudaStream_t s,
                                 unsigned long long *chg = nullptr);
cudaError_t launch_step_tick(unsigned long long *ctr, cudaStream_t s);
cudaError_t launch_sweep_imp(const SweepArgs &a, const int2 *tasks, int ntasks, int *prog, unsigned *ticket,
                             cudaStream_t s);
cudaError_t launch_iso_table(const Material &m, const double *Tw, int64_t nf, double *gtab,
                             cudaStream_t s);
cudaError_t launch_refresh(const Material &m, const double *T, int64_t nc, double *I0c,
                           double *dI0c, double *beta, cudaStream_t s);
cudaError_t launch_fill_equilibrium(const Geometry &g, const double *I0c, double *I,
                                    cudaStream_t s);
cudaError_t launch_permute(const Geometry &g, const int *dmap, int nd, const double *canon,
                           int64_t c0, int64_t nc_chunk, double *I, int to_layout,
                           cudaStream_t s);
cudaError_t launch_random_T(const Geometry &g, int64_t nz_cross_dummy, double dx, double dy,
                            double dz, const double *phase, double T_mean, double T_amp,
                            double *T, cudaStream_t s);
cudaError_t launch_gather_cells(const Geometry &g, const int *dmap, int nd, const int64_t *cells, int64_t n,
                                const double *I, double *out, cudaStream_t s);
cudaError_t launch_relax(const Geometry &g, double *I, const double *I0c, const double *beta, double dt,
                         cudaStream_t s);
cudaError_t launch_pack_cells(const Geometry &g, const int64_t *cells, int64_t n, const double *I, double *out,
                              cudaStream_t s);
cudaError_t launch_random_I(const Geometry &g, const int *canon_d, int nd, uint64_t seed,
                            double I_amp, const double *I0c, double *I, cudaStream_t s);
cudaError_t launch_octant_tree_g(const Geometry &g, const double *Dpart, int64_t nc, double *D,
                                 cudaStream_t s);
cudaError_t launch_dpart_from_I(const Geometry &g, const double *I, const double *I0c, double *Dpart,
                               cudaStream_t s);
cudaError_t launch_energy(const Geometry &g, const double *I, const double *v, double *Ec,
                          cudaStream_t s);
cudaError_t launch_usweep(const USweepArgs &a, cudaStream_t s);
cudaError_t launch_udiffuse(const Geometry &g, const UMeshDev &u, const double *I, int region, double *gtab,
                            cudaStream_t s);
cudaError_t launch_random_T_u(int64_t nc, int dim, const double *cen, const double *lo, const double *L,
                              const double *phase, double T_mean, double T_amp, double *T, cudaStream_t s);
cudaError_t launch_band_partial(const Geometry &g, const Material &mF, const double *Dpart, const double *T,
                                int64_t nc, double *S, cudaStream_t s);

}  // namespace bte
