// kernels.cu -- sm_100a kernels of the explicit phonon-BTE step (arXiv 2305.19400).
//
//   k_sweep     a1 (specular/isothermal ghosts inline) + a2: fused upwind flux +
//               relaxation update (Eq. 5 with forward Euler, P:L378-387,
//               P:L159-184) and the per-(cell, octant, channel) partial
//               sum_j w_j (I0c - I^{n+1}) of a3.  HBM-bound: 16 B/DOF.
//   k_diffuse   a1 for diffuse-adiabatic walls (reading #11).
//   k_newton    a3 (octant tree) + a4: per-cell Newton for T^{n+1} against the
//               Bose-Einstein band intensity, refresh of I0c and beta
//               (P:L277-298).  FP64-ALU-bound (expm1).
//   helpers     layout permutation, equilibrium fill, random start, tables.
//
// No tensor cores: nothing on this path is a dense contraction.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "bte_internal.cuh"

namespace bte {

// ---------------------------------------------------------------- material

__device__ __forceinline__ double beta_of_T(const double *__restrict__ bc, int b, double T) {
  const double *q = bc + 5 * b;
  const double T2 = T * T;
  double r = q[0] + q[1] * (T2 * T) + q[2] * (T2 * T2);
  if (q[3] != 0.0) r += q[3] / sinh(q[4] / T);
  return r;
}

// d beta_b / dT: 3 p3 T^2 + 4 p4 T^3 + pu theta cosh(theta/T) / (T^2 sinh^2(theta/T))
__device__ __forceinline__ double dbeta_of_T(const double *__restrict__ bc, int b, double T) {
  const double *q = bc + 5 * b;
  const double T2 = T * T;
  double r = 3.0 * q[1] * T2 + 4.0 * q[2] * (T2 * T);
  if (q[3] != 0.0) {
    const double x = q[4] / T, sh = sinh(x);
    r += q[3] * q[4] * cosh(x) / (T2 * (sh * sh));
  }
  return r;
}

// I0_b(T) and dI0_b/dT (reading #1).  BE: sum_j A_bj / expm1(X_bj / T),
// derivative term A/em1 * (X/T)/T * (1 + 1/em1) = integrand * x/T * e^x/(e^x-1).
__device__ __forceinline__ double I0_of_T(const Material &m, int b, double T, double *dI0) {
  if (m.mode == 0) {
    if (dI0) *dI0 = m.slope[b];
    return m.I_ref[b] + m.slope[b] * (T - m.T_ref);
  }
  const double *A = m.A + b * kNGL;
  const double *X = m.X + b * kNGL;
  const double rT = 1.0 / T;
  double s = 0.0, ds = 0.0;
#pragma unroll 4
  for (int j = 0; j < kNGL; ++j) {
    const double x = X[j] * rT;
    const double em1 = expm1(x);
    const double r = 1.0 / em1;
    const double f = A[j] * r;
    s += f;
    ds += f * x * (1.0 + r);
  }
  if (dI0) *dI0 = ds * rT;
  return s;
}

// ---------------------------------------------------------------- sweep

__device__ __forceinline__ double ldg(const double *p) { return __ldg(p); }

// Ghost intensity on a wall for element (slot, j, b) of the cell at `cell_base`
// ((plane + plane_off)*plane_stride + cross*E) -- Eq. 6.
__device__ __forceinline__ double ghost_value(const Geometry &g, const double *__restrict__ Iin,
                                              int region, int64_t face, int64_t cell_base, int slot,
                                              int j, int b) {
  const int kind = g.kind[region];
  if (kind == BC_ISO || kind == BC_DIFF) return ldg(g.gtab[region] + face * g.nb + b);
  double spec;
  if (g.rot) {  // slot rotation: the reflected octant may be overwritten; snapshot
    spec = ldg(g.gspec[region] + ((face * g.nslot + slot) * g.nj + j) * g.nb + b);
  } else {
    const int axis = region >> 1;
    const int64_t off = g.refl_off[(int64_t)axis * g.nslot * g.nj + slot * g.nj + j];
    spec = ldg(Iin + off + cell_base + b);
  }
  if (kind == BC_SPEC) return spec;
  // BC_PART (reading R-i): p*I_r + (1-p)*g_diffuse, products rounded separately
  return __dadd_rn(__dmul_rn(g.spec_p[region], spec), __dmul_rn(g.spec_q[region], ldg(g.gtab[region] + face * g.nb + b)));
}

// Element update shared by both sweeps.  Flux in axis order x, y, z (per-axis
// difference form, reading #19), v_b factored out of the face sum as in Eq. 5:
//   I^{n+1} = I + dt*beta*(I0c - I) - v_b * sum_a (dt|s_a|/D_a) (I - I_up,a)
template <int DIM>
__device__ __forceinline__ double bte_update(double Ic, double xu, double yu, double mu, const double *cf,
                                             double v, double I0, double dtb) {
  double fl = cf[0] * (Ic - xu);
  if (DIM == 3) fl = fma(cf[1], Ic - yu, fl);
  fl = fma(cf[DIM - 1], Ic - mu, fl);
  return fma(dtb, I0 - Ic, Ic) - v * fl;
}

// Column of this CTA.  raster = W > 0 (3-D): the columns go in strips of W
// along x, y fastest inside a strip, so the y-upwind neighbour is W launches
// back instead of nx -- its block is still in L2 when this CTA re-reads it,
// which lets the segments grow (fewer march-axis restarts).  The x-upwind
// column of a strip's first column is one strip back (a re-read from DRAM
// on 1/W of the columns).
__device__ __forceinline__ int sweep_column(const SweepArgs &A, int id) {
  const Geometry &g = A.g;
  if (g.dim != 3 || A.raster <= 0 || A.ncols > 0) return A.col0 + id;
  const int W = A.raster, ny = g.ny;
  const int strip = id / (W * ny);
  const int r = id - strip * W * ny;
  const int w = min(W, g.nx - strip * W);
  const int y = r / w;
  return strip * W + (r - y * w) + g.nx * y;
}

// One CTA = one (cross cell, octant slot, segment of the march axis).  The CTA
// walks its column in the upwind-to-downwind order of that octant, so the
// march-axis upwind value is the previous iteration's I^n kept in registers.
// Thread (grp, b) owns channel b and the directions j in [grp*jpt, grp*jpt+jpt)
// of the octant: consecutive threads touch consecutive channels of one
// direction (coalesced 8*nb-byte rows), I0c/beta are loaded once per cell per
// thread, and the octant partial sum over j accumulates in a register before
// a JG-way fixed-order smem combine.
template <int DIM, int JMAX>
__global__ void __launch_bounds__(JMAX == 1 ? 448 : 1024, JMAX == 1 ? 4 : 1) k_sweep(const SweepArgs A) {
  extern __shared__ double sm[];  // coef[nj][4] | red[2][JG][nb]
  const Geometry &g = A.g;
  const int nb = g.nb, nj = g.nj, Es = g.Es;
  const int tid = threadIdx.x;
  const int grp = tid / nb;
  const int b = tid - grp * nb;
  const int JG = blockDim.x / nb;
  const int j0 = grp * A.jpt;
  const int nloc = max(0, min(A.jpt, nj - j0));
  double *coef = sm;
  double *red = sm + 4 * nj;

  const int slot = A.slot0 + blockIdx.y;
  const int oct = g.slot_oct[slot];
  const int col = sweep_column(A, blockIdx.x);
  const int x = (DIM == 3) ? col % g.nx : col;
  const int y = (DIM == 3) ? col / g.nx : 0;
  const bool xneg = oct & 4;
  const bool yneg = oct & 2;
  const bool mneg = (DIM == 3) ? (oct & 1) : (oct & 2);

  const bool xghost = xneg ? (x == g.nx - 1) : (x == 0);
  const int xregion = xneg ? 1 : 0;
  const int64_t xoff = xneg ? (int64_t)Es : -(int64_t)Es;
  bool yghost = false;
  int yregion = 2;
  int64_t yoff = 0;
  if (DIM == 3) {
    yghost = yneg ? (y == g.ny - 1) : (y == 0);
    yregion = yneg ? 3 : 2;
    yoff = (yneg ? 1 : -1) * (int64_t)g.nx * Es;
  }
  const int mregion = (DIM == 3) ? (mneg ? 5 : 4) : (mneg ? 3 : 2);

  for (int i = tid; i < 4 * nj; i += blockDim.x) coef[i] = g.coef[(int64_t)slot * nj * 4 + i];

  const int pb = A.p_lo + blockIdx.z * A.seg_len;
  const int pe = min(A.p_hi, pb + A.seg_len);
  const int np = pe - pb;
  const int step = mneg ? -1 : 1;
  int p = mneg ? pe - 1 : pb;

  const double *__restrict__ Iin = A.Iin;
  const double *__restrict__ Is = A.Iin + g.slot_off[slot];
  double *__restrict__ Os = A.Iout + A.out_off[slot];
  const int64_t colE = (int64_t)col * Es;
  const double dt = A.dt;
  const double v = A.v[b];
  const bool active = grp < JG && tid < JG * nb;

  double prev[JMAX];
  // march-axis upwind value of the first cell of the segment
  {
    const int pm = p - step;
    const bool stored = (pm >= 0 && pm < g.nplanes) || (pm < 0 ? !g.has_lo_wall : !g.has_hi_wall);
    const int64_t base = (int64_t)(p + g.plane_off) * g.plane_stride + colE;
    const int64_t face = (DIM == 3) ? (int64_t)x + (int64_t)g.nx * y : x;
#pragma unroll
    for (int k = 0; k < JMAX; ++k) {
      prev[k] = 0.0;
      if (active && k < nloc) {
        const int e = (j0 + k) * nb + b;
        if (stored)
          prev[k] = ldg(Is + (int64_t)(pm + g.plane_off) * g.plane_stride + colE + e);
        else
          prev[k] = ghost_value(g, Iin, mregion, face, base, slot, j0 + k, b);
      }
    }
  }
  __syncthreads();

  if (!xghost && (DIM == 2 || !yghost)) {
    // interior column (every column but the wall ones): running pointers along
    // the march, no per-cell 64-bit index products, no ghost branches
    const int e0 = j0 * nb + b;
    const int64_t pstep = (int64_t)step * g.plane_stride;
    const int64_t cstep = (int64_t)step * g.ncross * nb;
    const int64_t dstep = cstep * g.nslot;
    const int64_t c0 = (int64_t)col + (int64_t)p * g.ncross;
    const double *ip = Is + (int64_t)(p + g.plane_off) * g.plane_stride + colE + e0;
    double *op = Os + (int64_t)(p + g.plane_off) * g.plane_stride + colE + e0;
    const double *i0p = A.I0c + c0 * nb + b;
    const double *bp = A.beta + c0 * nb + b;
    double *dp = A.Dpart + (c0 * g.nslot + slot) * nb + (tid < nb ? tid : 0);
    const double *cq = coef + 4 * j0;
    const int pf = A.pf;
    double *rbw = red + tid, *rbw_alt = red + JG * nb + tid;  // this thread's partial slot
    const double *rbr = red + (tid < nb ? tid : 0), *rbr_alt = rbr + JG * nb;  // reducer's column
    for (int i = 0; i < np; ++i) {
      double acc = 0.0;
      if (active && pf > 0 && i + pf < np) {
        // L2 prefetch of this thread's elements pf cells ahead (no registers held)
#pragma unroll
        for (int k = 0; k < JMAX; ++k)
          if (k < nloc) asm volatile("prefetch.global.L2 [%0];" ::"l"(ip + pf * pstep + k * nb));
        if (grp == 0) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(i0p + pf * cstep));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(bp + pf * cstep));
        }
      }
      if (active) {
        const double I0 = ldg(i0p);
        const double dtb = dt * ldg(bp);
#pragma unroll
        for (int k = 0; k < JMAX; ++k) {
          if (k < nloc) {
            const double Ic = ldg(ip + k * nb);
            const double xu = ldg(ip + xoff + k * nb);
            const double yu = DIM == 3 ? ldg(ip + yoff + k * nb) : 0.0;
            const double In = bte_update<DIM>(Ic, xu, yu, prev[k], cq + 4 * k, v, I0, dtb);
            op[k * nb] = In;
            acc = fma(cq[4 * k + 3], I0 - In, acc);
            prev[k] = Ic;
          }
        }
      }
      // reduction buffer of this cell: two halves, pointer swapped per cell
      // (no per-cell address rebuild)
      if (active) *rbw = acc;
      __syncthreads();
      if (tid < nb) {
        double s = 0.0;
        for (int q = 0; q < JG; ++q) s += rbr[q * nb];
        *dp = s;
      }
      {
        double *t = rbw;
        rbw = rbw_alt;
        rbw_alt = t;
        const double *u = rbr;
        rbr = rbr_alt;
        rbr_alt = u;
      }
      ip += pstep;
      op += pstep;
      i0p += cstep;
      bp += cstep;
      dp += dstep;
    }
    return;
  }

  int buf = 0;
  for (int i = 0; i < np; ++i, p += step) {
    const int64_t cell = (int64_t)col + (int64_t)p * g.ncross;  // local canonical cell
    const int64_t base = (int64_t)(p + g.plane_off) * g.plane_stride + colE;
    const int64_t mg = g.m0 + p;
    double acc = 0.0;
    if (active) {
      const double I0 = ldg(A.I0c + cell * nb + b);
      const double dtb = dt * ldg(A.beta + cell * nb + b);
#pragma unroll
      for (int k = 0; k < JMAX; ++k) {
        if (k < nloc) {
          const int j = j0 + k;
          const int e = j * nb + b;
          const double Ic = ldg(Is + base + e);
          double xu, yu = 0.0;
          if (!xghost) {
            xu = ldg(Is + base + xoff + e);
          } else {
            const int64_t face = (DIM == 3) ? (int64_t)y + (int64_t)g.ny * mg : mg;
            xu = ghost_value(g, Iin, xregion, face, base, slot, j, b);
          }
          if (DIM == 3) {
            if (!yghost) {
              yu = ldg(Is + base + yoff + e);
            } else {
              const int64_t face = (int64_t)x + (int64_t)g.nx * mg;
              yu = ghost_value(g, Iin, yregion, face, base, slot, j, b);
            }
          }
          const double *cf = coef + 4 * j;
          const double In = bte_update<DIM>(Ic, xu, yu, prev[k], cf, v, I0, dtb);
          Os[base + e] = In;
          acc = fma(cf[3], I0 - In, acc);
          prev[k] = Ic;
        }
      }
    }
    double *rb = red + buf * JG * nb;
    if (active) rb[tid] = acc;
    __syncthreads();
    if (tid < nb) {
      double s = 0.0;
      for (int q = 0; q < JG; ++q) s += rb[q * nb + tid];
      A.Dpart[(cell * g.nslot + slot) * nb + tid] = s;
    }
    buf ^= 1;
  }
}

// per-warp Newton scratch (doubles): c_b during the solve, node/band factors in the refresh
// node-major GL tables in shared memory: entry (b, j) at j*R + b, row stride
// R = nb rounded up to 2 (mod 4) so that the 4 node groups of a warp load
// fall on disjoint bank sets
__host__ __device__ __forceinline__ int gl_stride(int nb) { return nb + ((6 - nb % 4) % 4); }

__host__ __device__ __forceinline__ int newton_scratch(const Material &m, int nb) {
  return 4 * nb + 2 * kNGL + m.imax + 1;  // c | E | M | R | I0 | dI0 | d2I0
}

template <bool BAND = false>
__device__ void newton_cell(const NewtonArgs &a, int64_t c, const double *sA, const double *sX, const int *sI,
                            double *cs, int lane);

// ---------------------------------------------------------------- TMA-pipelined sweep

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (UBLKCP), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same decomposition as k_sweep, but the (cell, octant) blocks of the cell and
// of its cross-axis upwind neighbours (16 KB each at 50 x 40), plus the cell's
// I0c/beta rows, stream into an S-stage shared-memory ring with cp.async.bulk
// + mbarrier, issued S cells ahead by one thread.  Keeps S x (2 or 3) x 16 KB
// of HBM/L2 reads in flight per CTA.  NBT > 0 fixes the channel count at
// compile time (immediate smem/global offsets); NBT = 0 is the generic path.
// SS > 0 fixes the ring depth at compile time (stage index and phase kept as
// running counters, no division per cell); the 40-channel specialisation is
// bounded to 448 threads x 2 CTAs/SM, so ptxas may use 72 registers and keeps
// the loop-invariant addresses in registers instead of re-deriving them from
// the kernel parameters every cell.
template <int DIM, int JMAX, int NBT, int SS>
__global__ void __launch_bounds__(NBT == 40 ? 448 : 1024, NBT == 40 ? 2 : 1) k_sweep_tma(const SweepArgs A) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const Geometry &g = A.g;
  const int nb = NBT > 0 ? NBT : g.nb;
  const int nj = g.nj, Es = g.Es;
  const int S = SS > 0 ? SS : A.stages;
  const int tid = threadIdx.x;
  const int grp = tid / nb;
  const int b = tid - grp * nb;
  const int JG = A.jg;
  const int j0 = grp * A.jpt;
  const int nloc = max(0, min(A.jpt, nj - j0));
  const bool active = grp < JG;
  // side jobs on the spare threads past the JG*nb compute threads when the
  // launch provides them (reducers [JG*nb, JG*nb + nb), issuer JG*nb + nb),
  // else on threads 0..nb-1 / 0
  const int spare0 = JG * nb;
  const bool spare = (int)blockDim.x >= spare0 + nb + 1;
  const int rtid = spare ? tid - spare0 : tid;  // reducer index (channel) when in [0, nb)
  const bool reducer = rtid >= 0 && rtid < nb;
  const int tis = spare ? spare0 + nb : 0;

  const int slot = A.slot0 + blockIdx.y;
  const int oct = g.slot_oct[slot];
  const int col = sweep_column(A, blockIdx.x);
  const int x = (DIM == 3) ? col % g.nx : col;
  const int y = (DIM == 3) ? col / g.nx : 0;
  const bool xneg = oct & 4;
  const bool yneg = oct & 2;
  const bool mneg = (DIM == 3) ? (oct & 1) : (oct & 2);
  const bool xghost = xneg ? (x == g.nx - 1) : (x == 0);
  const int xregion = xneg ? 1 : 0;
  const int64_t xoff = xneg ? (int64_t)Es : -(int64_t)Es;
  bool yghost = false;
  int yregion = 2;
  int64_t yoff = 0;
  if (DIM == 3) {
    yghost = yneg ? (y == g.ny - 1) : (y == 0);
    yregion = yneg ? 3 : 2;
    yoff = (yneg ? 1 : -1) * (int64_t)g.nx * Es;
  }
  const bool interior = !xghost && !yghost;
  const int mregion = (DIM == 3) ? (mneg ? 5 : 4) : (mneg ? 3 : 2);

  // shared memory carve-up
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);          // [S] (S <= 16)
  double *coef = reinterpret_cast<double *>(smraw + 128);        // [nj][4]
  double *red = coef + 4 * nj;                                   // [2][JG*nb]
  double *stage0 = red + 2 * JG * nb;                            // [S][stage_doubles]
  const int64_t sd = A.stage_doubles;                            // own | xup | (yup) | I0 | beta
  constexpr bool ystage = DIM == 3;  // y-upwind block in the stage
  const int nblk = 1 + (xghost ? 0 : 1) + ((ystage && !yghost) ? 1 : 0);
  const int o_x = Es, o_y = 2 * Es, o_i0 = (ystage ? 3 : 2) * Es, o_be = o_i0 + nb;
  const bool rows_tma = (nb % 2) == 0;  // 16-B bulk-copy granularity; else direct loads

  const int pb = A.p_lo + blockIdx.z * A.seg_len;
  const int pe = min(A.p_hi, pb + A.seg_len);
  const int np = pe - pb;
  const int step = mneg ? -1 : 1;
  const int pfirst = mneg ? pe - 1 : pb;

  const double *__restrict__ Iin = A.Iin;
  const double *__restrict__ Is = A.Iin + g.slot_off[slot];
  double *__restrict__ Os = A.Iout + A.out_off[slot];
  const int64_t colE = (int64_t)col * Es;
  const double dt = A.dt;

  auto issue = [&](int i, int st) {
    const int pp = pfirst + i * step;
    const int64_t base = (int64_t)(pp + g.plane_off) * g.plane_stride + colE;
    const int64_t cell = (int64_t)col + (int64_t)pp * g.ncross;
    double *sp = stage0 + st * sd;
    const uint32_t blk = (uint32_t)Es * 8u;
    const uint32_t row = (uint32_t)nb * 8u;
    mbar_expect_tx(&full[st], blk * nblk + (rows_tma ? 2u * row : 0u));
    bulk_g2s(sp, Is + base, blk, &full[st]);
    if (!xghost) bulk_g2s(sp + o_x, Is + base + xoff, blk, &full[st]);
    if (ystage && !yghost) bulk_g2s(sp + o_y, Is + base + yoff, blk, &full[st]);
    if (rows_tma) {
      bulk_g2s(sp + o_i0, A.I0c + cell * nb, row, &full[st]);
      bulk_g2s(sp + o_be, A.beta + cell * nb, row, &full[st]);
    }
  };

  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 4 * nj; i += blockDim.x) coef[i] = g.coef[(int64_t)slot * nj * 4 + i];
  __syncthreads();
  if (tid == tis)
    for (int i = 0; i < min(S, np); ++i) issue(i, i);

  const double v = A.v[active ? b : 0];
  const int e0 = j0 * nb + b;  // this thread's first element; element k is e0 + k*nb
  const double *cq = coef + 4 * j0;
  double prev[JMAX];
  {
    const int p = pfirst;
    const int pm = p - step;
    const bool stored = (pm >= 0 && pm < g.nplanes) || (pm < 0 ? !g.has_lo_wall : !g.has_hi_wall);
    const int64_t base = (int64_t)(p + g.plane_off) * g.plane_stride + colE;
    const int64_t face = (DIM == 3) ? (int64_t)x + (int64_t)g.nx * y : x;
#pragma unroll
    for (int k = 0; k < JMAX; ++k) {
      prev[k] = 0.0;
      if (active && k < nloc) {
        if (stored)
          prev[k] = ldg(Is + (int64_t)(pm + g.plane_off) * g.plane_stride + colE + e0 + k * nb);
        else
          prev[k] = ghost_value(g, Iin, mregion, face, base, slot, j0 + k, b);
      }
    }
  }

  // running addresses along the march: this thread's output row and the
  // reducer's octant-partial entry
  const int64_t pstep = (int64_t)step * g.plane_stride;
  double *op = Os + (int64_t)(pfirst + g.plane_off) * g.plane_stride + colE + e0;
  const int64_t dstep = (int64_t)step * g.ncross * g.nslot * nb;
  double *dp = A.Dpart + (((int64_t)col + (int64_t)pfirst * g.ncross) * g.nslot + slot) * nb + (reducer ? rtid : 0);
  const double *rb0 = red, *rb1 = red + JG * nb;
  int st = 0;
  uint32_t ph = 0;
  int p = pfirst;
  for (int i = 0; i < np; ++i, p += step) {
    const double *sp = stage0 + st * sd;
    mbar_wait(&full[st], ph);
    double acc = 0.0;
    if (active) {
      const double I0 = rows_tma ? sp[o_i0 + b] : ldg(A.I0c + ((int64_t)col + (int64_t)p * g.ncross) * nb + b);
      const double dtb = dt * (rows_tma ? sp[o_be + b] : ldg(A.beta + ((int64_t)col + (int64_t)p * g.ncross) * nb + b));
      const double *so = sp + e0;
      if (interior && nloc == JMAX) {
        const double *sx = so + o_x;
        const double *sy = so + o_y;
#pragma unroll
        for (int k = 0; k < JMAX; ++k) {
          const double Ic = so[k * nb];
          const double In = bte_update<DIM>(Ic, sx[k * nb], DIM == 3 ? sy[k * nb] : 0.0, prev[k],
                                            cq + 4 * k, v, I0, dtb);
          __stcs(op + k * nb, In);  // evict-first: I^{n+1} is not re-read this step
          acc = fma(cq[4 * k + 3], I0 - In, acc);
          prev[k] = Ic;
        }
      } else {
        const int64_t base = (int64_t)(p + g.plane_off) * g.plane_stride + colE;
        const int64_t mg = g.m0 + p;
#pragma unroll
        for (int k = 0; k < JMAX; ++k) {
          if (k < nloc) {
            const int j = j0 + k;
            const double Ic = so[k * nb];
            double xu, yu = 0.0;
            if (!xghost) {
              xu = so[o_x + k * nb];
            } else {
              const int64_t face = (DIM == 3) ? (int64_t)y + (int64_t)g.ny * mg : mg;
              xu = ghost_value(g, Iin, xregion, face, base, slot, j, b);
            }
            if (DIM == 3) {
              if (!yghost) {
                yu = so[o_y + k * nb];
              } else {
                const int64_t face = (int64_t)x + (int64_t)g.nx * mg;
                yu = ghost_value(g, Iin, yregion, face, base, slot, j, b);
              }
            }
            const double In = bte_update<DIM>(Ic, xu, yu, prev[k], cq + 4 * k, v, I0, dtb);
            __stcs(op + k * nb, In);
            acc = fma(cq[4 * k + 3], I0 - In, acc);
            prev[k] = Ic;
          }
        }
      }
    }
    double *rb = const_cast<double *>((i & 1) ? rb1 : rb0);
    if (active) rb[tid] = acc;
    __syncthreads();  // stage st fully consumed, rb complete
    if (tid == tis && i + S < np) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S, st);
    }
    if (reducer) {
      double s = 0.0;
      for (int q = 0; q < JG; ++q) s += rb[q * nb + rtid];
      *dp = s;
    }
    op += pstep;
    dp += dstep;
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  }
}

// thread shape: JG groups of nb threads, jpt directions per thread
static void sweep_shape(int nb, int nj, int target, int *jpt, int *JG) {
  int jg = (target + nb / 2) / nb;
  jg = std::max(1, std::min(jg, nj));
  while (jg * nb > 1024) --jg;
  if (jg < 1) jg = 1;
  int j = (nj + jg - 1) / jg;
  jg = (nj + j - 1) / j;
  *jpt = j;
  *JG = jg;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size:
// the launchers run on every step, the attribute only has to grow
static cudaError_t smem_attr(const void *fn, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void *, size_t> done;
  std::lock_guard<std::mutex> lk(mu);
  size_t &cur = done[fn];
  if (smem <= cur || smem <= 48 * 1024) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

template <int DIM>
static cudaError_t launch_sweep_dim(const SweepArgs &a0, cudaStream_t s) {
  SweepArgs a = a0;
  const Geometry &g = a.g;
  int jpt, JG;
  sweep_shape(g.nb, g.nj, a.target_threads > 0 ? a.target_threads : 448, &jpt, &JG);
  a.jpt = jpt;
  const int threads = JG * g.nb;
  if (threads > 1024 || g.nb > 1024) return cudaErrorInvalidConfiguration;
  if (a.p_hi <= a.p_lo) {  // default: every owned plane
    a.p_lo = 0;
    a.p_hi = g.nplanes;
  }
  const int nseg = (a.p_hi - a.p_lo + a.seg_len - 1) / a.seg_len;
  dim3 grid(a.ncols > 0 ? a.ncols : g.ncross, a.nslots > 0 ? a.nslots : g.nslot, nseg);
  const int jcase = jpt <= 1 ? 1 : jpt <= 2 ? 2 : jpt <= 4 ? 4 : jpt <= 5 ? 5 : jpt <= 8 ? 8 : jpt <= 10 ? 10 : jpt <= 16 ? 16 : 0;
  const bool tma = a.use_tma && (g.Es % 2 == 0);
  // blocks under 384 doubles: the direct-load kernel keeps more cells in
  // flight than a per-cell TMA ring (measured: demo 0.089 vs 0.110 ms)
  if (tma && g.E >= 384) {
    // stage: own | xup | (yup) | I0 row | beta row, rounded to 128 B (y-direct: no yup)
    const int64_t stage_d = ((int64_t)(DIM == 3 ? 3 : 2) * g.Es + 2 * g.nb + 15) / 16 * 16;
    const size_t fixed = 128 + (4 * (size_t)g.nj + 2 * (size_t)threads) * sizeof(double);
    const size_t budget = (size_t)(a.smem_budget_kb > 0 ? a.smem_budget_kb : 113) * 1024;  // two CTAs/SM
    int S = (int)((budget > fixed ? budget - fixed : 0) / (stage_d * sizeof(double)));
    S = std::max(2, std::min(4, S));
    if (a.stages_override > 0) S = std::min(16, a.stages_override);
    a.stages = S;
    a.stage_doubles = stage_d;
    a.jg = JG;
    const size_t smem = fixed + (size_t)S * stage_d * sizeof(double);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    // spare threads for the side jobs (reducers + issuer) unless disabled at create
    const int tthreads = ((a.no_spare ? threads : threads + g.nb + 1) + 31) / 32 * 32;
    cudaError_t e;
#define BTE_LAUNCH_S(N, NB, SV)                                                      \
  {                                                                                  \
    if ((e = smem_attr((const void *)k_sweep_tma<DIM, N, NB, SV>, smem))) return e;  \
    k_sweep_tma<DIM, N, NB, SV><<<grid, tthreads, smem, s>>>(a);                     \
    break;                                                                           \
  }
#define BTE_LAUNCH(N, NB) BTE_LAUNCH_S(N, NB, 0)

    if (g.nb == 40 && jcase == 5 && tthreads <= 448 && S >= 2 && S <= 4) {
      switch (S) {
        case 2: BTE_LAUNCH_S(5, 40, 2)
        case 3: BTE_LAUNCH_S(5, 40, 3)
        default: BTE_LAUNCH_S(5, 40, 4)
      }
    } else if (g.nb == 55 && jcase == 8 && S >= 2 && S <= 4) {
      switch (S) {
        case 2: BTE_LAUNCH_S(8, 55, 2)
        case 3: BTE_LAUNCH_S(8, 55, 3)
        default: BTE_LAUNCH_S(8, 55, 4)
      }
    } else {
      switch (jcase) {
        case 1: BTE_LAUNCH(1, 0)
        case 2: BTE_LAUNCH(2, 0)
        case 4: BTE_LAUNCH(4, 0)
        case 5: BTE_LAUNCH(5, 0)
        case 8: BTE_LAUNCH(8, 0)
        case 10: BTE_LAUNCH(10, 0)
        case 16: BTE_LAUNCH(16, 0)
        default:
          return cudaErrorInvalidConfiguration;
      }
    }
#undef BTE_LAUNCH
#undef BTE_LAUNCH_S

    return cudaGetLastError();
  }
  const size_t smem = (4 * (size_t)g.nj + 2 * (size_t)threads) * sizeof(double);
  cudaError_t e;
  switch (jcase) {
#define BTE_CASE(N)                                                       \
  case N:                                                                 \
    if ((e = smem_attr((const void *)k_sweep<DIM, N>, smem))) return e;   \
    k_sweep<DIM, N><<<grid, threads, smem, s>>>(a);                       \
    break;
    BTE_CASE(1)
    BTE_CASE(2)
    BTE_CASE(4)
    BTE_CASE(5)
    BTE_CASE(8)
    BTE_CASE(10)
    BTE_CASE(16)
#undef BTE_CASE
    default:
      return cudaErrorInvalidConfiguration;
  }
  return cudaGetLastError();
}

const char *sweep_kernel_name(const SweepArgs &a) {
  const Geometry &g = a.g;
  const bool tma = a.use_tma && (g.Es % 2 == 0) && g.E >= 384;
  if (g.dim == 3) return tma ? "k_sweep_tma<3>" : "k_sweep<3>";
  return tma ? "k_sweep_tma<2>" : "k_sweep<2>";
}

cudaError_t launch_sweep(const SweepArgs &a, cudaStream_t s) {
  return a.g.dim == 3 ? launch_sweep_dim<3>(a, s) : launch_sweep_dim<2>(a, s);
}

// ---------------------------------------------------------------- implicit transport sweep (R-n)

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One source iteration's transport sweep of the implicit step (reading R-n):
//   I^{k+1} = I^n + [dt beta (I0c - I^n) + sum_a kk_a (I^{k+1}_up,a - I^n)] / (1 + dt beta + sum_a kk_a),
// kk_a = v_b dt |s_a| / D_a, axis terms in x, y, z order.  I'_up is THIS sweep's
// value of the upwind cell (a wavefront: exact inversion of the upwind operator
// for the scattering source I0c = I0(T^k)), or the wall ghost of I^k (snapshot
// / tables, the g.rot path of ghost_value).
//
// One CTA per (octant slot, column) task.  Tasks are taken by ticket in a
// topological order of the upwind dependence (host table: the column's
// distance from its octant's upwind corner), so every column a CTA waits for
// belongs to a CTA that took its ticket earlier and is running or done -- no
// deadlock whatever the block scheduler does.  The CTA marches its column
// from the upwind wall along the march axis (upwind value in registers, the
// CTA's own previous result) and publishes each plane it has written
// (release counter per (slot, column), one 128-B line each).  Its stage ring
// holds per plane the own I^n block + I0c / beta rows (barrier A, issued S
// planes ahead: independent of the wavefront) and the x- / y-upwind columns'
// I^{k+1} blocks (barrier B): a dedicated issuer warp copies a neighbour plane
// as soon as both counters have passed it -- often planes ahead of the
// compute, since the upwind columns started earlier -- so the compute warps
// never poll and the L2 latency of the neighbour data overlaps other work.
template <int DIM, int JMAX, int MT, int MB>
__global__ void __launch_bounds__(MT, MB) k_sweep_imp(const SweepArgs A, const int2 *__restrict__ tasks,
                                                    int *__restrict__ prog, unsigned *__restrict__ ticket) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ int s_task;
  const Geometry &g = A.g;
  const int nb = g.nb;
  const int nj = g.nj, Es = g.Es;
  const int S = A.stages;
  const int tid = threadIdx.x;
  const int grp = tid / nb;
  const int b = tid - grp * nb;
  const int JG = A.jg;
  const int j0 = grp * A.jpt;
  const int nloc = max(0, min(A.jpt, nj - j0));
  const bool active = grp < JG;
  const int rtid = tid - JG * nb;            // reducers: [0, nb)
  const int tis = (int)blockDim.x - 32;      // issuer: lane 0 of the last warp (the launcher adds it)

  if (tid == 0) s_task = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int2 task = tasks[s_task];
  const int slot = task.x, col = task.y;
  const int oct = g.slot_oct[slot];
  const int x = (DIM == 3) ? col % g.nx : col;
  const int y = (DIM == 3) ? col / g.nx : 0;
  const bool xneg = oct & 4;
  const bool yneg = oct & 2;
  const bool mneg = (DIM == 3) ? (oct & 1) : (oct & 2);
  const bool xghost = xneg ? (x == g.nx - 1) : (x == 0);
  const int xregion = xneg ? 1 : 0;
  const int64_t xoff = xneg ? (int64_t)Es : -(int64_t)Es;
  const int xcol = xneg ? col + 1 : col - 1;
  bool yghost = true;
  int yregion = 2;
  int64_t yoff = 0;
  int ycol = 0;
  if (DIM == 3) {
    yghost = yneg ? (y == g.ny - 1) : (y == 0);
    yregion = yneg ? 3 : 2;
    yoff = (yneg ? 1 : -1) * (int64_t)g.nx * Es;
    ycol = yneg ? col + g.nx : col - g.nx;
  }
  const bool hasB = !xghost || (DIM == 3 && !yghost);
  const int mregion = (DIM == 3) ? (mneg ? 5 : 4) : (mneg ? 3 : 2);
  constexpr int kProgStride = 32;  // counters one 128-B line apart
  int *pr = prog + (int64_t)slot * g.ncross * kProgStride;

  uint64_t *fullA = reinterpret_cast<uint64_t *>(smraw);  // [S] own + rows
  uint64_t *fullB = fullA + 8;                            // [S] upwind neighbours (S <= 8)
  double *coef = reinterpret_cast<double *>(smraw + 128);
  double *red = coef + 4 * nj;
  double *stage0 = red + 2 * JG * nb;
  const int64_t sd = A.stage_doubles;  // own I^n | x-up | y-up | I0 | beta
  const int o_x = Es, o_y = 2 * Es, o_i0 = (DIM == 3 ? 3 : 2) * Es, o_be = o_i0 + nb;
  const bool rows_tma = (nb % 2) == 0;
  const int np = g.nplanes;
  const int step = mneg ? -1 : 1;
  const int pfirst = mneg ? np - 1 : 0;

  const double *__restrict__ In = A.Iin + g.slot_off[slot];
  double *__restrict__ Os = A.Iout + A.out_off[slot];
  const int64_t colE = (int64_t)col * Es;
  const double dt = A.dt;
  const uint32_t blk = (uint32_t)Es * 8u;

  auto issueA = [&](int i, int st) {
    const int pp = pfirst + i * step;
    const int64_t base = (int64_t)pp * g.plane_stride + colE;
    const int64_t cell = (int64_t)col + (int64_t)pp * g.ncross;
    double *sp = stage0 + st * sd;
    const uint32_t row = (uint32_t)nb * 8u;
    mbar_expect_tx(&fullA[st], blk + (rows_tma ? 2u * row : 0u));
    bulk_g2s(sp, In + base, blk, &fullA[st]);
    if (rows_tma) {
      bulk_g2s(sp + o_i0, A.I0c + cell * nb, row, &fullA[st]);
      bulk_g2s(sp + o_be, A.beta + cell * nb, row, &fullA[st]);
    }
  };
  // plane i of the upwind columns, once published (their stores are generic-
  // proxy writes of other SMs: acquire, then order the bulk reads after it)
  // the issuer caches the counters it last saw: the upwind columns usually run
  // far ahead, so one acquire load clears many planes (each costs an L2 round trip)
  int xseen = xghost ? np : 0, yseen = (DIM == 3 && !yghost) ? 0 : np;
  auto nb_ready = [&](int i) {
    if (i >= xseen) {
      xseen = ld_acquire_gpu(pr + (int64_t)xcol * kProgStride);
      if (i >= xseen) return false;
    }
    if (i >= yseen) {
      yseen = ld_acquire_gpu(pr + (int64_t)ycol * kProgStride);
      if (i >= yseen) return false;
    }
    return true;
  };
  auto issueB = [&](int i, int st) {
    const int pp = pfirst + i * step;
    const int64_t base = (int64_t)pp * g.plane_stride + colE;
    double *sp = stage0 + st * sd;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&fullB[st], blk * ((xghost ? 0u : 1u) + ((DIM == 3 && !yghost) ? 1u : 0u)));
    if (!xghost) bulk_g2s(sp + o_x, Os + base + xoff, blk, &fullB[st]);
    if (DIM == 3 && !yghost) bulk_g2s(sp + o_y, Os + base + yoff, blk, &fullB[st]);
  };

  if (tid == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&fullA[st], 1);
      mbar_init(&fullB[st], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 4 * nj; i += blockDim.x) coef[i] = g.coef[(int64_t)slot * nj * 4 + i];
  __syncthreads();
  if (tid == tis)
    for (int i = 0; i < min(S, np); ++i) issueA(i, i);

  const double v = A.v[active ? b : 0];
  const int e0 = j0 * nb + b;
  const double *cq = coef + 4 * j0;
  double prev[JMAX];  // march-axis upwind I^{k+1}: the wall ghost, then this CTA's own results
  {
    const int64_t base = (int64_t)pfirst * g.plane_stride + colE;
    const int64_t face = (DIM == 3) ? (int64_t)x + (int64_t)g.nx * y : x;
#pragma unroll
    for (int k = 0; k < JMAX; ++k) {
      prev[k] = 0.0;
      if (active && k < nloc) prev[k] = ghost_value(g, A.Iin, mregion, face, base, slot, j0 + k, b);
    }
  }

  int nbq = 0;  // issuer: next plane whose neighbour blocks are to be copied
  int st = 0;
  uint32_t ph = 0;
  int p = pfirst;
  for (int i = 0; i < np; ++i, p += step) {
    const int64_t cell = (int64_t)col + (int64_t)p * g.ncross;
    const int64_t base = (int64_t)p * g.plane_stride + colE;
    const double *sp = stage0 + st * sd;
    if (tid == tis && hasB) {
      // copy every published neighbour plane whose stage is free (planes < i + S);
      // plane i itself is needed now: wait for it
      while (nbq < np && nbq < i + S) {
        if (!nb_ready(nbq)) {
          if (nbq > i) break;
          __nanosleep(64);
          continue;
        }
        issueB(nbq, nbq % S);
        ++nbq;
      }
    }
    mbar_wait(&fullA[st], ph);
    if (hasB) mbar_wait(&fullB[st], ph);
    double acc = 0.0;
    if (active) {
      const double I0 = rows_tma ? sp[o_i0 + b] : ldg(A.I0c + cell * nb + b);
      const double dtb = dt * (rows_tma ? sp[o_be + b] : ldg(A.beta + cell * nb + b));
      const int64_t mg = g.m0 + p;
      if (!xghost && (DIM == 2 || !yghost) && nloc == JMAX) {
        // interior column: no ghost branches; the flux terms without the
        // s_a == 0 tests (a zero coefficient adds exactly 0 to num and den)
#pragma unroll
        for (int k = 0; k < JMAX; ++k) {
          const int e = e0 + k * nb;
          const double Inn = sp[e];
          const double *cf = cq + 4 * k;
          const double kx = v * cf[0], km = v * cf[DIM - 1];
          double num = dtb * (I0 - Inn), den = 1.0 + dtb;
          num = fma(kx, sp[o_x + e] - Inn, num);
          den += kx;
          if (DIM == 3) {
            const double ky = v * cf[1];
            num = fma(ky, sp[o_y + e] - Inn, num);
            den += ky;
          }
          num = fma(km, prev[k] - Inn, num);
          den += km;
          // 1/den (den >= 1): MUFU seed + two Newton-Raphson steps (~1 ulp)
          double r;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
          r = fma(r, fma(-den, r, 1.0), r);
          r = fma(r, fma(-den, r, 1.0), r);
          const double Inew = fma(num, r, Inn);
          __stcg(Os + base + e, Inew);
          acc = fma(cf[3], I0 - Inew, acc);
          prev[k] = Inew;
        }
      } else {
#pragma unroll
      for (int k = 0; k < JMAX; ++k) {
        if (k < nloc) {
          const int j = j0 + k;
          const int e = e0 + k * nb;
          const double Inn = sp[e];
          double xu, yu = 0.0;
          if (!xghost) {
            xu = sp[o_x + e];
          } else {
            const int64_t face = (DIM == 3) ? (int64_t)y + (int64_t)g.ny * mg : mg;
            xu = ghost_value(g, A.Iin, xregion, face, base, slot, j, b);
          }
          if (DIM == 3) {
            if (!yghost) {
              yu = sp[o_y + e];
            } else {
              const int64_t face = (int64_t)x + (int64_t)g.nx * mg;
              yu = ghost_value(g, A.Iin, yregion, face, base, slot, j, b);
            }
          }
          const double *cf = cq + 4 * k;
          double num = dtb * (I0 - Inn), den = 1.0 + dtb;
          if (cf[0] != 0.0) {
            const double kk = v * cf[0];
            num = fma(kk, xu - Inn, num);
            den += kk;
          }
          if (DIM == 3 && cf[1] != 0.0) {
            const double kk = v * cf[1];
            num = fma(kk, yu - Inn, num);
            den += kk;
          }
          if (cf[DIM - 1] != 0.0) {
            const double kk = v * cf[DIM - 1];
            num = fma(kk, prev[k] - Inn, num);
            den += kk;
          }
          // I^{k+1} = I^n + num/den: a correctly rounded reciprocal refined by
          // one Newton step, then the product (within 2 ulp of the quotient)
          double r = __drcp_rn(den);
          r = fma(r, fma(-den, r, 1.0), r);
          const double Inew = fma(num, r, Inn);
          __stcg(Os + base + e, Inew);
          acc = fma(cf[3], I0 - Inew, acc);
          prev[k] = Inew;
        }
      }
      }
    }
    double *rb = red + (i & 1) * JG * nb;
    if (active) rb[tid] = acc;
    __syncthreads();  // stage st consumed, rb complete, this plane's stores issued
    // publish the plane: a gpu-scope release after the CTA barrier orders every
    // thread's stores before it (cumulativity; the pattern of CUTLASS's
    // GenericBarrier), no membar.gl.  (A separate publisher warp on named
    // barriers was 3 % faster but lets the compute warps arrive for the next
    // plane before it has synchronised -- a barrier-phase race; reverted.)
    if (tid == 0) st_release_gpu(pr + (int64_t)col * kProgStride, i + 1);
    if (tid == tis && i + S < np) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issueA(i + S, st);
    }
    if (rtid >= 0 && rtid < nb) {
      double s = 0.0;
      for (int q = 0; q < JG; ++q) s += rb[q * nb + rtid];
      A.Dpart[(cell * g.nslot + slot) * nb + rtid] = s;
    }
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  }
}

template <int DIM>
static cudaError_t launch_sweep_imp_dim(const SweepArgs &a0, const int2 *tasks, int ntasks, int *prog,
                                        unsigned *ticket, cudaStream_t s) {
  SweepArgs a = a0;
  const Geometry &g = a.g;
  int jpt, JG;
  sweep_shape(g.nb, g.nj, a.target_threads > 0 ? a.target_threads : 448, &jpt, &JG);
  a.jpt = jpt;
  a.jg = JG;
  const int threads = JG * g.nb;
  if (threads > 1024 || (g.Es & 1)) return cudaErrorInvalidConfiguration;
  // stage: own | x-up | (y-up) | I0 | beta
  const int64_t stage_d = ((int64_t)(DIM == 3 ? 3 : 2) * g.Es + 2 * g.nb + 15) / 16 * 16;
  const size_t fixed = 128 + (4 * (size_t)g.nj + 2 * (size_t)threads) * sizeof(double);
  const int tthreads = ((threads + g.nb + 31) / 32) * 32 + 32;  // compute + reducers, then the issuer warp
  if (tthreads > 1024) return cudaErrorInvalidConfiguration;
  const bool small = tthreads <= 288;
  const size_t budget = (size_t)(a.smem_budget_kb > 0 ? a.smem_budget_kb : (small ? 75 : 113)) * 1024;
  int S = (int)((budget > fixed ? budget - fixed : 0) / (stage_d * sizeof(double)));
  S = std::max(2, std::min(4, S));
  if (a.stages_override > 0) S = std::min(8, a.stages_override);
  a.stages = S;
  a.stage_doubles = stage_d;
  const size_t smem = fixed + (size_t)S * stage_d * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const int jcase = jpt <= 1 ? 1 : jpt <= 2 ? 2 : jpt <= 4 ? 4 : jpt <= 5 ? 5 : jpt <= 8 ? 8 : jpt <= 10 ? 10 : jpt <= 16 ? 16 : 0;
  cudaError_t e;
  switch (jcase) {
#define BTE_IMP(N)                                                                          \
  case N:                                                                                   \
    if (tthreads <= 288) {                                                                  \
      if ((e = smem_attr((const void *)k_sweep_imp<DIM, N, 288, 3>, smem))) return e;       \
      k_sweep_imp<DIM, N, 288, 3><<<ntasks, tthreads, smem, s>>>(a, tasks, prog, ticket);   \
    } else {                                                                                \
      if ((e = smem_attr((const void *)k_sweep_imp<DIM, N, 1024, 1>, smem))) return e;      \
      k_sweep_imp<DIM, N, 1024, 1><<<ntasks, tthreads, smem, s>>>(a, tasks, prog, ticket);  \
    }                                                                                       \
    break;
    BTE_IMP(1)
    BTE_IMP(2)
    BTE_IMP(4)
    BTE_IMP(5)
    BTE_IMP(8)
    BTE_IMP(10)
    BTE_IMP(16)
#undef BTE_IMP
    default:
      return cudaErrorInvalidConfiguration;
  }
  return cudaGetLastError();
}

cudaError_t launch_sweep_imp(const SweepArgs &a, const int2 *tasks, int ntasks, int *prog, unsigned *ticket,
                             cudaStream_t s) {
  return a.g.dim == 3 ? launch_sweep_imp_dim<3>(a, tasks, ntasks, prog, ticket, s)
                      : launch_sweep_imp_dim<2>(a, tasks, ntasks, prog, ticket, s);
}

// CUDA-graph replay of steps: the step index of the error key lives on the device
__global__ void k_step_tick(unsigned long long *ctr) { ++*ctr; }

cudaError_t launch_step_tick(unsigned long long *ctr, cudaStream_t s) {
  k_step_tick<<<1, 1, 0, s>>>(ctr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- diffuse ghosts

// g_b = [octant tree of sum_{j in outgoing octant} w_j|s_a| I_{j,b}] / den (reading #11).
// One CTA per boundary face of this rank; threads over channels.
// Boundary face lf (0.. this rank's faces of `region`) -> global face index
// (the ghost-table row) and the (plane, cross) offset of its boundary cell.
__device__ __forceinline__ void wall_face(const Geometry &g, int region, int64_t lf, int64_t *face,
                                          int64_t *cell_base) {
  const int axis = region >> 1;
  const bool hi = region & 1;
  int x = 0, y = 0, p = 0;
  if (g.dim == 3) {
    if (axis == 0) {
      y = (int)(lf % g.ny);
      p = (int)(lf / g.ny);
      x = hi ? g.nx - 1 : 0;
      *face = y + (int64_t)g.ny * (g.m0 + p);
    } else if (axis == 1) {
      x = (int)(lf % g.nx);
      p = (int)(lf / g.nx);
      y = hi ? g.ny - 1 : 0;
      *face = x + (int64_t)g.nx * (g.m0 + p);
    } else {
      x = (int)(lf % g.nx);
      y = (int)(lf / g.nx);
      p = hi ? g.nplanes - 1 : 0;
      *face = x + (int64_t)g.nx * y;
    }
  } else {
    if (axis == 0) {
      p = (int)lf;
      x = hi ? g.nx - 1 : 0;
      *face = g.m0 + p;
    } else {
      x = (int)lf;
      p = hi ? g.nplanes - 1 : 0;
      *face = x;
    }
  }
  const int64_t cross = (g.dim == 3) ? x + (int64_t)g.nx * y : x;
  *cell_base = (int64_t)(p + g.plane_off) * g.plane_stride + cross * g.Es;
}

static int64_t wall_faces_local(const Geometry &g, int region) {
  const int axis = region >> 1;
  if (g.dim == 3)
    return axis == 0 ? (int64_t)g.ny * g.nplanes : (axis == 1 ? (int64_t)g.nx * g.nplanes : (int64_t)g.nx * g.ny);
  return axis == 0 ? g.nplanes : g.nx;
}

__device__ __forceinline__ void diffuse_face(const Geometry &g, const double *__restrict__ I, int region,
                                             int64_t face, int64_t cell_base, double *__restrict__ gtab,
                                             double *chg = nullptr) {
  const int axis = region >> 1;
  const bool hi = region & 1;
  // outgoing octants: s_a < 0 on the low wall (bit set), s_a >= 0 on the high wall
  const int bit = axis == 0 ? 4 : (axis == 1 ? 2 : 1);
  for (int b = threadIdx.x; b < g.nb; b += blockDim.x) {
    double q[8];  // compile-time octant indices: registers, not local memory
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int sl = g.oct_slot[o];
      const bool out = hi ? !(o & bit) : (o & bit);
      double acc = 0.0;
      if (sl >= 0 && out) {
        const double *ws = g.ws + (int64_t)axis * g.nslot * g.nj + (int64_t)sl * g.nj;
        const double *Ip = I + g.slot_off[sl] + cell_base + b;
        for (int j = 0; j < g.nj; ++j) acc += ws[j] * Ip[(int64_t)j * g.nb];
      }
      q[o] = acc;
    }
    const double num = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    const double gv = num / g.diff_den[region];
    if (chg) {  // relative change against the table's previous content (R-n convergence)
      const double old = gtab[face * g.nb + b];
      *chg = fmax(*chg, fabs(gv - old) / fabs(old));
    }
    gtab[face * g.nb + b] = gv;
  }
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *w, double x) {
  // non-negative doubles order like their bit patterns
  if (x > 0.0) atomicMax(w, (unsigned long long)__double_as_longlong(x));
}

// block-wide max of a non-negative value, then one atomic per block (the
// per-thread atomics on one word serialised: 12 ms per snapshot on config 3)
__device__ __forceinline__ void block_max_to(unsigned long long *w, double x) {
  __shared__ double wm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // wm may still be read by a previous call
  if (lane == 0) wm[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)((blockDim.x + 31) >> 5); ++k) m = fmax(m, wm[k]);
    atomic_max_nonneg(w, m);
  }
}

__global__ void k_diffuse(const Geometry g, const double *__restrict__ I, int region,
                          double *__restrict__ gtab, unsigned long long *chg) {
  int64_t face, cell_base;
  wall_face(g, region, blockIdx.x, &face, &cell_base);
  double m = 0.0;
  diffuse_face(g, I, region, face, cell_base, gtab, chg ? &m : nullptr);
  if (chg) block_max_to(chg, m);
}

cudaError_t launch_diffuse(const Geometry &g, const double *I, int region, double *gtab,
                           cudaStream_t s, unsigned long long *chg) {
  const int64_t nf = wall_faces_local(g, region);
  if (nf == 0) return cudaSuccess;
  int threads = ((g.nb + 31) / 32) * 32;
  if (threads > 256) threads = 256;
  k_diffuse<<<(unsigned)nf, threads, 0, s>>>(g, I, region, gtab, chg);
  return cudaGetLastError();
}

constexpr int kMaxSnapJ = 1024;  // directions per octant handled by k_spec_snapshot

// Octant-slot rotation: specular ghosts read the reflected
// octant, whose slot may already hold I^{n+1} or another octant when this
// octant is swept, so the boundary pass snapshots them from I^n first:
// out[face][slot][j][b] = I^n of the boundary cell at the reflection of (slot, j).
__global__ void k_spec_snapshot(const Geometry g, const double *__restrict__ I, int region,
                                double *__restrict__ out, const int4 ins_lo, const int4 ins_hi,
                                unsigned long long *chg) {
  const int axis = region >> 1;
  int64_t face, cell_base;
  wall_face(g, region, blockIdx.x, &face, &cell_base);
  // blockIdx.y: the y-th slot whose directions enter through this wall
  // (s_a >= 0 on the low wall, s_a < 0 on the high wall; host-built list)
  const int k = blockIdx.y;
  const int slot = k < 4 ? (k == 0 ? ins_lo.x : k == 1 ? ins_lo.y : k == 2 ? ins_lo.z : ins_lo.w)
                         : (k == 4 ? ins_hi.x : k == 5 ? ins_hi.y : k == 6 ? ins_hi.z : ins_hi.w);
  const int nsj = g.nslot * g.nj;
  const int64_t *ro = g.refl_off + (int64_t)axis * nsj + (int64_t)slot * g.nj;
  double *o = out + (face * g.nslot + slot) * (int64_t)g.E;
  // per direction j the source row (reflected slot region, reflected j) of this cell
  __shared__ const double *srow[kMaxSnapJ];
  for (int j = threadIdx.x; j < g.nj; j += blockDim.x) {
    const int64_t off = ro[j];  // slot_r * slot_stride + jr * nb
    const int64_t sr = off / g.slot_stride;
    srow[j] = I + g.slot_off[sr] + (off - sr * g.slot_stride) + cell_base;
  }
  __syncthreads();
  double m = 0.0;  // relative change against the previous snapshot (R-n convergence)
  if ((g.nb & 1) == 0) {  // 16-B rows: double2 copies
    const int hp = g.nb >> 1;
    for (int e = threadIdx.x; e < g.nj * hp; e += blockDim.x) {
      const int j = e / hp, q = e - j * hp;
      double2 *dst = reinterpret_cast<double2 *>(o + (int64_t)j * g.nb) + q;
      const double2 val = __ldg(reinterpret_cast<const double2 *>(srow[j]) + q);
      if (chg) {
        const double2 old = *dst;
        m = fmax(m, fmax(fabs(val.x - old.x) / fabs(old.x), fabs(val.y - old.y) / fabs(old.y)));
      }
      *dst = val;
    }
  } else {
    for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
      const int j = e / g.nb, b = e - j * g.nb;
      const double val = srow[j][b];
      if (chg) m = fmax(m, fabs(val - o[e]) / fabs(o[e]));
      o[e] = val;
    }
  }
  if (chg) block_max_to(chg, m);
}

cudaError_t launch_spec_snapshot(const Geometry &g, const double *I, int region, double *out, cudaStream_t s,
                                 unsigned long long *chg) {
  const int64_t nf = wall_faces_local(g, region);
  if (nf == 0) return cudaSuccess;
  if (g.nj > kMaxSnapJ) return cudaErrorInvalidValue;
  const int axis = region >> 1, bit = axis == 0 ? 4 : (axis == 1 ? 2 : 1);
  const bool hi = region & 1;
  int ins[8] = {0, 0, 0, 0, 0, 0, 0, 0}, nin = 0;
  for (int sl = 0; sl < g.nslot; ++sl) {
    const int oct = g.slot_oct[sl];
    if (hi ? (oct & bit) : !(oct & bit)) ins[nin++] = sl;  // entering through this wall
  }
  if (nin == 0) return cudaSuccess;
  const int thr = std::min(256, (g.E + 31) / 32 * 32);
  k_spec_snapshot<<<dim3((unsigned)nf, (unsigned)nin), thr, 0, s>>>(
      g, I, region, out, make_int4(ins[0], ins[1], ins[2], ins[3]), make_int4(ins[4], ins[5], ins[6], ins[7]), chg);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Newton

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // bitwise identical in every lane (IEEE addition is commutative)
}

constexpr int kNewtonWarps = 8;
#ifndef BTE_NEWTON_MINB
#define BTE_NEWTON_MINB 4  // resident blocks per SM (caps registers at 64)
#endif

// 1/x for x > 0 finite: MUFU seed + two Newton-Raphson steps (<= 1 ulp);
// +inf -> 0 (a Bose-Einstein term whose exponent overflowed contributes 0).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return x < 1e300 ? r : 0.0;
}

// a3 + a4.  One warp per cell (persistent grid, warps stride over cells).
// Channel-wise work (octant tree, beta_next, c_b) uses lanes over channels;
// the band integrals use lanes over (channel, Gauss node) pairs: lane l owns
// node j = l & 15 of channels b = (l >> 4) + 2m, so every lane evaluates
// ceil(nb/2) expm1 per F(T) instead of 16 * ceil(nb/32).
//   F(T)  = W sum_b c_b I0_b(T) + K0,  K0 = sum_b c_b (D_b - W I0c_b)
//   F'(T) = W sum_b c_b dI0_b/dT
// F(T^n) = sum_b c_b D_b exactly (I0c = I0(T^n)) and F'(T^n) uses the dI0/dT
// stored by the previous refresh, so the first Newton step costs no integral.
// Newton of one cell by one warp (a3 + a4).  sA/sX: GL tables [nb][16] in
// shared memory, cs: [nb] scratch of this warp.  Dpart is read with
// ld.global.cg because, when fused into the sweep, other CTAs wrote it.
// Per-channel band integrals at T on the uniform band grid, balanced over the
// warp: task k = round*32 + lane -> channel b = k/4, nodes 4(k%4)..4(k%4)+3;
// the quad of lanes of one channel combine with two xor-shuffles.  Writes
// I0_b(T), dI0_b/dT and d2I0_b/dT2 to sI0/sD0/sD2; returns W*sum c_b I0_b and
// W*sum c_b dI0_b/dT in *F (without K0) and *Fp (identical in every lane).
// Node term g = A/(e^x - 1), x = X/T, r = 1/(e^x - 1):
//   dg/dT = g (x/T)(1 + r),   d2g/dT2 = g (1 + r)(x/T^2)(x(1 + 2r) - 2).
__device__ __forceinline__ void eval_channels(const NewtonArgs &a, double T, const double *sA, const int *sIB,
                                           double *scr, int lane, double *F, double *Fp) {
  const int nb = a.nb;
  const double *cs = scr;
  double *sE = scr + nb, *sM = sE + kNGL, *sR = sM + kNGL;
  double *sI0 = sR + a.m.imax + 1, *sD0 = sI0 + nb, *sD2 = sD0 + nb;
  const double rT = 1.0 / T;
  const double aa = a.m.Xd * rT;
  __syncwarp();
  if (lane < kNGL) {
    const double x0 = aa * a.m.U[lane];
    sE[lane] = exp(x0);
    sM[lane] = expm1(x0);
  }
  for (int i = lane; i <= a.m.imax; i += 32) sR[i] = exp(aa * (double)i);
  __syncwarp();
  double facc = 0.0, fpacc = 0.0;
  const int R = gl_stride(nb);
  if (a.lpc) {
    // lane per channel: all 16 nodes of channel b in one lane, no cross-lane
    // sums; ceil(nb/32) rounds instead of ceil(nb/8) (chosen by channel count)
    for (int b = lane; b < nb; b += 32) {
      const int ib = sIB[b];
      const double Rb = sR[ib];
      const double bi = (double)ib;
      double f = 0.0, fp = 0.0, f2 = 0.0;
#pragma unroll 4
      for (int j = 0; j < kNGL; ++j) {
        const double em1 = (ib == 0) ? sM[j] : fma(sE[j], Rb, -1.0);
        const double rr = rcp_nr(em1);
        const double t = sA[j * R + b] * rr;
        const double x = aa * (bi + __ldg(a.m.U + j));
        const double tq = t * (1.0 + rr);
        f += t;
        fp = fma(tq, x, fp);
        f2 = fma(tq * x, fma(x, fma(2.0, rr, 1.0), -2.0), f2);
      }
      const double d = fp * rT;
      sI0[b] = f;
      sD0[b] = d;
      sD2[b] = f2 * rT * rT;
      facc += cs[b] * f;
      fpacc += cs[b] * d;
    }
    *F = a.W * warp_sum(facc);
    *Fp = a.W * warp_sum(fpacc);
    __syncwarp();
    return;
  }
  const int q = lane >> 3;            // node group: nodes 4q .. 4q+3
  double u[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) u[jj] = a.m.U[4 * q + jj];
  const int nrounds = (nb + 7) / 8;
  for (int rd = 0; rd < nrounds; ++rd) {
    const int b = rd * 8 + (lane & 7);
    double f = 0.0, fp = 0.0, f2 = 0.0;
    if (b < nb) {
      const int ib = sIB[b];  // band index of channel b (shared-memory copy of a.m.ib)
      const double Rb = sR[ib];
      const double bi = (double)ib;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = 4 * q + jj;
        const double em1 = (ib == 0) ? sM[j] : fma(sE[j], Rb, -1.0);
        const double rr = rcp_nr(em1);
        const double t = sA[j * R + b] * rr;
        const double x = aa * (bi + u[jj]);
        const double tq = t * (1.0 + rr);
        f += t;
        fp = fma(tq, x, fp);
        f2 = fma(tq * x, fma(x, fma(2.0, rr, 1.0), -2.0), f2);
      }
    }
    f += __shfl_xor_sync(0xffffffffu, f, 8);
    fp += __shfl_xor_sync(0xffffffffu, fp, 8);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 8);
    f += __shfl_xor_sync(0xffffffffu, f, 16);
    fp += __shfl_xor_sync(0xffffffffu, fp, 16);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 16);
    if (q == 0 && b < nb) {
      const double d = fp * rT;
      sI0[b] = f;
      sD0[b] = d;
      sD2[b] = f2 * rT * rT;
      facc += cs[b] * f;
      fpacc += cs[b] * d;
    }
  }
  *F = a.W * warp_sum(facc);
  *Fp = a.W * warp_sum(fpacc);
  __syncwarp();
}

template <bool BAND>
__device__ void newton_cell(const NewtonArgs &a, int64_t c, const double *sA, const double *sX, const int *sI,
                            double *cs, int lane) {
  const int nb = a.nb;
  const bool be = a.m.mode != 0;
  const int jn = lane & 15;
  const int par = lane >> 4;
  const double Tn = a.T[c];
  double F0 = 0.0, K0 = 0.0, Fp0 = 0.0;
  if (BAND) {
    // band partition: F(T^n) = sum_b c_b D_b arrives as one partial per part,
    // summed in part order (identical on every part)
    for (int r = 0; r < a.nparts; ++r) F0 += __ldcg(a.Sall + (int64_t)r * a.ncells + c);
    for (int b = lane; b < nb; b += 32) {
      const double bn = beta_of_T(a.m.bcoef, b, Tn);
      const double cb = bn * a.m.rv[b];
      cs[b] = cb;
      a.beta_next[c * nb + b] = bn;
      if (b >= a.b0s && b < a.b0s + a.nbs) a.betas[c * a.nbs + b - a.b0s] = bn;  // the sweep's rows
      K0 -= cb * (a.W * a.I0c[c * nb + b]);
      Fp0 += cb * (a.W * a.dI0c[c * nb + b]);
    }
    K0 = F0 + warp_sum(K0);
    Fp0 = warp_sum(Fp0);
  } else {
  for (int b = lane; b < nb; b += 32) {
    double q[8];  // octant-indexed with compile-time indices: stays in registers
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int sl = a.oct_slot[o];
      q[o] = sl >= 0 ? __ldcg(a.Dpart + (c * a.nslot + sl) * nb + b) : 0.0;
    }
    const double D = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    // implicit step (R-n): the step's beta(T^n), stored at its start, weights every iteration
    const double bn = a.beta_fixed ? a.beta_next[c * nb + b] : beta_of_T(a.m.bcoef, b, Tn);
    // semi-implicit step (reading R-l): weights beta / (v (1 + dt beta))
    const double cb = a.semi_dt > 0.0 ? bn * a.m.rv[b] / (1.0 + a.semi_dt * bn) : bn * a.m.rv[b];
    cs[b] = cb;
    if (!a.beta_fixed) a.beta_next[c * nb + b] = bn;
    F0 += cb * D;
    K0 += cb * (D - a.W * a.I0c[c * nb + b]);
    Fp0 += cb * (a.W * a.dI0c[c * nb + b]);
  }
  F0 = warp_sum(F0);
  K0 = warp_sum(K0);
  Fp0 = warp_sum(Fp0);
  }
  __syncwarp();
  double Tf = Tn;
  double evaluated_at = -1.0;  // T of the per-channel values held in sI0/sD0
  int status = ERR_NONE;
  if (!isfinite(F0) || !isfinite(K0)) {
    status = ERR_NONFINITE;
  } else if (F0 != 0.0) {
    if (a.stats && lane == 0) atomicAdd(a.stats + 2, 1ull);
    double T = Tn, lo = kTlo, hi = kThi, F = F0, Fp = Fp0;
    double Tprev = 0.0, Fpprev = 0.0;
    bool conv = false, final_eval = false;
    const bool uni = be && a.m.uniform;
    // one evaluation call site: the refresh evaluation (when the Taylor step of
    // reading R-g does not apply) runs as a final pass of this loop
    for (int it = 0; it <= kNewtonMaxIt + 1; ++it) {
      if (it > 0) {
        if (uni) {
          double fw, fpw;
          eval_channels(a, T, sA, sI + 4 * (a.m.imax + 1), cs, lane, &fw, &fpw);
          F = fw + K0;
          Fp = fpw;
          evaluated_at = T;
        } else {
          double f = 0.0, fp = 0.0;
          const double rT = 1.0 / T;
          if (be) {
            for (int b = par; b < nb; b += 2) {
              const double x = sX[jn * gl_stride(nb) + b] * rT;
              const double em1 = expm1(x);
              const double r = 1.0 / em1;
              const double t = cs[b] * (sA[jn * gl_stride(nb) + b] * r);
              f += t;
              fp += t * x * (1.0 + r);
            }
            fp *= rT;
          } else {
            for (int b = lane; b < nb; b += 32) {
              f += cs[b] * (a.m.I_ref[b] + a.m.slope[b] * (T - a.m.T_ref));
              fp += cs[b] * a.m.slope[b];
            }
          }
          F = a.W * warp_sum(f) + K0;
          Fp = a.W * warp_sum(fp);
        }
      }
      if (a.stats && lane == 0 && it > 0) atomicAdd(a.stats + (final_eval ? 1 : 0), 1ull);
      if (final_eval) break;
      if (!isfinite(F) || !isfinite(Fp)) {
        status = ERR_NONFINITE;
        break;
      }
      bool done = false;
      if (F == 0.0) {
        Tf = T;
        done = true;
      } else {
        if (it >= kNewtonMaxIt) break;
        if (F < 0.0)
          lo = T;
        else
          hi = T;
        const double stp = F / Fp;
        double Tn1 = T - stp;
        if (fabs(stp) <= kNewtonRtol * T) {  // reading R-a: step test before the bracket test
          Tf = Tn1;
          done = true;
        } else if (it > 0 && a.predict && Tn1 > lo && Tn1 < hi) {
          // reading R-f: quadratic convergence -- the next step would be about
          // |F''/(2F')| stp^2 (F'' from the secant of F'); accept T - stp when
          // that is 1000x below the tolerance, saving one evaluation.
          const double F2 = (Fp - Fpprev) / (T - Tprev);
          const double pred = fabs(F2 / (2.0 * Fp)) * stp * stp;
          if (pred <= 1e-3 * kNewtonRtol * T) {
            Tf = Tn1;
            done = true;
          }
        }
        if (!done) {
          Tprev = T;
          Fpprev = Fp;
          if (!(Tn1 > lo && Tn1 < hi)) Tn1 = 0.5 * (lo + hi);
          T = Tn1;
        }
      }
      if (done) {
        conv = true;
        if (uni && Tf != Tn) {
          const double rel = fabs(Tf - evaluated_at) / Tf;
          if (!(evaluated_at > 0.0 && 10.0 * rel * rel * rel <= 1e-16)) {
            final_eval = true;  // re-evaluate at T^{n+1} for the refresh
            T = Tf;
            continue;
          }
        }
        break;
      }
    }
    if (!conv && status == ERR_NONE) status = ERR_NEWTON;
  }
  if (status != ERR_NONE) {
    if (lane == 0) {
      const unsigned long long key = ((unsigned long long)(a.step_ctr ? *a.step_ctr : (unsigned long long)a.step) << 40) | ((unsigned long long)status << 36) |
                                     (unsigned long long)(a.cell0_global + c);
      atomicMin(a.err, key);
    }
    __syncwarp();
    return;
  }
  if (Tf != Tn) {
    // refresh I0c = I0(T^{n+1}) and its derivative
    if (lane == 0) a.T[c] = Tf;
    if (a.dTmax && lane == 0) atomic_max_nonneg(a.dTmax, fabs(Tf - Tn) / Tn);
    if (be && a.m.uniform) {
      // refresh from the per-channel values of the last evaluation (at Tf itself
      // after a final pass, else the second-order Taylor step of reading R-g)
      double *sI0 = cs + nb + 2 * kNGL + a.m.imax + 1;
      double *sD0 = sI0 + nb, *sD2 = sD0 + nb;
      const double dT = Tf - evaluated_at;
      for (int b = lane; b < nb; b += 32) {
        const double i0 = sI0[b], d0 = sD0[b], d2 = sD2[b];
        a.I0c[c * nb + b] = dT != 0.0 ? fma(fma(0.5 * d2, dT, d0), dT, i0) : i0;
        a.dI0c[c * nb + b] = dT != 0.0 ? fma(d2, dT, d0) : d0;
      }
    } else if (be) {
      const double rT = 1.0 / Tf;
      for (int b0 = 0; b0 < nb; b0 += 2) {
        const int b = b0 + par;
        double f = 0.0, fp = 0.0;
        if (b < nb) {
          const double x = sX[jn * gl_stride(nb) + b] * rT;
          const double em1 = expm1(x);
          const double r = 1.0 / em1;
          f = sA[jn * gl_stride(nb) + b] * r;
          fp = f * x * (1.0 + r);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          f += __shfl_xor_sync(0xffffffffu, f, o);
          fp += __shfl_xor_sync(0xffffffffu, fp, o);
        }
        if (jn == 0 && b < nb) {
          a.I0c[c * nb + b] = f;
          a.dI0c[c * nb + b] = fp * rT;
        }
      }
    } else {
      for (int b = lane; b < nb; b += 32) a.I0c[c * nb + b] = a.m.I_ref[b] + a.m.slope[b] * (Tf - a.m.T_ref);
    }
    if (BAND) {  // band partition: this part's slice for its sweep (__syncwarp orders the warp's writes)
      __syncwarp();
      for (int b = lane; b < a.nbs; b += 32) a.I0s[c * a.nbs + b] = a.I0c[c * nb + a.b0s + b];
    }
  }
  __syncwarp();
}

// a3 + a4 as a separate kernel: one warp per cell, persistent grid.
// Channel-wise work (octant tree, beta_next, c_b) uses lanes over channels;
// the band integrals use lanes over (channel, Gauss node) pairs: lane l owns
// node j = l & 15 of channels b = (l >> 4) + 2m, so every lane evaluates
// ceil(nb/2) expm1 per F(T).
//   F(T)  = W sum_b c_b I0_b(T) + K0,  K0 = sum_b c_b (D_b - W I0c_b)
//   F'(T) = W sum_b c_b dI0_b/dT
// F(T^n) = sum_b c_b D_b exactly (I0c = I0(T^n)) and F'(T^n) uses the dI0/dT
// stored by the previous refresh, so the first Newton step costs no integral.
template <int MINB, bool BAND>
__global__ void __launch_bounds__(32 * kNewtonWarps, MINB) k_newton(const NewtonArgs a) {
  extern __shared__ double nsh[];
  const int nb = a.nb;
  const int R = gl_stride(nb);
  double *sA = nsh;
  double *sX = sA + R * kNGL;
  const int warp = threadIdx.x >> 5;
  const int wsd = newton_scratch(a.m, nb);
  double *cs = sX + R * kNGL + warp * wsd;
  int *sI = reinterpret_cast<int *>(sX + R * kNGL + kNewtonWarps * wsd);
  if (a.m.mode != 0) {
    for (int i = threadIdx.x; i < nb * kNGL; i += blockDim.x) {  // node-major transpose
      const int b = i / kNGL, j = i - b * kNGL;
      sA[j * R + b] = a.m.A[i];
      sX[j * R + b] = a.m.X[i];
    }
    for (int i = threadIdx.x; i < 4 * (a.m.imax + 1); i += blockDim.x) sI[i] = a.m.ichan[i];
    if (a.m.uniform)  // band index per channel, after ichan (read every eval_channels round)
      for (int i = threadIdx.x; i < nb; i += blockDim.x) sI[4 * (a.m.imax + 1) + i] = a.m.ib[i];
  }
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * kNewtonWarps;
  // cells of the column range [col0, col0 + ncols) over all planes
  const int64_t ncol = a.ncols, nq = ncol * a.nplanes;
  const int lane = threadIdx.x & 31;
  for (int64_t q = (int64_t)blockIdx.x * kNewtonWarps + warp; q < nq; q += nwarps) {
    const int64_t p = q / ncol;
    newton_cell<BAND>(a, a.col0 + (q - p * ncol) + p * a.ncross, sA, sX, sI, cs, lane);
  }
}

// Self-consistent tau (reading R-k): one warp per cell, lanes
// over channels (up to kScCh per lane), direct band integrals.  Solves
//   F(T) = sum_b (beta_b(T)/v_b) [W (I0_b(T) - I0c_b) + D_b] = 0,
//   F'(T) = sum_b [(beta_b'(T)/v_b)(W (I0_b - I0c_b) + D_b) + (beta_b/v_b) W dI0_b/dT],
// with the bracket and step rules of the lagged Newton (reading #18, R-a; a
// bisection also when F' <= 0), then refreshes I0c, dI0c and beta at T^{n+1}.
constexpr int kScCh = kMaxBands / 32;

__global__ void __launch_bounds__(256) k_newton_sc(const NewtonArgs a) {
  const int lane = threadIdx.x & 31;
  const int nb = a.nb;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t ncol = a.ncols, nq = ncol * a.nplanes;
  for (int64_t qq = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); qq < nq; qq += nwarps) {
    const int64_t pl = qq / ncol;
    const int64_t c = a.col0 + (qq - pl * ncol) + pl * a.ncross;
    const double Tn = a.T[c];
    double D[kScCh], I0c[kScCh], i0v[kScCh], di0v[kScCh];
#pragma unroll
    for (int r = 0; r < kScCh; ++r) {
      const int b = lane + 32 * r;
      D[r] = 0.0;
      I0c[r] = 0.0;
      if (b < nb) {
        double q[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          const int sl = a.oct_slot[o];
          q[o] = sl >= 0 ? __ldcg(a.Dpart + (c * a.nslot + sl) * nb + b) : 0.0;
        }
        D[r] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
        I0c[r] = a.I0c[c * nb + b];
      }
    }
    double T = Tn, lo = kTlo, hi = kThi, Tf = Tn, evaluated_at = -1.0;
    int status = ERR_NEWTON;
    for (int it = 0; it <= kNewtonMaxIt; ++it) {
      double f = 0.0, fp = 0.0;
#pragma unroll
      for (int r = 0; r < kScCh; ++r) {
        const int b = lane + 32 * r;
        if (b < nb) {
          double d;
          const double i0 = I0_of_T(a.m, b, T, &d);
          i0v[r] = i0;
          di0v[r] = d;
          const double h = a.W * (i0 - I0c[r]) + D[r];
          const double rv = a.m.rv[b];
          f += beta_of_T(a.m.bcoef, b, T) * rv * h;
          fp += dbeta_of_T(a.m.bcoef, b, T) * rv * h + beta_of_T(a.m.bcoef, b, T) * rv * (a.W * d);
        }
      }
      const double F = warp_sum(f), Fp = warp_sum(fp);
      evaluated_at = T;
      if (!isfinite(F) || !isfinite(Fp)) {
        status = ERR_NONFINITE;
        break;
      }
      if (F == 0.0) {
        Tf = T;
        status = ERR_NONE;
        break;
      }
      if (it == kNewtonMaxIt) break;
      if (F < 0.0)
        lo = T;
      else
        hi = T;
      const double stp = F / Fp;
      double Tn1 = T - stp;
      if (fabs(stp) <= kNewtonRtol * T) {
        Tf = Tn1;
        status = ERR_NONE;
        break;
      }
      if (!(Tn1 > lo && Tn1 < hi) || !(Fp > 0.0)) Tn1 = 0.5 * (lo + hi);
      T = Tn1;
    }
    if (status != ERR_NONE) {
      if (lane == 0) {
        const unsigned long long key = ((unsigned long long)(a.step_ctr ? *a.step_ctr : (unsigned long long)a.step) << 40) | ((unsigned long long)status << 36) |
                                       (unsigned long long)(a.cell0_global + c);
        atomicMin(a.err, key);
      }
      continue;
    }
    if (lane == 0) a.T[c] = Tf;
#pragma unroll
    for (int r = 0; r < kScCh; ++r) {
      const int b = lane + 32 * r;
      if (b < nb) {
        double i0 = i0v[r], d = di0v[r];
        if (evaluated_at != Tf) i0 = I0_of_T(a.m, b, Tf, &d);
        a.I0c[c * nb + b] = i0;
        a.dI0c[c * nb + b] = d;
        a.beta_next[c * nb + b] = beta_of_T(a.m.bcoef, b, Tf);
      }
    }
  }
}

// Self-consistent tau on uniform band grids (reading R-k with the band
// integrals of reading R-d): one warp per cell; iteration 0 uses the exact
// F(T^n) = sum_b beta_b(T^n)/v_b D_b and F'(T^n) from the stored dI0/dT (no
// integral, exact fixed point); later iterations evaluate every channel's
// I0_b(T), dI0_b/dT with eval_channels.  Same bracket / step rules as
// k_newton_sc.
__global__ void __launch_bounds__(32 * kNewtonWarps, 4) k_newton_scu(const NewtonArgs a) {
  extern __shared__ double nsh[];
  const int nb = a.nb;
  const int R = gl_stride(nb);
  double *sA = nsh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ws0 = newton_scratch(a.m, nb);
  double *scr = sA + R * kNGL + warp * (ws0 + nb);
  double *sI0 = scr + nb + 2 * kNGL + a.m.imax + 1, *sD0 = sI0 + nb;
  double *sDb = scr + ws0;
  int *sIB = reinterpret_cast<int *>(sA + R * kNGL + kNewtonWarps * (ws0 + nb));  // [nb] band index per channel
  for (int i = threadIdx.x; i < nb * kNGL; i += blockDim.x) {
    const int b = i / kNGL, j = i - b * kNGL;
    sA[j * R + b] = a.m.A[i];
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sIB[i] = a.m.ib[i];
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * kNewtonWarps;
  const int64_t ncol = a.ncols, nq = ncol * a.nplanes;
  for (int64_t qq = (int64_t)blockIdx.x * kNewtonWarps + warp; qq < nq; qq += nwarps) {
    const int64_t pl = qq / ncol;
    const int64_t c = a.col0 + (qq - pl * ncol) + pl * a.ncross;
    const double Tn = a.T[c];
    double F0 = 0.0, Fp0 = 0.0;
    for (int b = lane; b < nb; b += 32) {
      double q[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int sl = a.oct_slot[o];
        q[o] = sl >= 0 ? __ldcg(a.Dpart + (c * a.nslot + sl) * nb + b) : 0.0;
      }
      const double D = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
      sDb[b] = D;
      scr[b] = 0.0;  // eval_channels' weights (its weighted sums are not used here)
      const double rv = a.m.rv[b];
      F0 += beta_of_T(a.m.bcoef, b, Tn) * rv * D;
      Fp0 += dbeta_of_T(a.m.bcoef, b, Tn) * rv * D + beta_of_T(a.m.bcoef, b, Tn) * rv * (a.W * a.dI0c[c * nb + b]);
    }
    F0 = warp_sum(F0);
    Fp0 = warp_sum(Fp0);
    __syncwarp();
    double T = Tn, lo = kTlo, hi = kThi, Tf = Tn, evaluated_at = -1.0;
    int status = ERR_NEWTON;
    for (int it = 0; it <= kNewtonMaxIt; ++it) {
      double F = F0, Fp = Fp0;
      if (it > 0) {
        double fw, fpw;
        eval_channels(a, T, sA, sIB, scr, lane, &fw, &fpw);
        evaluated_at = T;
        double f = 0.0, fp = 0.0;
        for (int b = lane; b < nb; b += 32) {
          const double h = a.W * (sI0[b] - a.I0c[c * nb + b]) + sDb[b];
          const double rv = a.m.rv[b];
          const double be = beta_of_T(a.m.bcoef, b, T);
          f += be * rv * h;
          fp += dbeta_of_T(a.m.bcoef, b, T) * rv * h + be * rv * (a.W * sD0[b]);
        }
        F = warp_sum(f);
        Fp = warp_sum(fp);
      }
      if (!isfinite(F) || !isfinite(Fp)) {
        status = ERR_NONFINITE;
        break;
      }
      if (F == 0.0) {
        Tf = T;
        status = ERR_NONE;
        break;
      }
      if (it == kNewtonMaxIt) break;
      if (F < 0.0)
        lo = T;
      else
        hi = T;
      const double stp = F / Fp;
      double Tn1 = T - stp;
      if (fabs(stp) <= kNewtonRtol * T) {
        Tf = Tn1;
        status = ERR_NONE;
        break;
      }
      if (!(Tn1 > lo && Tn1 < hi) || !(Fp > 0.0)) Tn1 = 0.5 * (lo + hi);
      T = Tn1;
    }
    if (status != ERR_NONE) {
      if (lane == 0) {
        const unsigned long long key = ((unsigned long long)(a.step_ctr ? *a.step_ctr : (unsigned long long)a.step) << 40) | ((unsigned long long)status << 36) |
                                       (unsigned long long)(a.cell0_global + c);
        atomicMin(a.err, key);
      }
      __syncwarp();
      continue;
    }
    if (Tf != Tn) {
      if (evaluated_at != Tf) {
        double fw, fpw;
        eval_channels(a, Tf, sA, sIB, scr, lane, &fw, &fpw);
      }
      if (lane == 0) a.T[c] = Tf;
      for (int b = lane; b < nb; b += 32) {
        a.I0c[c * nb + b] = sI0[b];
        a.dI0c[c * nb + b] = sD0[b];
        a.beta_next[c * nb + b] = beta_of_T(a.m.bcoef, b, Tf);
      }
    }
    __syncwarp();
  }
}

cudaError_t launch_newton_sc(const NewtonArgs &a, cudaStream_t s) {
  if (a.nb > kMaxBands) return cudaErrorInvalidValue;
  if (a.ncells == 0) return cudaSuccess;
  if (a.m.mode != 0 && a.m.uniform && !a.sc_direct) {
    const int64_t need = ((int64_t)a.ncols * a.nplanes + kNewtonWarps - 1) / kNewtonWarps;
    const int64_t nblk = std::min<int64_t>(need, 148 * 4);
    const size_t smem = ((size_t)gl_stride(a.nb) * kNGL + (size_t)kNewtonWarps * (newton_scratch(a.m, a.nb) + a.nb)) *
                            sizeof(double) + (size_t)a.nb * sizeof(int);
    if (cudaError_t e = smem_attr((const void *)k_newton_scu, smem)) return e;
    k_newton_scu<<<(unsigned)nblk, 32 * kNewtonWarps, smem, s>>>(a);
    return cudaGetLastError();
  }
  const int64_t need = ((int64_t)a.ncols * a.nplanes + 7) / 8;
  const int64_t nblk = std::min<int64_t>(need, 148 * 8);
  k_newton_sc<<<(unsigned)nblk, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_newton(const NewtonArgs &a, cudaStream_t s) {
  if (a.nb > kMaxBands) return cudaErrorInvalidValue;
  if (a.ncells == 0) return cudaSuccess;
  const int64_t need = ((int64_t)a.ncols * a.nplanes + kNewtonWarps - 1) / kNewtonWarps;
  const int64_t nblk = std::min<int64_t>(need, 148 * 8);
  const size_t smem = (2 * (size_t)gl_stride(a.nb) * kNGL + (size_t)kNewtonWarps * newton_scratch(a.m, a.nb)) * sizeof(double) +
                      (4 * (size_t)(a.m.imax + 1) + (size_t)a.nb) * sizeof(int);
  const int minb = a.minb > 0 ? a.minb : BTE_NEWTON_MINB;
  if (a.Sall) {  // band partition (bte_create_band)
    if (cudaError_t e = smem_attr((const void *)k_newton<BTE_NEWTON_MINB, true>, smem)) return e;
    k_newton<BTE_NEWTON_MINB, true><<<(unsigned)nblk, 32 * kNewtonWarps, smem, s>>>(a);
    return cudaGetLastError();
  }
#define BTE_NL(M)                                                                                   \
  case M:                                                                                           \
    if (cudaError_t e = smem_attr((const void *)k_newton<M, false>, smem)) return e;              \
    k_newton<M, false><<<(unsigned)nblk, 32 * kNewtonWarps, smem, s>>>(a);                          \
    break;
  switch (minb) {
    BTE_NL(2)
    BTE_NL(3)
    BTE_NL(4)
    BTE_NL(5)
    BTE_NL(6)
    default:
      return cudaErrorInvalidValue;
  }
#undef BTE_NL
  return cudaGetLastError();
}

// ---------------------------------------------------------------- tables / state helpers

__global__ void k_iso_table(const Material m, const double *__restrict__ Tw, int64_t nf,
                            double *__restrict__ g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf * m.nb) return;
  const int64_t f = i / m.nb;
  const int b = (int)(i - f * m.nb);
  g[i] = I0_of_T(m, b, Tw[f], nullptr);
}

cudaError_t launch_iso_table(const Material &m, const double *Tw, int64_t nf, double *gtab,
                             cudaStream_t s) {
  const int64_t n = nf * m.nb;
  if (n == 0) return cudaSuccess;
  k_iso_table<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m, Tw, nf, gtab);
  return cudaGetLastError();
}

__global__ void k_refresh(const Material m, const double *__restrict__ T, int64_t nc,
                          double *__restrict__ I0c, double *__restrict__ dI0c, double *__restrict__ beta) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc * m.nb) return;
  const int64_t c = i / m.nb;
  const int b = (int)(i - c * m.nb);
  const double t = T[c];
  if (I0c) {  // (null: beta only -- the implicit step's beta(T^n))
    double d;
    I0c[i] = I0_of_T(m, b, t, &d);
    dI0c[i] = d;
  }
  beta[i] = beta_of_T(m.bcoef, b, t);
}

cudaError_t launch_refresh(const Material &m, const double *T, int64_t nc, double *I0c, double *dI0c,
                           double *beta, cudaStream_t s) {
  const int64_t n = nc * m.nb;
  if (n == 0) return cudaSuccess;
  k_refresh<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m, T, nc, I0c, dI0c, beta);
  return cudaGetLastError();
}

// I[slot][plane][cross][j][b] = I0c[cell][b] over owned planes
// I = I0c(cell) for every direction: one (slot, cell) block per block-iteration
// (persistent grid), the cell's I0c row staged in shared memory, channel index
// carried incrementally -- a streaming write of the whole state (the previous
// one-thread-per-element version spent three 64-bit divisions per element and
// ran at ~1.2 TB/s: 107 ms for config 4's 128 GB).
__global__ void __launch_bounds__(256) k_fill_eq(const Geometry g, const double *__restrict__ I0c,
                                                 double *__restrict__ I) {
  __shared__ double row[kMaxBands];
  const int64_t ncell = (int64_t)g.nplanes * g.ncross;
  const int64_t items = ncell * g.nslot;
  const int nb = g.nb, E = g.E;
  const int b0 = (int)threadIdx.x % nb, db = (int)blockDim.x % nb;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int sl = (int)(it / ncell);
    const int64_t cell = it - (int64_t)sl * ncell;
    __syncthreads();  // previous item's row fully read
    for (int t = threadIdx.x; t < nb; t += blockDim.x) row[t] = I0c[cell * nb + t];
    __syncthreads();
    double *dst = I + g.slot_off[sl] + (int64_t)g.plane_off * g.plane_stride + cell * g.Es;
    int b = b0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      dst[e] = row[b];
      b += db;
      if (b >= nb) b -= nb;
    }
  }
}

cudaError_t launch_fill_equilibrium(const Geometry &g, const double *I0c, double *I, cudaStream_t s) {
  const int64_t items = (int64_t)g.nplanes * g.ncross * g.nslot;
  if (items == 0 || g.E == 0) return cudaSuccess;
  if (g.nb > kMaxBands) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nblk = std::min<int64_t>(items, (int64_t)sms * 8);
  k_fill_eq<<<(unsigned)nblk, 256, 0, s>>>(g, I0c, I);
  return cudaGetLastError();
}

// canonical chunk [c0, c0+nc)[d][b] <-> layout.  dmap[d] = slot*nj + j.
__global__ void k_permute(const Geometry g, const int *__restrict__ dmap, int nd,
                          double *__restrict__ canon, int64_t c0, int64_t ncc, double *__restrict__ I,
                          int to_layout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_cell = (int64_t)nd * g.nb;
  if (i >= ncc * per_cell) return;
  const int64_t cr = i / per_cell;
  const int rem = (int)(i - cr * per_cell);
  const int d = rem / g.nb;
  const int b = rem - d * g.nb;
  const int sj = dmap[d];
  const int sl = sj / g.nj;
  const int j = sj - sl * g.nj;
  const int64_t c = c0 + cr;
  const int64_t p = c / g.ncross;
  const int64_t cross = c - p * g.ncross;
  const int64_t dst = g.slot_off[sl] + (p + g.plane_off) * g.plane_stride + cross * g.Es +
                      (int64_t)j * g.nb + b;
  if (to_layout)
    I[dst] = canon[i];
  else
    canon[i] = I[dst];
}

cudaError_t launch_permute(const Geometry &g, const int *dmap, int nd, const double *canon, int64_t c0,
                           int64_t ncc, double *I, int to_layout, cudaStream_t s) {
  const int64_t n = ncc * nd * g.nb;
  if (n == 0) return cudaSuccess;
  k_permute<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, dmap, nd, const_cast<double *>(canon), c0,
                                                          ncc, I, to_layout);
  return cudaGetLastError();
}

// gather selected cells (local canonical indices) of the layout into canonical
// [i][d][b] rows (bte_get_intensity_cells)
__global__ void k_gather_cells(const Geometry g, const int *__restrict__ dmap, int nd,
                               const int64_t *__restrict__ cells, int64_t n, const double *__restrict__ I,
                               double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_cell = (int64_t)nd * g.nb;
  if (i >= n * per_cell) return;
  const int64_t k = i / per_cell;
  const int rem = (int)(i - k * per_cell);
  const int d = rem / g.nb;
  const int b = rem - d * g.nb;
  const int sj = dmap[d];
  const int sl = sj / g.nj;
  const int j = sj - sl * g.nj;
  const int64_t c = cells[k];
  const int64_t p = c / g.ncross;
  const int64_t cross = c - p * g.ncross;
  out[i] = I[g.slot_off[sl] + (p + g.plane_off) * g.plane_stride + cross * g.Es + (int64_t)j * g.nb + b];
}

cudaError_t launch_gather_cells(const Geometry &g, const int *dmap, int nd, const int64_t *cells, int64_t n,
                                const double *I, double *out, cudaStream_t s) {
  const int64_t m = n * nd * g.nb;
  if (m == 0) return cudaSuccess;
  k_gather_cells<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(g, dmap, nd, cells, n, I, out);
  return cudaGetLastError();
}

// Semi-implicit step (reading R-l), last part: I = (J + dt beta I0c) / (1 + dt beta)
// over the owned cells of the output buffer (beta lagged, I0c refreshed at T^{n+1}).
__global__ void k_relax(const Geometry g, double *__restrict__ I, const double *__restrict__ I0c,
                        const double *__restrict__ beta, double dt) {
  // block (cell, slot); threads (b, j-lane): no integer division per element
  const int64_t cell = blockIdx.x;
  const int sl = blockIdx.y;
  const int b = threadIdx.x;
  const int64_t p = cell / g.ncross, cross = cell - p * g.ncross;
  double *blk = I + g.slot_off[sl] + (p + g.plane_off) * g.plane_stride + cross * g.Es;
  const double db = dt * beta[cell * g.nb + b];
  const double i0 = I0c[cell * g.nb + b];
  const double inv = 1.0 / (1.0 + db);
  for (int j = threadIdx.y; j < g.nj; j += blockDim.y) {
    double *x = blk + (int64_t)j * g.nb + b;
    *x = (*x + db * i0) * inv;
  }
}

cudaError_t launch_relax(const Geometry &g, double *I, const double *I0c, const double *beta, double dt,
                         cudaStream_t s) {
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  if (nc == 0 || g.nb > 1024) return nc == 0 ? cudaSuccess : cudaErrorInvalidValue;
  const int ty = std::max(1, std::min(g.nj, 256 / g.nb));
  k_relax<<<dim3((unsigned)nc, g.nslot), dim3(g.nb, ty), 0, s>>>(g, I, I0c, beta, dt);
  return cudaGetLastError();
}

// partitioned unstructured mesh: gather the blocks of `cells` (all octant
// slots) into out[slot][k][Es] (the halo copies a neighbour rank receives)
__global__ void k_pack_cells(const Geometry g, const int64_t *__restrict__ cells, int64_t n,
                             const double *__restrict__ I, double *__restrict__ out) {
  const int64_t k = blockIdx.x;
  const int sl = blockIdx.y;
  const double *src = I + g.slot_off[sl] + cells[k] * g.Es;
  double *dst = out + ((int64_t)sl * n + k) * g.Es;
  for (int e = threadIdx.x; e < g.Es; e += blockDim.x) dst[e] = src[e];
}

cudaError_t launch_pack_cells(const Geometry &g, const int64_t *cells, int64_t n, const double *I, double *out,
                              cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_pack_cells<<<dim3((unsigned)n, g.nslot), 256, 0, s>>>(g, cells, n, I, out);
  return cudaGetLastError();
}

__global__ void k_random_T(const Geometry g, double dx, double dy, double dz, double p0, double p1,
                           double p2, double T_mean, double T_amp, double *__restrict__ T) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  if (c >= nc) return;
  const double twopi = 6.283185307179586;
  double v;
  if (g.dim == 3) {
    const int64_t x = c % g.nx, y = (c / g.nx) % g.ny, z = g.m0 + c / ((int64_t)g.nx * g.ny);
    const double fx = sin(twopi * (((x + 0.5) * dx) / (g.nx * dx) + p0));
    const double fy = sin(twopi * (((y + 0.5) * dy) / (g.ny * dy) + p1));
    const double fz = sin(twopi * (((z + 0.5) * dz) / (g.nplanes_global * dz) + p2));
    v = T_mean + T_amp * (fz * fy * fx);
  } else {
    const int64_t x = c % g.nx, y = g.m0 + c / g.nx;
    const double fx = sin(twopi * (((x + 0.5) * dx) / (g.nx * dx) + p0));
    const double fy = sin(twopi * (((y + 0.5) * dy) / (g.nplanes_global * dy) + p1));
    v = T_mean + T_amp * (1.0 * fy * fx);
  }
  T[c] = v;
}

cudaError_t launch_random_T(const Geometry &g, int64_t, double dx, double dy, double dz,
                            const double *phase, double T_mean, double T_amp, double *T,
                            cudaStream_t s) {
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  if (nc == 0) return cudaSuccess;
  k_random_T<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(g, dx, dy, dz, phase[0], phase[1], phase[2],
                                                           T_mean, T_amp, T);
  return cudaGetLastError();
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// I = I0c * (1 + amp*(2u - 1)), u from the canonical global index (c_g*nd + d)*nbT + b0 + b
__global__ void k_random_I(const Geometry g, const int *__restrict__ canon_d, int nd, uint64_t seed,
                           double amp, const double *__restrict__ I0c, double *__restrict__ I) {
  const int64_t n_per_slot = (int64_t)g.nplanes * g.ncross * g.E;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_per_slot * g.nslot) return;
  const int sl = (int)(i / n_per_slot);
  const int64_t r = i - sl * n_per_slot;
  const int64_t cell = r / g.E;
  const int e = (int)(r - cell * g.E);
  const int j = e / g.nb;
  const int b = e - j * g.nb;
  const int d = canon_d[sl * g.nj + j];
  const int64_t cg = g.cell0 + cell;
  const uint64_t idx = ((uint64_t)cg * nd + d) * g.nbT + g.b0 + b;
  const double u = (double)(splitmix64(seed ^ idx) >> 11) * 0x1.0p-53;
  I[g.slot_off[sl] + (int64_t)g.plane_off * g.plane_stride + cell * g.Es + e] =
      I0c[cell * g.nb + b] * (1.0 + amp * (2.0 * u - 1.0));
}

cudaError_t launch_random_I(const Geometry &g, const int *canon_d, int nd, uint64_t seed, double amp,
                            const double *I0c, double *I, cudaStream_t s) {
  const int64_t n = (int64_t)g.nplanes * g.ncross * g.E * g.nslot;
  if (n == 0) return cudaSuccess;
  k_random_I<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, canon_d, nd, seed, amp, I0c, I);
  return cudaGetLastError();
}

__global__ void k_octant_tree(const double *__restrict__ Dpart, int nslot, Geometry g, int64_t nc,
                              double *__restrict__ D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc * g.nb) return;
  const int64_t c = i / g.nb;
  const int b = (int)(i - c * g.nb);
  double q[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) q[o] = g.oct_slot[o] >= 0 ? Dpart[(c * nslot + g.oct_slot[o]) * g.nb + b] : 0.0;
  D[i] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
}

cudaError_t launch_octant_tree_g(const Geometry &g, const double *Dpart, int64_t nc, double *D,
                                 cudaStream_t s) {
  const int64_t n = nc * g.nb;
  if (n == 0) return cudaSuccess;
  k_octant_tree<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(Dpart, g.nslot, g, nc, D);
  return cudaGetLastError();
}

// Dpart[c][slot][b] = sum_j w_j (I0c - I) of the given state (set_state with I only)
__global__ void k_dpart_from_I(const Geometry g, const double *__restrict__ I, const double *__restrict__ I0c,
                               double *__restrict__ Dpart) {
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc * g.nslot * g.nb) return;
  const int b = (int)(i % g.nb);
  const int sl = (int)((i / g.nb) % g.nslot);
  const int64_t c = i / ((int64_t)g.nb * g.nslot);
  const int64_t p = c / g.ncross, cross = c - p * g.ncross;
  const double *Ip = I + g.slot_off[sl] + (p + g.plane_off) * g.plane_stride + cross * g.Es + b;
  const double i0 = I0c[c * g.nb + b];
  double s = 0.0;
  for (int j = 0; j < g.nj; ++j) s += g.coef[(int64_t)(sl * g.nj + j) * 4 + 3] * (i0 - Ip[(int64_t)j * g.nb]);
  Dpart[i] = s;
}

cudaError_t launch_dpart_from_I(const Geometry &g, const double *I, const double *I0c, double *Dpart,
                               cudaStream_t s) {
  const int64_t n = (int64_t)g.nplanes * g.ncross * g.nslot * g.nb;
  if (n == 0) return cudaSuccess;
  k_dpart_from_I<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, I, I0c, Dpart);
  return cudaGetLastError();
}

// Band partition (bte_create_band): this part's share of F(T^n),
// S_r(c) = sum_{b in [b0, b0+nb)} c_b D_{c,b}, c_b = beta_b(T^n_c) / v_b, with
// D_{c,b} the octant tree of the sweep's partials.  One warp per cell.
__global__ void k_band_partial(const Geometry g, const Material mF, const double *__restrict__ Dpart,
                               const double *__restrict__ T, int64_t nc, double *__restrict__ S) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nc) return;
  const double Tn = T[c];
  double part = 0.0;
  for (int b = lane; b < g.nb; b += 32) {
    double q[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) q[o] = g.oct_slot[o] >= 0 ? Dpart[(c * g.nslot + g.oct_slot[o]) * g.nb + b] : 0.0;
    const double D = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    const int bg = g.b0 + b;
    const double cb = beta_of_T(mF.bcoef, bg, Tn) * mF.rv[bg];
    part += cb * D;
  }
  part = warp_sum(part);
  if (lane == 0) S[c] = part;
}

cudaError_t launch_band_partial(const Geometry &g, const Material &mF, const double *Dpart, const double *T,
                                int64_t nc, double *S, cudaStream_t s) {
  if (nc == 0) return cudaSuccess;
  k_band_partial<<<(unsigned)((nc * 32 + 255) / 256), 256, 0, s>>>(g, mF, Dpart, T, nc, S);
  return cudaGetLastError();
}

// per-cell energy density sum_slot sum_j sum_b w_j/v_b I (warp per cell)
__global__ void k_energy(const Geometry g, const double *__restrict__ I, const double *__restrict__ v,
                         double *__restrict__ Ec) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  if (c >= nc) return;
  const int64_t p = c / g.ncross, cross = c - p * g.ncross;
  double acc = 0.0;
  for (int sl = 0; sl < g.nslot; ++sl) {
    const double *Ip = I + g.slot_off[sl] + (p + g.plane_off) * g.plane_stride + cross * g.Es;
    for (int e = lane; e < g.E; e += 32) {
      const int j = e / g.nb, b = e - j * g.nb;
      acc += g.coef[(int64_t)(sl * g.nj + j) * 4 + 3] / v[b] * Ip[e];
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) Ec[c] = acc;
}

cudaError_t launch_energy(const Geometry &g, const double *I, const double *v, double *Ec, cudaStream_t s) {
  const int64_t nc = (int64_t)g.nplanes * g.ncross;
  if (nc == 0) return cudaSuccess;
  k_energy<<<(unsigned)((nc + 3) / 4), 128, 0, s>>>(g, I, v, Ec);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- unstructured meshes

// Eq. 3 on a simplex: one CTA per (cell, octant slot).  The CTA
// first forms a_{f,j} = dt * s_j . (A_f n_f / V_c) for its K faces and nj
// directions in shared memory; thread (grp, b) then updates channel b of
// directions [grp*jpt, grp*jpt + jpt):
//   I' = I + dt beta (I0c - I) - v_b sum_f a_{f,j} I_up,
//   I_up = I (own) if a > 0, else the neighbour's value (same slot, j, b) or
//   the wall ghost (P:L150-157 strict ">").
// Neighbour reads are 8*nb-byte coalesced rows of the neighbour's block; the
// octant partial sum over j feeds the same Dpart[c][slot][b] as the
// structured sweep (fixed order: within a thread ascending j, then groups).
template <int JMAX, int KM>
__global__ void __launch_bounds__(1024) k_usweep(const USweepArgs A) {
  extern __shared__ double sm[];  // a[K][nj] | red[JG*nb]
  __shared__ int64_t snbr[KM];
  const Geometry &g = A.g;
  const UMeshDev &u = A.u;
  const int nb = g.nb, nj = g.nj, Es = g.Es, K = u.K;
  const int tid = threadIdx.x;
  const int grp = tid / nb;
  const int b = tid - grp * nb;
  const int JG = A.jg;
  const int j0 = grp * A.jpt;
  const int nloc = max(0, min(A.jpt, nj - j0));
  const int64_t cell = blockIdx.x;
  const int slot = blockIdx.y;
  double *a = sm;
  double *red = sm + KM * nj;
  if (tid < K) snbr[tid] = u.nbr[cell * u.KP + tid];
  for (int i = tid; i < K * nj; i += blockDim.x) {
    const int f = i / nj, j = i - f * nj;
    const double *sv = u.sw + (int64_t)(slot * nj + j) * 4;
    const double *an = u.an + cell * 3 * u.KP + f * 3;
    a[f * nj + j] = A.dt * fma(sv[2], an[2], fma(sv[1], an[1], sv[0] * an[0]));
  }
  __syncthreads();
  const bool active = grp < JG;
  const double *__restrict__ Is = A.Iin + g.slot_off[slot];
  double *__restrict__ Os = A.Iout + g.slot_off[slot];
  const int64_t base = cell * Es;
  double acc = 0.0;
  if (active) {
    const double I0 = __ldg(A.I0c + cell * nb + b);
    const double dtb = A.dt * __ldg(A.beta + cell * nb + b);
    const double v = A.v[b];
    double Ic[JMAX], up[JMAX][KM];
#pragma unroll
    for (int k = 0; k < JMAX; ++k) {  // issue every load of the cell first
      if (k < nloc) {
        const int j = j0 + k;
        const int e = j * nb + b;
        Ic[k] = __ldg(Is + base + e);
#pragma unroll
        for (int f = 0; f < KM; ++f) {
          up[k][f] = 0.0;
          if (f < K && !(a[f * nj + j] > 0.0)) {
            const int64_t n = snbr[f];
            if (n >= 0) up[k][f] = __ldg(Is + n * Es + e);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < JMAX; ++k) {
      if (k < nloc) {
        const int j = j0 + k;
        const int e = j * nb + b;
        double flux = 0.0;
#pragma unroll
        for (int f = 0; f < KM; ++f) {
          if (f < K) {
            const double af = a[f * nj + j];
            double w;
            if (af > 0.0) {
              w = Ic[k];
            } else {
              const int64_t n = snbr[f];
              if (n >= 0) {
                w = up[k][f];
              } else {
                const int64_t code = -1 - n;
                w = ghost_value(g, A.Iin, (int)(code & 7), code >> 3, base, slot, j, b);
              }
            }
            flux = fma(af, w, flux);
          }
        }
        const double In = fma(dtb, I0 - Ic[k], Ic[k]) - v * flux;
        Os[base + e] = In;
        acc = fma(u.sw[(int64_t)(slot * nj + j) * 4 + 3], I0 - In, acc);
      }
    }
    red[tid] = acc;
  }
  __syncthreads();
  if (tid < nb) {
    double s = 0.0;
    for (int q = 0; q < JG; ++q) s += red[q * nb + tid];
    A.Dpart[(cell * g.nslot + slot) * nb + tid] = s;
  }
}

// Pipelined unstructured sweep: one CTA per (chunk of Q consecutive cells,
// octant slot) walking its cells in order; thread (jg, q) owns the channel
// pair (2q, 2q+1) of directions j = jg + r*JG (16-B loads and stores).
//  - stage i (S-deep ring, cp.async.bulk issued S cells ahead by one thread):
//    the cell's own (cell, slot) block (the DRAM stream), its I0c and beta
//    rows, its face rows A_f n_f / V_c and neighbour indices;
//  - per-direction face lists of cell i+2 (the last nj threads): a_f = dt
//    s_j.(A_f n_f / V_c), the outflow sum aout = sum_{a_f > 0} a_f and KF-1
//    inflow slots (coefficient, source block offset; unused slots have a = 0);
//    a cell with a wall face or a direction with KF inflow faces is flagged
//    for the generic path;
//  - the inflow neighbour values of cell i+1 are staged in shared memory by
//    per-thread cp.async while cell i computes (L2: adjacent cells are read by
//    this or a concurrently running CTA);
//  - interior cells: I' = I + dt beta (I0c - I) - v (aout I + sum_slots a I_up),
//    branch-free (the face sum of Eq. 3 regrouped, outflow faces first);
//  - octant partials: per-thread, then 8 contiguous group ranges ascending,
//    then the fixed tree ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)); cell i's
//    partial is finalised after the next barrier.
constexpr int kUW = 10;  // face-list words per direction: aout, nin, ain[4], src[4]

// NBT/NJT > 0 fix the channel and direction counts at compile time (with JPT = 1).
// DB = 1 (default on triangles): one neighbour-value buffer (cell i+1's
// gather is issued after cell i's barrier) and the face lists prepared from
// the global geometry rows instead of the stage, so a 2-deep ring suffices and
// two CTAs (~105 KB each) fit an SM -- each hides the other's per-cell barrier
// (u2: 2.53 -> 2.11 ms, 0.45 -> 0.53 of HBM).  Tetrahedra / quadrilaterals
// (three inflow slots) do not fit twice and keep DB = 2.
template <int JPT, int KF, int NBT, int NJT, int DB = 2>
__global__ void __launch_bounds__(1024, 1) k_usweep_tma(const USweepArgs A) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const Geometry &g = A.g;
  const UMeshDev &u = A.u;
  constexpr bool FIX = NBT > 0 && NJT > 0 && NJT % JPT == 0;
  const int nb = FIX ? NBT : g.nb, nj = FIX ? NJT : g.nj;
  const int E = FIX ? NBT * NJT : g.E, Es = FIX ? (NBT * NJT + ((NBT * NJT) & 1)) : g.Es;
  const int NBP = nb >> 1;
  // face-list words per direction (aout, nin, ain[], src[]); staged inflow
  // slots (hexahedra: 3 -- a direction crossing more inflow faces takes the
  // generic path); device face-row width
  constexpr int KUW = KF > 4 ? 2 + 2 * KF : kUW, SRC = KF > 4 ? 2 + KF : 6;
  constexpr int NIN = KF > 4 ? 3 : KF - 1, KP = KF > 4 ? 8 : 4;
  const int S = A.stages, Q = A.chunk;  // S is a power of two
  const int Sm = S - 1, Sl = __ffs(S) - 1;
  const int tid = threadIdx.x;
  const int nt = FIX ? ((NJT / JPT) * (NBT / 2) > 9 * NBT ? (NJT / JPT) * (NBT / 2) : 9 * NBT) : (int)blockDim.x;
  const int q = tid % NBP;
  const int jg = tid / NBP;
  const int JG = FIX ? NJT / JPT : A.jg;
  const bool active = jg < JG;
  // stage layout (doubles): own[Es] | I0[nb] | beta[nb] | an[12] | nbr[4] (int64)
  const int o_i0 = Es, o_be = Es + nb, o_an = Es + 2 * nb, o_nb = o_an + 3 * KP;
  const int sd = DB == 2 ? o_nb + KP : o_an;  // DB = 1: the face rows are read from global
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);        // [S]
  int *slow = reinterpret_cast<int *>(smraw + 64);            // [4] cell needs the generic path
  double *stg = reinterpret_cast<double *>(smraw + 128);      // [S][sd]
  double *red = stg + (size_t)S * sd;                         // [2][JG][nb]
  double *red2 = red + 2 * JG * nb;                           // [2][8][nb]
  // [nj][4] s_x, s_y, s_z, w per direction (DB = 1: straight from global, L1)
  const double *sws = DB == 2 ? red2 + 2 * 8 * nb : u.sw + (int64_t)blockIdx.y * nj * 4;
  double *fl = red2 + 2 * 8 * nb + (DB == 2 ? 4 * nj : 0);  // [FLR][nj][KUW]
  constexpr int FLR = DB == 2 ? 4 : 3;  // face-list ring: cells i (compute), i+1 (gather), i+2 (prep)
  // inflow neighbour values: [2 cells][KF-1 slots][JPT][nt] (16 B each)
  double2 *nbuf = reinterpret_cast<double2 *>(fl + ((FLR * nj * KUW + 1) & ~1));
  const int slot = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * Q;
  const int n = (int)min((int64_t)Q, u.ncells - c0);
  const double *__restrict__ Is = A.Iin + g.slot_off[slot];
  double *__restrict__ Os = A.Iout + g.slot_off[slot];

  auto issue = [&](int i) {
    const int st = i & Sm;
    const int64_t cell = c0 + i;
    double *sp = stg + (size_t)st * sd;
    mbar_expect_tx(&full[st], (uint32_t)(E + 2 * nb + (DB == 2 ? 4 * KP : 0)) * 8u);
    bulk_g2s(sp, Is + cell * Es, (uint32_t)E * 8u, &full[st]);
    bulk_g2s(sp + o_i0, A.I0c + cell * nb, (uint32_t)nb * 8u, &full[st]);
    bulk_g2s(sp + o_be, A.beta + cell * nb, (uint32_t)nb * 8u, &full[st]);
    if (DB == 2) {
      bulk_g2s(sp + o_an, u.an + cell * 3 * KP, 24u * KP, &full[st]);
      bulk_g2s(sp + o_nb, u.nbr + cell * KP, 8u * KP, &full[st]);
    }
  };
  // face lists of cell i (the last nj threads: the reducers and the issuing
  // thread sit in other warps, so no warp carries two extra jobs), from its stage
  const int pj = tid - (nt - nj);
  const int tis = 9 * nb < nt - nj ? 9 * nb : 0;  // the issuing thread
  auto prep = [&](int i) {
    if (i >= n || pj < 0) return;
    const int st = i & Sm;
    const double *sp = stg + (size_t)st * sd;
    if (DB == 2) mbar_wait(&full[st], (uint32_t)((i >> Sl) & 1));
    const int64_t *rn = DB == 2 ? reinterpret_cast<const int64_t *>(sp + o_nb) : u.nbr + (c0 + i) * KP;
    const double *sv = sws + 4 * pj;
    double *w = fl + ((size_t)(i % FLR) * nj + pj) * KUW;
    int64_t *wi = reinterpret_cast<int64_t *>(w);
    double aout = 0.0;
    int nin = 0;
    bool generic = false;
#pragma unroll
    for (int f = 0; f < KF; ++f) {
      const double *an = DB == 2 ? sp + o_an + 3 * f : u.an + (c0 + i) * 3 * KP + 3 * f;
      const double a = A.dt * fma(sv[2], an[2], fma(sv[1], an[1], sv[0] * an[0]));
      if (rn[f] < 0) generic = true;
      if (a > 0.0) {
        aout += a;
      } else {
        w[2 + nin] = a;
        wi[SRC + nin] = rn[f] >= 0 ? rn[f] * Es : rn[f];  // source block offset, or the wall code (< 0)
        ++nin;
      }
    }
    if (nin > NIN) generic = true;
    for (int f = nin; f < KF; ++f) {
      w[2 + f] = 0.0;
      wi[SRC + f] = -1;
    }
    w[0] = aout;
    wi[1] = nin;
    if (generic) slow[i & 3] = 1;  // every writer stores the same value
  };

  if (DB == 2)
    for (int t = tid; t < 4 * nj; t += nt) const_cast<double *>(sws)[t] = u.sw[(int64_t)slot * nj * 4 + t];
  for (int t = tid; t < DB * NIN * JPT * nt; t += nt) nbuf[t] = make_double2(0.0, 0.0);
  if (tid < 4) slow[tid] = 0;
  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == tis)
    for (int i = 0; i < min(S, n); ++i) issue(i);
  prep(0);
  prep(1);
  __syncthreads();

  const double2 v2 = make_double2(A.v[2 * q], A.v[2 * q + 1]);
  const int e0 = jg * nb + 2 * q;  // this thread's element offset for r = 0; + r*JG*nb
  // stage the inflow values of cell i (slot f of direction r at nbuf[((i&1)(KF-1) + f) JPT + r][tid])
  auto prefetch = [&](int i) {
    if (active && i < n) {
      const double *w = fl + ((size_t)(i % FLR) * nj + jg) * KUW;
#pragma unroll
      for (int r = 0; r < JPT; ++r) {
        if (jg + r * JG < nj) {
          const int64_t *wi = reinterpret_cast<const int64_t *>(w + (size_t)r * JG * KUW);
#pragma unroll
          for (int f = 0; f < NIN; ++f) {
            const int64_t src = wi[SRC + f];
            if (src >= 0) {
              const uint32_t dst = smem_u32(nbuf + ((size_t)((((DB == 2 ? i : 0) & 1) * NIN + f) * JPT + r)) * nt + tid);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                           "l"(Is + src + e0 + r * JG * nb)
                           : "memory");
            }
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch(0);

  for (int i = 0; i < n; ++i) {
    const int64_t cell = c0 + i;
    const int st = i & Sm;
    if (DB == 2) prefetch(i + 1);
    double2 acc = make_double2(0.0, 0.0);
    if (DB == 2)
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // cell i's values (cell i+1's may pend)
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    mbar_wait(&full[st], (uint32_t)((i >> Sl) & 1));
    if (active) {
      const double *sp = stg + (size_t)st * sd;
      const double2 I0 = reinterpret_cast<const double2 *>(sp + o_i0)[q];
      const double2 be = reinterpret_cast<const double2 *>(sp + o_be)[q];
      const double dtb0 = A.dt * be.x, dtb1 = A.dt * be.y;
      const int64_t base = cell * Es;
      const bool generic = slow[i & 3] != 0;  // CTA-uniform
      const double2 *nb2 = nbuf + (size_t)(((DB == 2 ? i : 0) & 1) * NIN * JPT) * nt + tid;
#pragma unroll
      for (int r = 0; r < JPT; ++r) {
        const int j = jg + r * JG;
        if (j < nj) {
          const double *w = fl + ((size_t)(i % FLR) * nj + j) * KUW;
          const int e = e0 + r * JG * nb;
          const double2 Ic = *reinterpret_cast<const double2 *>(sp + e);
          double f0 = w[0] * Ic.x, f1 = w[0] * Ic.y;
          if (!generic) {
#pragma unroll
            for (int f = 0; f < NIN; ++f) {  // unused slots: a = 0 times a finite stale value
              const double a = w[2 + f];
              const double2 up = nb2[(size_t)(f * JPT + r) * nt];
              f0 = fma(a, up.x, f0);
              f1 = fma(a, up.y, f1);
            }
          } else {
            const int64_t *wi = reinterpret_cast<const int64_t *>(w);
            const int nin = (int)wi[1];
            for (int f = 0; f < nin; ++f) {
              const double a = w[2 + f];
              const int64_t src = wi[SRC + f];
              double2 up;
              if (src >= 0 && f < NIN) {
                up = nb2[(size_t)(f * JPT + r) * nt];
              } else if (src >= 0) {
                up = __ldg(reinterpret_cast<const double2 *>(Is + src + e));
              } else {
                const int64_t code = -1 - src;
                up.x = ghost_value(g, A.Iin, (int)(code & 7), code >> 3, base, slot, j, 2 * q);
                up.y = ghost_value(g, A.Iin, (int)(code & 7), code >> 3, base, slot, j, 2 * q + 1);
              }
              f0 = fma(a, up.x, f0);
              f1 = fma(a, up.y, f1);
            }
          }
          double2 In;
          In.x = fma(dtb0, I0.x - Ic.x, Ic.x) - v2.x * f0;
          In.y = fma(dtb1, I0.y - Ic.y, Ic.y) - v2.y * f1;
          __stcs(reinterpret_cast<double2 *>(Os + base + e), In);
          const double wj = sws[4 * j + 3];
          acc.x = fma(wj, I0.x - In.x, acc.x);
          acc.y = fma(wj, I0.y - In.y, acc.y);
        }
      }
      reinterpret_cast<double2 *>(red + (size_t)(i & 1) * JG * nb + jg * nb)[q] = acc;
    }
    // flag of ring entry (i+3)&3: last read at iteration i-1, next written by
    // prep(i+3) in iteration i+1 (after this iteration's barrier)
    // DB = 1: each thread's neighbour-buffer slots are its own (written and read
    // only by it), so cell i+1's gather goes out as soon as this thread's
    // compute of cell i has consumed them -- before the barrier
    if (DB == 1) prefetch(i + 1);
    if (tid == 0) slow[(i + 3) & 3] = 0;
    prep(i + 2);
    __syncthreads();  // stage st consumed, red[i&1] complete, face lists of i+2 written
    if (tid == tis && i + S < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S);
    }
    // octant partials: 8 contiguous group ranges of cell i; finalise cell i-1
    if (tid < 8 * nb) {
      const int b = tid % nb, p = tid / nb;
      const int ga = (p * JG) >> 3, gb = ((p + 1) * JG) >> 3;
      const double *rb = red + (size_t)(i & 1) * JG * nb;
      double sum = 0.0;
      for (int gq = ga; gq < gb; ++gq) sum += rb[gq * nb + b];
      red2[((i & 1) * 8 + p) * nb + b] = sum;
    }
    if (i > 0 && tid >= 8 * nb && tid < 9 * nb) {
      const int b = tid - 8 * nb;
      const double *r2 = red2 + ((i - 1) & 1) * 8 * nb + b;
      A.Dpart[((cell - 1) * g.nslot + slot) * nb + b] =
          ((r2[0] + r2[nb]) + (r2[2 * nb] + r2[3 * nb])) + ((r2[4 * nb] + r2[5 * nb]) + (r2[6 * nb] + r2[7 * nb]));
    }
  }
  __syncthreads();
  if (n > 0 && tid < nb) {
    const double *r2 = red2 + ((n - 1) & 1) * 8 * nb + tid;
    A.Dpart[((c0 + n - 1) * g.nslot + slot) * nb + tid] =
        ((r2[0] + r2[nb]) + (r2[2 * nb] + r2[3 * nb])) + ((r2[4 * nb] + r2[5 * nb]) + (r2[6 * nb] + r2[7 * nb]));
  }
}

cudaError_t launch_usweep(const USweepArgs &a0, cudaStream_t s) {
  USweepArgs a = a0;
  const Geometry &g = a.g;
  if (a.u.ncells == 0) return cudaSuccess;
  if (a.pipelined && (a.u.K <= 4 || a.u.K == 6) && g.nb % 2 == 0 && 8 * g.nb <= 1024) {
    const int NBP = g.nb / 2;
    // 2 directions x 2 channels per thread on triangles (measured 3 % faster on u2),
    // 1 x 2 on tetrahedra (their 4-face lists fill the registers)
    // (tetrahedra / quadrilaterals also at 500 threads when the single-buffer two-CTA shape applies)
    const int tgt = a.target_threads > 0 ? a.target_threads
                                         : (a.u.K == 3 || (a.u.K == 4 && a.single_buf && g.nb == 40 && g.nj == 50 && !a.generic) ? 500 : 1024);
    int JG = std::max(1, std::min(g.nj, tgt / NBP));
    const int jpt = (g.nj + JG - 1) / JG;
    JG = (g.nj + jpt - 1) / jpt;
    const int threads = std::max(JG * NBP, 9 * g.nb);
    if (jpt <= 2 && threads <= 1024 && JG >= 8) {
      a.jpt = jpt;
      a.jg = JG;
      a.chunk = a.chunk > 0 ? a.chunk : 64;
      // red, red2, sws, face lists (+ alignment), then the cp.async neighbour buffers
      const int K = a.u.K, KUW = K > 4 ? 2 + 2 * K : kUW, NIN = K > 4 ? 3 : K - 1, KP = K > 4 ? 8 : 4;
      // triangles: one neighbour buffer, face lists from global, 2-deep ring, 2 CTAs/SM
      const int DBN = (a.single_buf && (K == 3 || K == 4) && jpt == 2 && g.nb == 40 && g.nj == 50 && !a.generic) ? 1 : 2;
      const size_t fixed = 128 + (2 * (size_t)JG * g.nb + 16 * (size_t)g.nb + (DBN == 2 ? 4 * (size_t)g.nj : 0) +
                                  (DBN == 2 ? 4 : 3) * (size_t)g.nj * KUW + 2) * sizeof(double) +
                           (size_t)DBN * NIN * jpt * threads * 16;
      const size_t sd = (size_t)g.Es + 2 * g.nb + (DBN == 2 ? 4 * KP : 0);
      int S = a.stages > 0 ? a.stages : (int)(((size_t)(DBN == 2 ? 226 : 113) * 1024 - fixed) / (sd * 8));
      // S >= 4: the face lists of cell i+2 are prepared (waiting on its stage)
      // before the barrier after which cell i+S is issued (DB = 1 reads them from global)
      S = std::max(DBN == 2 ? 4 : 2, std::min(8, S));
      while (S & (S - 1)) --S;  // power of two (stage index and phase by mask/shift)
      a.stages = S;
      const size_t smem = fixed + (size_t)S * sd * 8;
      if (smem <= 227 * 1024) {
        dim3 grid((unsigned)((a.u.ncells + a.chunk - 1) / a.chunk), g.nslot);
#define BTE_UTMA_(N, KK, B, J)                                                                          \
  {                                                                                                     \
    if (cudaError_t e = smem_attr((const void *)k_usweep_tma<N, KK, B, J>, smem)) return e;              \
    k_usweep_tma<N, KK, B, J><<<grid, threads, smem, s>>>(a);                                           \
    return cudaGetLastError();                                                                          \
  }
#define BTE_UTMA(N, KK) \
  if (jpt == N && a.u.K == KK) BTE_UTMA_(N, KK, 0, 0)
        if (g.nb == 40 && g.nj == 50 && !a.generic) {
          if (jpt == 1 && JG == 50 && threads == 1000) {
            if (a.u.K == 3) BTE_UTMA_(1, 3, 40, 50)
            if (a.u.K == 4) BTE_UTMA_(1, 4, 40, 50)
            if (a.u.K == 6) BTE_UTMA_(1, 6, 40, 50)
          }
          if (jpt == 2 && JG == 25 && threads == 500) {
            if (a.u.K == 3 && DBN == 1) {
              if (cudaError_t e = smem_attr((const void *)k_usweep_tma<2, 3, 40, 50, 1>, smem)) return e;
              k_usweep_tma<2, 3, 40, 50, 1><<<grid, threads, smem, s>>>(a);
              return cudaGetLastError();
            }
            if (a.u.K == 3) BTE_UTMA_(2, 3, 40, 50)
            if (a.u.K == 4 && DBN == 1) {
              if (cudaError_t e = smem_attr((const void *)k_usweep_tma<2, 4, 40, 50, 1>, smem)) return e;
              k_usweep_tma<2, 4, 40, 50, 1><<<grid, threads, smem, s>>>(a);
              return cudaGetLastError();
            }
            if (a.u.K == 4) BTE_UTMA_(2, 4, 40, 50)
          }
        }
        BTE_UTMA(1, 3)
        BTE_UTMA(2, 3)
        BTE_UTMA(1, 4)
        BTE_UTMA(2, 4)
        BTE_UTMA(1, 6)
        BTE_UTMA(2, 6)
#undef BTE_UTMA
#undef BTE_UTMA_
      }
    }
  }
  int jpt, JG;
  sweep_shape(g.nb, g.nj, a.target_threads > 0 ? a.target_threads : 448, &jpt, &JG);
  a.jpt = jpt;
  a.jg = JG;
  const int threads = JG * g.nb;
  if (threads > 1024) return cudaErrorInvalidConfiguration;
  const int KM = a.u.K <= 4 ? 4 : 8;  // face slots (hexahedra: 6 faces in 8)
  const size_t smem = ((size_t)KM * g.nj + (size_t)threads) * sizeof(double);
  dim3 grid((unsigned)a.u.ncells, g.nslot);
  const int jcase = jpt <= 1 ? 1 : jpt <= 2 ? 2 : jpt <= 4 ? 4 : jpt <= 5 ? 5 : jpt <= 8 ? 8 : jpt <= 10 ? 10 : jpt <= 16 ? 16 : 0;
  switch (jcase) {
#define BTE_UCASE(N)                                                                          \
  case N:                                                                                     \
    if (KM == 4) {                                                                            \
      if (cudaError_t e = smem_attr((const void *)k_usweep<N, 4>, smem)) return e;            \
      k_usweep<N, 4><<<grid, threads, smem, s>>>(a);                                          \
    } else {                                                                                  \
      if (cudaError_t e = smem_attr((const void *)k_usweep<N, 8>, smem)) return e;            \
      k_usweep<N, 8><<<grid, threads, smem, s>>>(a);                                          \
    }                                                                                         \
    break;
    BTE_UCASE(1)
    BTE_UCASE(2)
    BTE_UCASE(4)
    BTE_UCASE(5)
    BTE_UCASE(8)
    BTE_UCASE(10)
    BTE_UCASE(16)
#undef BTE_UCASE
    default:
      return cudaErrorInvalidConfiguration;
  }
  return cudaGetLastError();
}

__global__ void k_udiffuse(const Geometry g, const UMeshDev u, const double *__restrict__ I, int region,
                           double *__restrict__ gtab) {
  const int64_t f = blockIdx.x;  // owned wall face f: global row rface, local cell rcell
  diffuse_face(g, I, region, u.rface[region][f], u.rcell[region][f] * g.Es, gtab);
}

cudaError_t launch_udiffuse(const Geometry &g, const UMeshDev &u, const double *I, int region, double *gtab,
                            cudaStream_t s) {
  const int64_t nf = u.rn[region];
  if (nf == 0) return cudaSuccess;
  int threads = ((g.nb + 31) / 32) * 32;
  if (threads > 256) threads = 256;
  k_udiffuse<<<(unsigned)nf, threads, 0, s>>>(g, u, I, region, gtab);
  return cudaGetLastError();
}

// random start on an unstructured mesh: the structured recipe with the
// centroid (measured from the box corner lo) in place of the cell centre
__global__ void k_random_T_u(int64_t nc, int dim, const double *__restrict__ cen, double lo0, double lo1,
                             double lo2, double L0, double L1, double L2, double p0, double p1, double p2,
                             double T_mean, double T_amp, double *__restrict__ T) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const double twopi = 6.283185307179586;
  const double fx = sin(twopi * ((cen[3 * c] - lo0) / L0 + p0));
  const double fy = sin(twopi * ((cen[3 * c + 1] - lo1) / L1 + p1));
  const double fz = dim == 3 ? sin(twopi * ((cen[3 * c + 2] - lo2) / L2 + p2)) : 1.0;
  T[c] = T_mean + T_amp * (fz * fy * fx);
}

cudaError_t launch_random_T_u(int64_t nc, int dim, const double *cen, const double *lo, const double *L,
                              const double *phase, double T_mean, double T_amp, double *T, cudaStream_t s) {
  if (nc == 0) return cudaSuccess;
  k_random_T_u<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, dim, cen, lo[0], lo[1], lo[2], L[0], L[1], L[2],
                                                            phase[0], phase[1], phase[2], T_mean, T_amp, T);
  return cudaGetLastError();
}

}  // namespace bte
