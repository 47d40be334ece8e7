// bte_api.cu -- C ABI (include/bte.h) and host runtime of the B200 BTE step:
// validation, octant grouping of the direction set, geometry/coefficient
// precompute (a0), device state, step orchestration, error latching.
// Every step of the hot path runs in kernels.cu; this file only launches.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bte.h"
#include "bte_internal.cuh"
#include "nccl_shim.h"

// NVTX phase ranges of a step (a1 boundary / a2 sweep / a3+a4 Newton / a5
// halo), mirroring the paper's intensity / temperature / communication
// breakdown.  No-ops unless a tool attaches.
static inline void nvtx_push(const char *name) { nvtxRangePushA(name); }
static inline void nvtx_pop() { nvtxRangePop(); }

using namespace bte;

namespace {

constexpr double kHbar = 1.054571817e-34;  // J s   (CODATA 2018)
constexpr double kKB = 1.380649e-23;       // J/K   (exact SI)

// 16-point Gauss-Legendre rule on [-1, 1] (nodes ascending; literal table of
// the standard rule, 17 significant digits).
const double kGL16[16][2] = {
    {-0.9894009349916499, 0.027152459411754176}, {-0.9445750230732326, 0.062253523938647456},
    {-0.8656312023878318, 0.0951585116824926},   {-0.755404408355003, 0.12462897125553407},
    {-0.6178762444026438, 0.1495959888165767},   {-0.45801677765722737, 0.16915651939500265},
    {-0.2816035507792589, 0.18260341504492364},  {-0.09501250983763744, 0.18945061045506864},
    {0.09501250983763744, 0.18945061045506864},  {0.2816035507792589, 0.18260341504492364},
    {0.45801677765722737, 0.16915651939500265},  {0.6178762444026438, 0.1495959888165767},
    {0.755404408355003, 0.12462897125553407},    {0.8656312023878318, 0.0951585116824926},
    {0.9445750230732326, 0.062253523938647456},  {0.9894009349916499, 0.027152459411754176}};

}  // namespace

struct UPeer {                  // one neighbour rank of a partitioned unstructured mesh
  int peer = 0;
  int64_t recv_off = 0, recv_cnt = 0;  // its cells in my halo: halo positions [off, off + cnt)
  std::vector<int64_t> send_cells;     // my cells (local indices) in its halo, in its halo order
};

struct bte_ctx {
  std::string err;
  // configuration
  bte_mesh mesh;
  int nd = 0, nb = 0;
  double dt = 0, T_init = 0, W = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, nranks = 1;
  // band partition (bte_create_band): this context sweeps channels [b0, b0+nb)
  // of nbT; slab_ranks = nranks for slab contexts, 1 for band contexts
  int band = 0, b0 = 0, nbT = 0, slab_ranks = 1;
  double *Sall = nullptr;  // [nranks][ncells] gathered partials (band)
  // the sweep's I0c / beta rows [cell][nb]: aliases of I0c / beta, or (band)
  // copies of this part's channel slice kept by the Newton
  double *I0s = nullptr, *betas = nullptr;
  void *(*alloc)(size_t, void *) = nullptr;
  void (*dealloc)(void *, void *) = nullptr;
  void *alloc_ctx = nullptr;
  std::vector<void *> allocs;
  int64_t bytes = 0;
  // host copies of tables
  std::vector<double> s, w, v, bcoef;
  int mode = 0;
  std::vector<int> dmap, canon_d;  // d -> slot*nj+j ; slot*nj+j -> d
  bool refl_closed[3] = {false, false, false};
  double Tmax = 0;
  // device
  Geometry g{};
  Material m{};   // the channels this context sweeps (a view into mF for band contexts)
  Material mF{};  // all channels (Newton, refresh)
  double *I[2] = {nullptr, nullptr};
  int cur = 0;
  // octant-slot rotation: one buffer of nslot + 1 slot regions;
  // I[0] == I[1]; g.slot_off maps each slot to its region, `spare` is free
  int rot = 0, spare = 0;
  double *gspec[6] = {nullptr};
  double *I0c = nullptr, *dI0c = nullptr, *beta = nullptr, *T = nullptr, *Dpart = nullptr;
  double *gtab[6] = {nullptr};
  int *d_dmap = nullptr, *d_canon_d = nullptr;
  unsigned long long *d_err = nullptr;
  int newton_predict = 1;  // env BTE_NEWTON_PREDICT=0 disables (reading R-f)
  int newton_minb = 0;     // env BTE_NEWTON_MINB (k_newton occupancy variant)
  unsigned long long *d_stats = nullptr;  // env BTE_NEWTON_STATS=1: Newton counters printed by bte_step
  int no_spare = 0;        // env BTE_SPARE=0: side jobs on compute threads (A/B)
  int newton_lpc = -1;      // env BTE_NEWTON_LPC=0/1 forces the band-integral lane mapping (-1: by channel count)
  int pf = 1;              // env BTE_PF: k_sweep L2 prefetch distance in cells (demo sweep 0.093 -> 0.086 ms)
  int raster = 0;          // 3-D sweep column order (SweepArgs.raster); env BTE_RASTER
  int sc_direct = 0;       // env BTE_SC_DIRECT=1: direct band integrals in the self-consistent Newton (A/B)
  int ugeneric = 0;        // env BTE_UGENERIC=1: generic unstructured sweep (A/B)
  int usingle = 1;         // env BTE_USINGLE=0: two neighbour buffers, 1 CTA/SM on triangles too (A/B)
  int dbg_skip_exchange = 0;  // bte_set_debug(BTE_DEBUG_SKIP_EXCHANGE): mutation tests only
  double *d_energy = nullptr; // bte_get_energy scratch
  // CUDA-graph replay of explicit steps (SURVEY 8(b) "graph replay"): one
  // captured step per buffer parity, rebuilt when a setter changes the step
  int use_graph = 1;           // env BTE_GRAPH=0 disables (A/B)
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t graph_launches = 0;  // kernels in one captured step
  bool graph_capture = false;  // step_launch is being captured (Newton reads the device step index)
  cudaStream_t cap_stream = nullptr;  // private stream the step graphs are captured on
  // rotation: the next step's boundary pass overlapped with this step's Newton
  int prefetch_bnd = 0;        // set by bte_step while more steps follow in the call
  bool bnd_ready = false;      // the side stream has run the current step's boundary pass
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_swept = nullptr, ev_side = nullptr;
  unsigned long long *d_stepctr = nullptr;
  unsigned long long h_stepctr = 0;
  double *staging = nullptr;
  int64_t staging_cells = 0;
  int seg_len = 0;
  int use_tma = 1, stages_override = 0, seg_override = 0, target_threads = 0, smem_budget_kb = 0;  // env BTE_SWEEP / BTE_STAGES / BTE_SEGS (A/B runs)
  int64_t ncells_local = 0, ncells_global = 0;
  int64_t steps_done = 0;
  // timing: (kind, first event) spans over a preallocated event pool
  bool timing = false;
  int64_t timing_max = 0, timing_used = 0;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> spans;  // kind 0 sweep, 1 newton, 2 boundary, 3 halo
  bte_timing tacc{};
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;  // boundary planes swept / halo delivered
  int overlap = 1;  // env BTE_OVERLAP=0: exchange after the whole sweep
  // unstructured mesh (bte_create_umesh): the layout sees one plane of ncells
  int tau_mode = 0;  // 0 lagged tau (reading #15), 1 self-consistent (reading R-k)
  int semi = 0;      // 1: semi-implicit step (reading R-l)
  // implicit step by source iteration (reading R-n): bte_run.step_mode 2
  int implicit = 0, imp_max_iter = 20;
  double imp_tol = 1e-10;
  int2 *d_tasks = nullptr;       // [nslot*ncross] (slot, column) in upwind-topological order
  int *d_prog = nullptr;         // [nslot][ncross] planes published this iteration
  unsigned *d_ticket = nullptr;  // task ticket
  unsigned long long *d_conv = nullptr;  // [2]: max |dT|/T, max wall-data change (double bits)
  std::vector<int64_t> imp_iters;        // iterations of each step of the last bte_step
  double *zbeta = nullptr;  // zeros [ncells][nb]: the semi-implicit sweep advects only
  int umesh = 0;
  UMeshDev u{};
  std::vector<double> uvol;  // V_c
  std::vector<double> uKd;   // per direction: max_c sum_{f: s.an > 0} s.an (dt check)
  double *d_ucen = nullptr;  // [nc][3] centroids (random start)
  int64_t urn_global[6] = {0, 0, 0, 0, 0, 0};  // wall faces per region (whole mesh)
  std::vector<UPeer> upeers;                    // partition: neighbour ranks
  int64_t unhalo = 0;
  std::vector<int64_t *> d_usend;               // per peer: device send-cell lists
  double *d_usendbuf = nullptr, *d_urecvbuf = nullptr;  // packed [peer][slot][k][Es]
  double ulo[3] = {0, 0, 0}, uL[3] = {0, 0, 0};
  // NCCL
  bte_slab_plan plan{};
  void *nccl_comm = nullptr;
  cudaStream_t comm_stream = nullptr;
};

static bte_status fail(bte_ctx *c, bte_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return st;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, BTE_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

static void *dev_alloc(bte_ctx *ctx, size_t bytes) {
  if (bytes == 0) bytes = 256;
  void *p = nullptr;
  if (ctx->alloc) {
    p = ctx->alloc(bytes, ctx->alloc_ctx);
  } else {
    if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
  }
  if (p) {
    ctx->allocs.push_back(p);
    ctx->bytes += (int64_t)bytes;
  }
  return p;
}

template <typename T>
static bte_status upload(bte_ctx *ctx, T **dst, const T *src, size_t n) {
  *dst = (T *)dev_alloc(ctx, n * sizeof(T));
  if (!*dst) return fail(ctx, BTE_ENOMEM, "device allocation of %zu bytes failed", n * sizeof(T));
  CU(cudaMemcpyAsync(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return BTE_OK;
}

static double host_beta(const bte_ctx *ctx, int b, double T) {
  const double *q = ctx->bcoef.data() + 5 * b;
  double r = q[0] + q[1] * T * T * T + q[2] * T * T * T * T;
  if (q[3] != 0.0) r += q[3] / std::sinh(q[4] / T);
  return r;
}

// positivity of the explicit update (reading #9): every coefficient of I^n in
// I^{n+1} must be >= 0 at the hottest temperature seen.
static bte_status check_dt(bte_ctx *ctx) {
  // implicit step (R-n): every iterate is a convex combination of I^n, I0 and
  // upwind values -- positive for any dt, no bound
  if (ctx->implicit) return BTE_OK;
  const int na = ctx->mesh.dim == 3 ? 3 : 2;
  const double D[3] = {ctx->mesh.dx, ctx->mesh.dy, ctx->mesh.dz};
  double worst = 1e300;
  for (int b = ctx->b0; b < ctx->b0 + ctx->nb; ++b) {  // this context's channels
    const double be = ctx->semi ? 0.0 : host_beta(ctx, b, ctx->Tmax);  // semi-implicit: advection bound only
    for (int d = 0; d < ctx->nd; ++d) {
      double k = 0;
      if (ctx->umesh)
        k = ctx->uKd[d];  // general mesh: the largest outflow factor of direction d
      else
        for (int a = 0; a < na; ++a) k += std::fabs(ctx->s[3 * d + a]) / D[a];
      worst = std::min(worst, 1.0 - ctx->dt * be - ctx->dt * ctx->v[b] * k);
    }
  }
  if (!(worst >= 0.0))
    return fail(ctx, BTE_EUNSTABLE,
                "dt = %g violates the positivity bound at T = %g K (margin %g < 0)", ctx->dt,
                ctx->Tmax, worst);
  return BTE_OK;
}

// I0c, dI0c, beta at the current T (all channels), plus the band slice the sweep reads
static bte_status refresh(bte_ctx *ctx) {
  const int64_t ncl = ctx->ncells_local;
  CU(launch_refresh(ctx->mF, ctx->T, ncl, ctx->I0c, ctx->dI0c, ctx->beta, ctx->stream));
  if (ctx->band && ncl > 0) {
    const size_t w = (size_t)ctx->nb * sizeof(double), pitch = (size_t)ctx->nbT * sizeof(double);
    CU(cudaMemcpy2DAsync(ctx->I0s, w, ctx->I0c + ctx->b0, pitch, w, (size_t)ncl, cudaMemcpyDeviceToDevice,
                         ctx->stream));
    CU(cudaMemcpy2DAsync(ctx->betas, w, ctx->beta + ctx->b0, pitch, w, (size_t)ncl, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  }
  return BTE_OK;
}

static int64_t ncl_of(const bte_ctx *ctx) { return ctx->ncells_local; }

static int64_t n_faces_global(const bte_ctx *ctx, int region) {
  if (ctx->umesh) return ctx->urn_global[region];
  const int a = region / 2;
  const bte_mesh &m = ctx->mesh;
  if (a == 0) return m.ny * m.nz;
  if (a == 1) return m.nx * m.nz;
  return m.nx * m.ny;
}

static int octant_of(const double *s) {
  return (s[0] < 0.0 ? 4 : 0) | (s[1] < 0.0 ? 2 : 0) | (s[2] < 0.0 ? 1 : 0);
}

static bte_status sync_check(bte_ctx *ctx) {
  CU(cudaStreamSynchronize(ctx->stream));
  unsigned long long key = ~0ull;
  CU(cudaMemcpy(&key, ctx->d_err, sizeof key, cudaMemcpyDeviceToHost));
  if (key != ~0ull) {
    const unsigned long long step = key >> 40;
    const int kind = (int)((key >> 36) & 0xF);
    const unsigned long long cell = key & ((1ull << 36) - 1);
    const unsigned long long reset = ~0ull;
    CU(cudaMemcpy(ctx->d_err, &reset, sizeof reset, cudaMemcpyHostToDevice));
    if (kind == ERR_NEWTON)
      return fail(ctx, BTE_ENEWTON, "temperature Newton did not converge in %d iterations at step %llu, cell %llu",
                  kNewtonMaxIt, step, cell);
    return fail(ctx, BTE_ENONFINITE, "non-finite value in the temperature update at step %llu, cell %llu",
                step, cell);
  }
  return BTE_OK;
}

extern "C" {

static void graph_invalidate(bte_ctx *ctx);

static bte_status halo_exchange(bte_ctx *ctx, double *Ibuf, cudaStream_t stream = nullptr);
static bte_status uhalo_exchange(bte_ctx *ctx, double *Ibuf, cudaStream_t stream);

const char *bte_version(void) { return "bte-b200 0.1 (sm_100a, fp64)"; }

const char *bte_last_error(const bte_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

bte_status bte_plan_slab(const bte_mesh *mesh, const bte_dirs *dirs, int nb, int nranks, int rank,
                         bte_slab_plan *out) {
  if (!mesh || !dirs || !out || nranks < 1 || rank < 0 || rank >= nranks || nb < 1) return BTE_EINVAL;
  if (mesh->dim != 2 && mesh->dim != 3) return BTE_EINVAL;
  std::memset(out, 0, sizeof *out);
  const int axis = mesh->dim == 3 ? 2 : 1;
  const int64_t nplanes = axis == 2 ? mesh->nz : mesh->ny;
  const int64_t base = nplanes / nranks, rem = nplanes % nranks;
  out->axis = axis;
  out->n_local = base + (rank < rem ? 1 : 0);
  out->m0 = (int64_t)rank * base + std::min<int64_t>(rank, rem);
  if (out->n_local < 1) return BTE_EINVAL;
  int count[8] = {0};
  for (int d = 0; d < dirs->nd; ++d) count[octant_of(dirs->s + 3 * d)]++;
  const int bit = axis == 2 ? 1 : 2;
  const int64_t cross = axis == 2 ? mesh->nx * mesh->ny : mesh->nx;
  int slot = 0, n = 0;
  for (int o = 0; o < 8; ++o) {
    if (!count[o]) continue;
    const int64_t Eo = (int64_t)count[o] * nb;
    const int64_t cnt = cross * (Eo + (Eo & 1));  // device plane incl. the even-stride pad
    const bool down = o & bit;  // slab-axis component < 0: upwind side is above
    const int to = down ? rank - 1 : rank + 1, from = down ? rank + 1 : rank - 1;
    if (to >= 0 && to < nranks) {
      if (n >= BTE_MAX_MSGS) return BTE_EINVAL;
      out->msg[n++] = bte_msg{1, to, o, slot, down ? out->m0 : out->m0 + out->n_local - 1, cnt};
    }
    if (from >= 0 && from < nranks) {
      if (n >= BTE_MAX_MSGS) return BTE_EINVAL;
      out->msg[n++] = bte_msg{0, from, o, slot, down ? out->m0 + out->n_local : out->m0 - 1, cnt};
    }
    ++slot;
  }
  out->n_msgs = n;
  return BTE_OK;
}

bte_status bte_plan_band(int nb, int nparts, int part, int *b0, int *b1) {
  if (!b0 || !b1 || nparts < 1 || nparts > nb || part < 0 || part >= nparts) return BTE_EINVAL;
  *b0 = (int)((int64_t)part * nb / nparts);
  *b1 = (int)((int64_t)(part + 1) * nb / nparts);
  return BTE_OK;
}

struct UHost;
static bte_status create_impl(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                              const bte_run *run, bool band, bte_ctx **out, const UHost *uh = nullptr);

// ---- unstructured simplex meshes: host geometry precompute (a0)
struct UHost {
  int dim = 0, K = 0;
  int64_t nc = 0;             // cells held (owned), local numbering
  int64_t nc_global = 0, c0 = 0, nhalo = 0;
  std::vector<int64_t> nbr;   // [nc][K]: local neighbour (owned or n_own + halo position) or wall code
  std::vector<double> an;     // [nc][K][3] A_f n_f / V_c
  std::vector<double> vol;    // [nc]
  std::vector<double> cen;    // [nc][3]
  std::vector<int64_t> rcell[6];  // owned wall faces: local cell
  std::vector<int64_t> rface[6];  // ... and global face index
  int64_t rn_global[6] = {0, 0, 0, 0, 0, 0};
  std::vector<UPeer> peers;
  std::vector<int64_t> halo;  // canonical index of each halo copy
  double lo[3], L[3];
};

// Partition of an unstructured mesh over P ranks (SURVEY 8(f) f3 "graph
// partitioning"): rank r owns the contiguous canonical range
// [r*nc/P, (r+1)*nc/P) -- the generators and locality-ordered inputs make that a
// spatially compact part -- plus read-only halo copies of the face neighbours
// of its cells owned elsewhere, numbered after its own cells grouped by owner
// rank (canonical order inside a group).  Every rank derives the same plan
// from the global mesh.
static void partition_uhost(const UHost &G, int P, int rank, UHost *L) {
  const int K = G.K;
  const int64_t nc = G.nc;
  std::vector<int64_t> cut(P + 1);
  for (int r = 0; r <= P; ++r) cut[r] = (int64_t)r * nc / P;
  auto owner = [&](int64_t c) { return (int)(std::upper_bound(cut.begin(), cut.end(), c) - cut.begin()) - 1; };
  const int64_t c0 = cut[rank], c1 = cut[rank + 1];
  auto halo_of = [&](int r) {  // canonical cells outside part r adjacent to it, sorted (owner, cell)
    std::vector<int64_t> h;
    for (int64_t c = cut[r]; c < cut[r + 1]; ++c)
      for (int f = 0; f < K; ++f) {
        const int64_t e = G.nbr[c * K + f];
        if (e >= 0 && (e < cut[r] || e >= cut[r + 1])) h.push_back(e);
      }
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
    std::stable_sort(h.begin(), h.end(), [&](int64_t a, int64_t b) { return owner(a) < owner(b); });
    return h;
  };
  const std::vector<int64_t> halo = halo_of(rank);
  *L = UHost();
  L->dim = G.dim;
  L->K = K;
  L->nc = c1 - c0;
  L->nc_global = nc;
  L->c0 = c0;
  L->nhalo = (int64_t)halo.size();
  L->halo = halo;
  for (int a = 0; a < 3; ++a) {
    L->lo[a] = G.lo[a];
    L->L[a] = G.L[a];
  }
  auto local = [&](int64_t e) -> int64_t {
    if (e >= c0 && e < c1) return e - c0;
    // halo position: the halo is sorted by (owner, cell)
    auto it = std::lower_bound(halo.begin(), halo.end(), e, [&](int64_t a, int64_t b) {
      const int oa = owner(a), ob = owner(b);
      return oa != ob ? oa < ob : a < b;
    });
    return L->nc + (int64_t)(it - halo.begin());
  };
  L->nbr.resize(L->nc * K);
  L->an.assign(G.an.begin() + c0 * K * 3, G.an.begin() + c1 * K * 3);
  L->vol.assign(G.vol.begin() + c0, G.vol.begin() + c1);
  L->cen.assign(G.cen.begin() + c0 * 3, G.cen.begin() + c1 * 3);
  for (int64_t c = c0; c < c1; ++c)
    for (int f = 0; f < K; ++f) {
      const int64_t e = G.nbr[c * K + f];
      L->nbr[(c - c0) * K + f] = e >= 0 ? local(e) : e;  // wall codes keep the global face index
    }
  for (int r = 0; r < 6; ++r) {
    L->rn_global[r] = (int64_t)G.rcell[r].size();
    for (int64_t f = 0; f < (int64_t)G.rcell[r].size(); ++f) {
      const int64_t c = G.rcell[r][f];
      if (c >= c0 && c < c1) {
        L->rcell[r].push_back(c - c0);
        L->rface[r].push_back(f);
      }
    }
  }
  for (int q = 0; q < P; ++q) {
    if (q == rank) continue;
    UPeer pe;
    pe.peer = q;
    for (int64_t i = 0; i < (int64_t)halo.size(); ++i)
      if (owner(halo[i]) == q) {
        if (pe.recv_cnt == 0) pe.recv_off = i;
        ++pe.recv_cnt;
      }
    for (int64_t e : halo_of(q))
      if (e >= c0 && e < c1) pe.send_cells.push_back(e - c0);
    if (pe.recv_cnt || !pe.send_cells.empty()) L->peers.push_back(pe);
  }
}

// Eq. 3 geometry without square roots: triangle A_f n_f / V_c = 2 perp(edge) /
// |cross| (depth cancels), tetrahedron = 3 cross(b - a, c - a) / |det|, each
// oriented away from the opposite vertex.  Faces matched by their vertex sets;
// unmatched faces classified onto the box walls (region order -x,+x,-y,+y,-z,+z).
// hexahedron faces as vertex cycles (Gmsh order: bottom 0-1-2-3, top 4-5-6-7)
static const int kHexF[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};

static bool build_uhost(const bte_umesh *um, UHost *h, std::string *err) {
  const int dim = um->dim, nvc = um->nvc > 0 ? um->nvc : dim + 1;
  if (!((dim == 2 && (nvc == 3 || nvc == 4)) || (dim == 3 && (nvc == 4 || nvc == 8)))) {
    *err = "vertices per cell: dim 2 takes 3 or 4, dim 3 takes 4 (tetrahedra) or 8 (hexahedra)";
    return false;
  }
  const bool hexa = dim == 3 && nvc == 8;
  const int K = hexa ? 6 : nvc;  // faces per cell
  const int64_t nc = um->ncells, nv = um->nverts;
  h->dim = dim;
  h->K = K;
  h->nc = nc;
  h->nbr.assign(nc * K, -1);
  h->an.assign(nc * K * 3, 0.0);
  h->vol.assign(nc, 0.0);
  h->cen.assign(nc * 3, 0.0);
  double hi[3];
  for (int a = 0; a < 3; ++a) {
    h->lo[a] = INFINITY;
    hi[a] = -INFINITY;
  }
  for (int64_t i = 0; i < nv; ++i)
    for (int a = 0; a < 3; ++a) {
      h->lo[a] = std::min(h->lo[a], um->verts[3 * i + a]);
      hi[a] = std::max(hi[a], um->verts[3 * i + a]);
    }
  for (int a = 0; a < 3; ++a) h->L[a] = hi[a] - h->lo[a];
  struct FaceKey {
    int64_t v[4];
    int64_t slot;  // c*K + k
  };
  std::vector<FaceKey> keys(nc * K);
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t *cv = um->cells + c * nvc;
    const double *X[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    for (int k = 0; k < nvc; ++k) {
      if (cv[k] < 0 || cv[k] >= nv) {
        *err = "cell " + std::to_string(c) + ": vertex index out of range";
        return false;
      }
      X[k] = um->verts + 3 * cv[k];
    }
    double cen[3] = {X[0][0], X[0][1], X[0][2]};
    for (int k = 1; k < nvc; ++k)
      for (int a = 0; a < 3; ++a) cen[a] = cen[a] + X[k][a];
    for (int a = 0; a < 3; ++a) h->cen[3 * c + a] = cen[a] / nvc;
    if (hexa) {
      // bilinear faces: area vector S = (q2 - q0) x (q3 - q1) / 2 away from the
      // vertex mean, V = sum_f qbar_f . S_f / 3 (divergence theorem); A n / V = S / V
      double S[6][3], vol = 0.0;
      for (int k = 0; k < 6; ++k) {
        const double *q0 = X[kHexF[k][0]], *q1 = X[kHexF[k][1]], *q2 = X[kHexF[k][2]], *q3 = X[kHexF[k][3]];
        double d1[3], d2[3], qb[3];
        for (int a = 0; a < 3; ++a) {
          d1[a] = q2[a] - q0[a];
          d2[a] = q3[a] - q1[a];
          qb[a] = 0.25 * (q0[a] + q1[a] + q2[a] + q3[a]);
        }
        S[k][0] = 0.5 * (d1[1] * d2[2] - d1[2] * d2[1]);
        S[k][1] = 0.5 * (d1[2] * d2[0] - d1[0] * d2[2]);
        S[k][2] = 0.5 * (d1[0] * d2[1] - d1[1] * d2[0]);
        double o = 0.0;
        for (int a = 0; a < 3; ++a) o += S[k][a] * (qb[a] - h->cen[3 * c + a]);
        if (o < 0.0)
          for (int a = 0; a < 3; ++a) S[k][a] = -S[k][a];
        vol += qb[0] * S[k][0] + qb[1] * S[k][1] + qb[2] * S[k][2];
      }
      vol /= 3.0;
      if (!(vol > 0.0) || !std::isfinite(vol)) {
        *err = "cell " + std::to_string(c) + " is degenerate (zero volume)";
        return false;
      }
      h->vol[c] = vol;
      for (int k = 0; k < 6; ++k) {
        for (int a = 0; a < 3; ++a) h->an[(c * K + k) * 3 + a] = S[k][a] / vol;
        FaceKey &fk = keys[c * K + k];
        int64_t vv[4] = {cv[kHexF[k][0]], cv[kHexF[k][1]], cv[kHexF[k][2]], cv[kHexF[k][3]]};
        std::sort(vv, vv + 4);
        for (int a = 0; a < 4; ++a) fk.v[a] = vv[a];
        fk.slot = c * K + k;
      }
      continue;
    }
    double scale = 0.0;  // 2/|cross| (2/|shoelace|) or 3/|det|
    if (dim == 2 && K == 4) {  // convex quadrilateral: shoelace area
      double sh = 0.0;
      for (int k = 0; k < 4; ++k) sh += X[k][0] * X[(k + 1) & 3][1] - X[(k + 1) & 3][0] * X[k][1];
      h->vol[c] = std::fabs(sh) * 0.5 * um->depth;
      scale = 2.0 / std::fabs(sh);
    } else if (dim == 2) {
      const double cr = (X[1][0] - X[0][0]) * (X[2][1] - X[0][1]) - (X[1][1] - X[0][1]) * (X[2][0] - X[0][0]);
      h->vol[c] = std::fabs(cr) * 0.5 * um->depth;
      scale = 2.0 / std::fabs(cr);
    } else {
      double e[3][3];
      for (int r = 0; r < 3; ++r)
        for (int a = 0; a < 3; ++a) e[r][a] = X[r + 1][a] - X[0][a];
      const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                         e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                         e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
      h->vol[c] = std::fabs(det) / 6.0;
      scale = 3.0 / std::fabs(det);
    }
    if (!(h->vol[c] > 0.0) || !std::isfinite(scale)) {
      *err = "cell " + std::to_string(c) + " is degenerate (zero volume)";
      return false;
    }
    for (int k = 0; k < K; ++k) {
      int q[3], n = 0;
      if (dim == 2) {  // edge (v_{k+1}, v_{k+2})
        q[0] = (k + 1) % K;
        q[1] = (k + 2) % K;
        q[2] = q[1];
        n = 2;
      } else {
        for (int i = 0; i < K; ++i)
          if (i != k) q[n++] = i;
      }
      double An[3];
      if (dim == 2) {
        const double ex = X[q[1]][0] - X[q[0]][0], ey = X[q[1]][1] - X[q[0]][1];
        An[0] = ey;
        An[1] = -ex;
        An[2] = 0.0;
      } else {
        double u[3], w[3];
        for (int a = 0; a < 3; ++a) {
          u[a] = X[q[1]][a] - X[q[0]][a];
          w[a] = X[q[2]][a] - X[q[0]][a];
        }
        An[0] = u[1] * w[2] - u[2] * w[1];
        An[1] = u[2] * w[0] - u[0] * w[2];
        An[2] = u[0] * w[1] - u[1] * w[0];
      }
      // outward: away from the opposite vertex (simplices) or the vertex mean (quadrilaterals)
      double o = 0.0;
      for (int a = 0; a < 3; ++a) o += An[a] * ((K == 4 && dim == 2 ? h->cen[3 * c + a] : X[k][a]) - X[q[0]][a]);
      const double sg = o > 0.0 ? -scale : scale;
      for (int a = 0; a < 3; ++a) h->an[(c * K + k) * 3 + a] = sg * An[a];
      FaceKey &fk = keys[c * K + k];
      int64_t vv[3] = {cv[q[0]], cv[q[1]], dim == 3 ? cv[q[2]] : -1};
      std::sort(vv, vv + (dim == 3 ? 3 : 2));
      for (int a = 0; a < 3; ++a) fk.v[a] = vv[a];
      fk.v[3] = -1;
      fk.slot = c * K + k;
    }
  }
  std::sort(keys.begin(), keys.end(), [](const FaceKey &x, const FaceKey &y) {
    for (int a = 0; a < 4; ++a)
      if (x.v[a] != y.v[a]) return x.v[a] < y.v[a];
    return x.slot < y.slot;
  });
  for (size_t i = 0; i < keys.size();) {
    size_t j = i + 1;
    while (j < keys.size() && keys[j].v[0] == keys[i].v[0] && keys[j].v[1] == keys[i].v[1] &&
           keys[j].v[2] == keys[i].v[2] && keys[j].v[3] == keys[i].v[3])
      ++j;
    if (j - i > 2) {
      *err = "a face is shared by more than two cells";
      return false;
    }
    if (j - i == 2) {
      h->nbr[keys[i].slot] = keys[i + 1].slot / K;
      h->nbr[keys[i + 1].slot] = keys[i].slot / K;
    }
    i = j;
  }
  int64_t count[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t c = 0; c < nc; ++c)
    for (int k = 0; k < K; ++k) {
      if (h->nbr[c * K + k] >= 0) continue;
      const int64_t *cv = um->cells + c * nvc;
      int reg = -1;
      for (int r = 0; r < 2 * dim && reg < 0; ++r) {
        const int a = r / 2;
        const double wall = (r & 1) ? hi[a] : h->lo[a];
        bool on = true;
        if (hexa) {
          for (int i = 0; i < 4; ++i)
            if (um->verts[3 * cv[kHexF[k][i]] + a] != wall) on = false;
        } else if (dim == 2) {
          on = um->verts[3 * cv[(k + 1) % K] + a] == wall && um->verts[3 * cv[(k + 2) % K] + a] == wall;
        } else {
          for (int i = 0; i < K; ++i)
            if (i != k && um->verts[3 * cv[i] + a] != wall) on = false;
        }
        if (on) reg = r;
      }
      if (reg < 0) {
        *err = "cell " + std::to_string(c) + " face " + std::to_string(k) + ": boundary face off the box walls";
        return false;
      }
      h->nbr[c * K + k] = -1 - (count[reg] * 8 + reg);
      h->rcell[reg].push_back(c);
      h->rface[reg].push_back(count[reg]);
      ++count[reg];
    }
  for (int r = 0; r < 6; ++r) h->rn_global[r] = count[r];
  h->nc_global = nc;
  return true;
}

bte_status bte_create_umesh(const bte_umesh *um, const bte_dirs *dirs, const bte_bands *bands, const bte_run *run,
                            bte_ctx **out) {
  if (!out) return BTE_EINVAL;
  *out = nullptr;
  auto early = [&](const char *msg) {
    bte_ctx *c = new bte_ctx();
    c->err = msg;
    *out = c;
    return BTE_EINVAL;
  };
  if (!um || !um->verts || !um->cells) return early("null unstructured mesh");
  if (um->dim != 2 && um->dim != 3) return early("unstructured dim must be 2 (triangles, quadrilaterals) or 3 (tetrahedra, hexahedra)");
  if (um->ncells < 1 || um->nverts < um->dim + 1) return early("empty unstructured mesh");
  if (um->ncells > (1ll << 30)) return early("unstructured mesh too large");
  if (um->dim == 2 && !(um->depth > 0)) return early("depth must be > 0");
  if (um->nvc != 0 && !(um->nvc == um->dim + 1 || (um->dim == 2 && um->nvc == 4) || (um->dim == 3 && um->nvc == 8)))
    return early("vertices per cell: dim 2 takes 3 or 4, dim 3 takes 4 or 8");
  if (run && (run->nranks < 1 || run->rank < 0 || run->rank >= run->nranks || run->nranks > um->ncells))
    return early("bad rank/nranks for the unstructured partition");
  UHost uh;
  std::string err;
  if (!build_uhost(um, &uh, &err)) return early(err.c_str());
  if (run && run->nranks > 1) {
    UHost part;
    partition_uhost(uh, run->nranks, run->rank, &part);
    uh = std::move(part);
  }
  // the state layout sees one plane of the owned cells (the halo copies follow
  // them inside each octant-slot region)
  bte_mesh fm{um->dim, uh.nc, 1, 1, 1.0, 1.0, 1.0};
  return create_impl(&fm, dirs, bands, run, false, out, &uh);
}

bte_status bte_set_step_mode(bte_ctx *ctx, int mode) {
  if (!ctx) return BTE_EINVAL;
  graph_invalidate(ctx);
  if (mode < 0 || mode > 2)
    return fail(ctx, BTE_EINVAL, "step mode must be 0 (explicit), 1 (semi-implicit) or 2 (implicit)");
  if (mode == 1 && ctx->band) return fail(ctx, BTE_EINVAL, "semi-implicit step: not for band contexts");
  if (mode != 0 && ctx->tau_mode == 1)
    return fail(ctx, BTE_EINVAL, "semi-implicit / implicit step: lagged tau only (bte_set_tau_mode 0)");
  if (mode == 2 && (ctx->band || ctx->umesh || ctx->nranks > 1 || ctx->rot))
    return fail(ctx, BTE_EINVAL,
                "implicit step: one structured context with two intensity buffers (no band / unstructured / "
                "multi-rank / octant-slot rotation)");
  const int old_s = ctx->semi, old_i = ctx->implicit;
  ctx->semi = mode == 1;
  ctx->implicit = mode == 2;
  bte_status st = check_dt(ctx);
  if (st) {
    ctx->semi = old_s;
    ctx->implicit = old_i;
  }
  return st;
}

bte_status bte_set_implicit(bte_ctx *ctx, int max_iter, double tol) {
  if (!ctx) return BTE_EINVAL;
  if (max_iter < 1 || max_iter > 100000 || !(tol >= 0.0) || !std::isfinite(tol))
    return fail(ctx, BTE_EINVAL, "implicit iterations: max_iter in [1, 100000], tol >= 0");
  ctx->imp_max_iter = max_iter;
  ctx->imp_tol = tol;
  return BTE_OK;
}

bte_status bte_get_iterations(const bte_ctx *ctx, int64_t *out, int64_t n, int64_t *count) {
  if (!ctx || !count || n < 0 || (n > 0 && !out)) return BTE_EINVAL;
  *count = (int64_t)ctx->imp_iters.size();
  for (int64_t k = 0; k < std::min<int64_t>(n, *count); ++k) out[k] = ctx->imp_iters[k];
  return BTE_OK;
}

bte_status bte_set_tau_mode(bte_ctx *ctx, int mode) {
  if (!ctx) return BTE_EINVAL;
  graph_invalidate(ctx);
  if (mode != 0 && mode != 1) return fail(ctx, BTE_EINVAL, "tau mode must be 0 (lagged) or 1 (self-consistent)");
  if (mode == 1 && (ctx->semi || ctx->implicit)) return fail(ctx, BTE_EINVAL, "self-consistent tau: explicit step only");
  if (mode == 1 && ctx->band)
    return fail(ctx, BTE_EINVAL, "self-consistent tau needs every channel's reduction in the Newton (not band contexts)");
  ctx->tau_mode = mode;
  if (mode == 1) {  // I0c, dI0c, beta at the current T (the next sweep's beta is beta(T^n))
    bte_status st = refresh(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return BTE_OK;
}

bte_status bte_plan_umesh(const bte_umesh *um, int nranks, int rank, bte_umesh_plan *out, int64_t *halo_cells,
                          int64_t halo_cap, int64_t *send_cells, int64_t send_cap) {
  if (!um || !out || !um->verts || !um->cells || nranks < 1 || rank < 0 || rank >= nranks || nranks > um->ncells)
    return BTE_EINVAL;
  if (um->dim != 2 && um->dim != 3) return BTE_EINVAL;
  UHost G, L;
  std::string err;
  if (!build_uhost(um, &G, &err)) return BTE_EINVAL;
  partition_uhost(G, nranks, rank, &L);
  std::memset(out, 0, sizeof *out);
  out->cell0 = L.c0;
  out->n_own = L.nc;
  out->n_halo = L.nhalo;
  if ((int)L.peers.size() > BTE_MAX_MSGS) return BTE_EINVAL;
  out->n_peers = (int)L.peers.size();
  int64_t off = 0;
  for (int k = 0; k < out->n_peers; ++k) {
    const UPeer &pe = L.peers[k];
    out->peer[k] = bte_upeer{pe.peer, pe.recv_off, pe.recv_cnt, off, (int64_t)pe.send_cells.size()};
    if (send_cells) {
      if (off + (int64_t)pe.send_cells.size() > send_cap) return BTE_EINVAL;
      std::copy(pe.send_cells.begin(), pe.send_cells.end(), send_cells + off);
    }
    off += (int64_t)pe.send_cells.size();
  }
  if (halo_cells) {
    if ((int64_t)L.halo.size() > halo_cap) return BTE_EINVAL;
    std::copy(L.halo.begin(), L.halo.end(), halo_cells);
  }
  return BTE_OK;
}

bte_status bte_get_region_faces(const bte_ctx *ctx, int region, int64_t *nfaces) {
  if (!ctx || !nfaces || region < 0 || region >= 6) return BTE_EINVAL;
  *nfaces = n_faces_global(ctx, region);
  return BTE_OK;
}

bte_status bte_create(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands, const bte_run *run,
                      bte_ctx **out) {
  return create_impl(mesh, dirs, bands, run, false, out);
}

bte_status bte_create_band(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                           const bte_run *run, bte_ctx **out) {
  return create_impl(mesh, dirs, bands, run, true, out);
}

static bte_status create_impl(const bte_mesh *mesh, const bte_dirs *dirs, const bte_bands *bands,
                              const bte_run *run, bool band, bte_ctx **out, const UHost *uh) {
  if (!out) return BTE_EINVAL;
  *out = nullptr;
  bte_ctx *ctx = new bte_ctx();
  bte_status st = BTE_OK;
  auto bail = [&](bte_status s) {
    *out = ctx;  // caller reads bte_last_error, then bte_destroy
    return s;
  };
  if (!mesh || !dirs || !bands || !run) return bail(fail(ctx, BTE_EINVAL, "null argument"));
  ctx->mesh = *mesh;
  if (mesh->dim != 2 && mesh->dim != 3) return bail(fail(ctx, BTE_EINVAL, "dim must be 2 or 3"));
  if (mesh->nx < 1 || mesh->ny < 1 || mesh->nz < 1 || (mesh->dim == 2 && mesh->nz != 1))
    return bail(fail(ctx, BTE_EINVAL, "bad mesh extents (dim 2 needs nz == 1)"));
  if (!(mesh->dx > 0 && mesh->dy > 0 && mesh->dz > 0)) return bail(fail(ctx, BTE_EINVAL, "cell sizes must be > 0"));
  if (mesh->nx > (1 << 30) || mesh->ny > (1 << 30)) return bail(fail(ctx, BTE_EINVAL, "mesh too large"));
  // cells per plane are int32 in the kernels (column index = blockIdx.x)
  if (mesh->dim == 3 && mesh->nx * mesh->ny >= (int64_t)1 << 31)
    return bail(fail(ctx, BTE_EINVAL, "nx*ny = %lld cells per plane exceeds 2^31 - 1",
                     (long long)(mesh->nx * mesh->ny)));
  if (dirs->nd < 1 || !dirs->s || !dirs->w) return bail(fail(ctx, BTE_EINVAL, "empty direction set"));
  if (bands->nb < 1 || bands->nb > kMaxBands || !bands->v || !bands->beta_coef)
    return bail(fail(ctx, BTE_EINVAL, "channel count must be in [1, %d]", kMaxBands));
  if (!(run->dt > 0) || !(run->T_init > 0)) return bail(fail(ctx, BTE_EINVAL, "dt and T_init must be > 0"));
  if (run->nranks < 1 || run->rank < 0 || run->rank >= run->nranks)
    return bail(fail(ctx, BTE_EINVAL, "bad rank/nranks"));
  ctx->nd = dirs->nd;
  ctx->nbT = bands->nb;
  ctx->nb = bands->nb;
  ctx->band = band ? 1 : 0;
  ctx->slab_ranks = (band || uh) ? 1 : run->nranks;  // unstructured parts exchange halo cells, not planes
  if (band) {
    int b1 = 0;
    if (bte_plan_band(bands->nb, run->nranks, run->rank, &ctx->b0, &b1) != BTE_OK)
      return bail(fail(ctx, BTE_EINVAL, "band partition: need 1 <= nranks (%d) <= channels (%d)", run->nranks,
                       bands->nb));
    ctx->nb = b1 - ctx->b0;
  }
  const int nbT = ctx->nbT;
  ctx->dt = run->dt;
  ctx->T_init = run->T_init;
  ctx->Tmax = run->T_init;
  ctx->device = run->device;
  ctx->stream = (cudaStream_t)run->stream;
  ctx->rank = run->rank;
  ctx->nranks = run->nranks;
  ctx->alloc = run->alloc;
  ctx->dealloc = run->dealloc;
  ctx->alloc_ctx = run->alloc_ctx;
  ctx->s.assign(dirs->s, dirs->s + 3 * dirs->nd);
  ctx->w.assign(dirs->w, dirs->w + dirs->nd);
  ctx->v.assign(bands->v, bands->v + bands->nb);
  ctx->bcoef.assign(bands->beta_coef, bands->beta_coef + 5 * bands->nb);
  ctx->mode = bands->mode;
  for (int b = 0; b < nbT; ++b) {
    if (!(ctx->v[b] > 0)) return bail(fail(ctx, BTE_EINVAL, "group speed of channel %d must be > 0", b));
    for (int k = 0; k < 5; ++k)
      if (!(ctx->bcoef[5 * b + k] >= 0)) return bail(fail(ctx, BTE_EINVAL, "beta coefficients must be >= 0"));
    if (!(host_beta(ctx, b, run->T_init) >= 0)) return bail(fail(ctx, BTE_EINVAL, "beta must be >= 0"));
  }
  if (bands->mode == BTE_I0_LINEAR) {
    if (!bands->I_ref || !bands->slope) return bail(fail(ctx, BTE_EINVAL, "linear mode needs I_ref and slope"));
  } else if (bands->mode == BTE_I0_BOSE_EINSTEIN) {
    if (!bands->w_lo || !bands->w_hi || !bands->vs || !bands->c2 || !bands->g)
      return bail(fail(ctx, BTE_EINVAL, "Bose-Einstein mode needs w_lo, w_hi, vs, c2, g"));
  } else {
    return bail(fail(ctx, BTE_EINVAL, "unknown I0 mode"));
  }
  double W = 0;
  for (int d = 0; d < ctx->nd; ++d) {
    if (!(ctx->w[d] > 0)) return bail(fail(ctx, BTE_EINVAL, "direction weights must be > 0"));
    W += ctx->w[d];
  }
  ctx->W = W;

  // ---- octant grouping: slots = non-empty octants ascending
  int count[8] = {0};
  std::vector<int> oct(ctx->nd), jidx(ctx->nd);
  for (int d = 0; d < ctx->nd; ++d) {
    oct[d] = octant_of(&ctx->s[3 * d]);
    jidx[d] = count[oct[d]]++;
  }
  int slot_of[8];
  int nslot = 0, nj = -1;
  for (int o = 0; o < 8; ++o) {
    slot_of[o] = -1;
    if (count[o]) {
      if (nj < 0) nj = count[o];
      if (count[o] != nj)
        return bail(fail(ctx, BTE_EINVAL, "every non-empty octant must hold the same number of directions"));
      ctx->g.slot_oct[nslot] = o;
      slot_of[o] = nslot++;
    }
  }
  for (int o = 0; o < 8; ++o) ctx->g.oct_slot[o] = slot_of[o];
  ctx->dmap.resize(ctx->nd);
  ctx->canon_d.resize(ctx->nd);
  for (int d = 0; d < ctx->nd; ++d) {
    const int sj = slot_of[oct[d]] * nj + jidx[d];
    ctx->dmap[d] = sj;
    ctx->canon_d[sj] = d;
  }

  // ---- geometry / slab decomposition along the slowest axis
  Geometry &g = ctx->g;
  g.dim = mesh->dim;
  g.nx = (int)mesh->nx;
  g.ny = mesh->dim == 3 ? (int)mesh->ny : 1;
  g.ncross = mesh->dim == 3 ? (int)(mesh->nx * mesh->ny) : (int)mesh->nx;
  const int64_t nm = mesh->dim == 3 ? mesh->nz : mesh->ny;
  g.nplanes_global = nm;
  const int srank = ctx->slab_ranks > 1 ? ctx->rank : 0;
  if (bte_plan_slab(mesh, dirs, ctx->nb, ctx->slab_ranks, srank, &ctx->plan) != BTE_OK)
    return bail(fail(ctx, BTE_EINVAL, "more ranks than planes along the slab axis"));
  g.nplanes = (int)ctx->plan.n_local;
  g.m0 = ctx->plan.m0;
  g.plane_off = ctx->slab_ranks > 1 ? 1 : 0;
  g.has_lo_wall = (srank == 0) ? 1 : 0;
  g.has_hi_wall = (srank == ctx->slab_ranks - 1) ? 1 : 0;
  g.nslot = nslot;
  g.nj = nj;
  g.nb = ctx->nb;
  g.nbT = nbT;
  g.b0 = ctx->b0;
  g.E = nj * ctx->nb;
  g.Es = g.E + (g.E & 1);
  g.plane_stride = (int64_t)g.ncross * g.Es;
  g.slot_stride = (int64_t)(g.nplanes + 2 * g.plane_off) * g.plane_stride;
  if (uh) g.slot_stride = (uh->nc + uh->nhalo) * (int64_t)g.Es;  // owned blocks, then the halo copies
  ctx->ncells_local = (int64_t)g.nplanes * g.ncross;
  ctx->ncells_global = uh ? uh->nc_global : mesh->nx * mesh->ny * mesh->nz;
  g.cell0 = uh ? uh->c0 : g.m0 * g.ncross;  // canonical index of the first owned cell

  if (cudaSetDevice(ctx->device) != cudaSuccess) return bail(fail(ctx, BTE_ECUDA, "cudaSetDevice(%d) failed", ctx->device));

  // ---- per-(slot, j) tables
  const double Dl[3] = {mesh->dx, mesh->dy, mesh->dz};
  const int nsj = nslot * nj;
  std::vector<double> coef(4 * nsj), ws(3 * nsj, 0.0);
  std::vector<int64_t> roff(3 * nsj, 0);
  for (int sj = 0; sj < nsj; ++sj) {
    const int d = ctx->canon_d[sj];
    for (int a = 0; a < 3; ++a) {
      coef[4 * sj + a] = ctx->dt * std::fabs(ctx->s[3 * d + a]) / Dl[a];
      ws[a * nsj + sj] = ctx->w[d] * std::fabs(ctx->s[3 * d + a]);
    }
    coef[4 * sj + 3] = ctx->w[d];
  }
  for (int a = 0; a < 3; ++a) {
    bool closed = true;
    for (int d = 0; d < ctx->nd && closed; ++d) {
      double t[3] = {ctx->s[3 * d], ctx->s[3 * d + 1], ctx->s[3 * d + 2]};
      t[a] = -t[a];
      int hit = -1;
      for (int e = 0; e < ctx->nd; ++e)
        if (ctx->s[3 * e] == t[0] && ctx->s[3 * e + 1] == t[1] && ctx->s[3 * e + 2] == t[2] && ctx->w[e] == ctx->w[d]) {
          hit = e;
          break;
        }
      if (hit < 0) {
        closed = false;
        break;
      }
      const int sj = ctx->dmap[d], sje = ctx->dmap[hit];
      roff[a * nsj + sj] = (int64_t)(sje / nj) * g.slot_stride + (int64_t)(sje % nj) * ctx->nb;
    }
    ctx->refl_closed[a] = closed;
  }

  // ---- material tables: A_bj, X_bj (Bose-Einstein, reading #1)
  std::vector<double> A(nbT * kNGL, 0.0), X(nbT * kNGL, 0.0);
  std::vector<double> Iref(nbT, 0.0), slope(nbT, 0.0);
  if (bands->mode == BTE_I0_BOSE_EINSTEIN) {
    for (int b = 0; b < nbT; ++b) {
      const double lo = bands->w_lo[b], hi = bands->w_hi[b];
      if (!(hi > lo && lo >= 0)) return bail(fail(ctx, BTE_EINVAL, "band %d: need 0 <= w_lo < w_hi", b));
      const double half = 0.5 * (hi - lo), mid = 0.5 * (hi + lo);
      const double pref = bands->g[b] * kHbar / (8.0 * M_PI * M_PI * M_PI) * half;
      for (int j = 0; j < kNGL; ++j) {
        const double w = mid + half * kGL16[j][0];
        const double vs = bands->vs[b], c2 = bands->c2[b];
        const double disc = vs * vs + 4.0 * c2 * w;
        if (!(disc > 0)) return bail(fail(ctx, BTE_EINVAL, "band %d beyond the dispersion maximum", b));
        const double k = c2 == 0.0 ? w / vs : 2.0 * w / (vs + std::sqrt(disc));
        A[b * kNGL + j] = pref * kGL16[j][1] * w * k * k;
        X[b * kNGL + j] = kHbar * w / kKB;
      }
    }
  } else {
    for (int b = 0; b < nbT; ++b) {
      Iref[b] = bands->I_ref[b];
      slope[b] = bands->slope[b];
    }
  }

  // uniform band grid detection (exact): channel b spans [i_b dw, (i_b + 1) dw]
  std::vector<int> ichan, ibv(nbT, 0);
  std::vector<double> Ugl(kNGL);
  int uniform = 0, imax = 0;
  double Xd = 0;
  if (bands->mode == BTE_I0_BOSE_EINSTEIN) {
    const double dw = bands->w_hi[0] - bands->w_lo[0];
    uniform = dw > 0;
    std::vector<int> ib(nbT);
    for (int b = 0; b < nbT && uniform; ++b) {
      const double q = std::nearbyint(bands->w_lo[b] / dw);
      if (!(q >= 0 && q < 4096) || bands->w_lo[b] != q * dw || bands->w_hi[b] != (q + 1.0) * dw) uniform = 0;
      ib[b] = (int)q;
      ibv[b] = ib[b];
      imax = std::max(imax, ib[b]);
    }
    if (uniform) {
      ichan.assign(4 * (imax + 1), -1);
      for (int b = 0; b < nbT && uniform; ++b) {
        int q = 0;
        while (q < 4 && ichan[4 * ib[b] + q] >= 0) ++q;
        if (q == 4) uniform = 0;  // > 4 channels share one band: use the direct path
        else ichan[4 * ib[b] + q] = b;
      }
    }
    if (const char *e = getenv("BTE_I0_DIRECT")) uniform = uniform && !atoi(e);
    Xd = kHbar * dw / kKB;
    for (int j = 0; j < kNGL; ++j) Ugl[j] = 0.5 * (1.0 + kGL16[j][0]);
  }
  if (!uniform) {
    ichan.assign(4, -1);
    imax = 0;
  }

  if (uh) {
    ctx->umesh = 1;
    ctx->uvol = uh->vol;
    ctx->uKd.assign(ctx->nd, 0.0);
    for (int d = 0; d < ctx->nd; ++d) {
      const double *sd = &ctx->s[3 * d];
      double kmax = 0.0;
      for (int64_t c = 0; c < uh->nc; ++c) {
        double k = 0.0;
        for (int f = 0; f < uh->K; ++f) {
          const double *an = &uh->an[(c * uh->K + f) * 3];
          const double sa = fma(sd[2], an[2], fma(sd[1], an[1], sd[0] * an[0]));
          if (sa > 0.0) k += sa;
        }
        kmax = std::max(kmax, k);
      }
      ctx->uKd[d] = kmax;
    }
    for (int a = 0; a < 3; ++a) {
      ctx->ulo[a] = uh->lo[a];
      ctx->uL[a] = uh->L[a];
    }
    ctx->u.K = uh->K;
    ctx->u.KP = uh->K <= 4 ? 4 : 8;
    ctx->u.ncells = uh->nc;
    for (int r = 0; r < 6; ++r) {
      ctx->u.rn[r] = (int64_t)uh->rcell[r].size();
      ctx->urn_global[r] = uh->rn_global[r];
    }
    ctx->upeers = uh->peers;
    ctx->unhalo = uh->nhalo;
  }
  if (run->step_mode < 0 || run->step_mode > 2) return bail(fail(ctx, BTE_EINVAL, "step_mode must be 0, 1 or 2"));
  if (run->step_mode == 1 && band) return bail(fail(ctx, BTE_EINVAL, "semi-implicit step: not for band contexts"));
  if (run->step_mode == 2 && (band || ctx->umesh || ctx->nranks > 1))
    return bail(fail(ctx, BTE_EINVAL, "implicit step: one structured context (no band / unstructured / multi-rank)"));
  ctx->semi = run->step_mode == 1;
  ctx->implicit = run->step_mode == 2;
  if ((st = check_dt(ctx)) != BTE_OK) return bail(st);

  // ---- device allocations
  double *d_coef, *d_ws, *d_v, *d_bc, *d_A, *d_X, *d_Iref, *d_slope;
  int64_t *d_roff;
  if ((st = upload(ctx, &d_coef, coef.data(), coef.size()))) return bail(st);
  if ((st = upload(ctx, &d_ws, ws.data(), ws.size()))) return bail(st);
  if ((st = upload(ctx, &d_roff, roff.data(), roff.size()))) return bail(st);
  if ((st = upload(ctx, &d_v, ctx->v.data(), ctx->v.size()))) return bail(st);
  if ((st = upload(ctx, &d_bc, ctx->bcoef.data(), ctx->bcoef.size()))) return bail(st);
  if ((st = upload(ctx, &d_A, A.data(), A.size()))) return bail(st);
  if ((st = upload(ctx, &d_X, X.data(), X.size()))) return bail(st);
  if ((st = upload(ctx, &d_Iref, Iref.data(), Iref.size()))) return bail(st);
  if ((st = upload(ctx, &d_slope, slope.data(), slope.size()))) return bail(st);
  if ((st = upload(ctx, &ctx->d_dmap, ctx->dmap.data(), ctx->dmap.size()))) return bail(st);
  if ((st = upload(ctx, &ctx->d_canon_d, ctx->canon_d.data(), ctx->canon_d.size()))) return bail(st);
  g.coef = d_coef;
  g.ws = d_ws;
  g.refl_off = d_roff;
  ctx->m.nb = nbT;
  ctx->m.mode = bands->mode;
  ctx->m.v = d_v;
  ctx->m.bcoef = d_bc;
  ctx->m.I_ref = d_Iref;
  ctx->m.slope = d_slope;
  ctx->m.T_ref = bands->T_ref;
  ctx->m.A = d_A;
  ctx->m.X = d_X;
  {
    double *d_U;
    int *d_ichan;
    if ((st = upload(ctx, &d_U, Ugl.data(), Ugl.size()))) return bail(st);
    if ((st = upload(ctx, &d_ichan, ichan.data(), ichan.size()))) return bail(st);
    ctx->m.uniform = uniform;
    ctx->m.imax = imax;
    ctx->m.Xd = Xd;
    ctx->m.U = d_U;
    ctx->m.ichan = d_ichan;
    int maxcnt = 0;
    for (int i = 0; i <= imax; ++i) {
      int c = 0;
      while (c < 4 && ichan[4 * i + c] >= 0) ++c;
      maxcnt = std::max(maxcnt, c);
    }
    ctx->m.maxcnt = maxcnt;
    int *d_ib;
    if ((st = upload(ctx, &d_ib, ibv.data(), ibv.size()))) return bail(st);
    ctx->m.ib = d_ib;
    std::vector<double> rv(nbT);
    for (int b = 0; b < nbT; ++b) rv[b] = 1.0 / ctx->v[b];
    double *d_rv;
    if ((st = upload(ctx, &d_rv, rv.data(), rv.size()))) return bail(st);
    ctx->m.rv = d_rv;
  }
  // m: the swept channels [b0, b0+nb) as a view of the full tables mF
  ctx->mF = ctx->m;
  {
    Material &m = ctx->m;
    const int b0 = ctx->b0;
    m.nb = ctx->nb;
    m.v += b0;
    m.bcoef += 5 * b0;
    m.I_ref += b0;
    m.slope += b0;
    m.A += kNGL * b0;
    m.X += kNGL * b0;
    m.ib += b0;
    m.rv += b0;
    if (ctx->band) m.uniform = 0;  // the band-grid fields index all channels: Newton only (mF)
  }

  const size_t ibytes = (size_t)g.slot_stride * nslot * sizeof(double);
  // two full buffers, or (when they would not fit next to ~2 GB of tables and
  // workspace, or BTE_ROTATE=1) octant-slot rotation in (nslot + 1)/nslot of one
  {
    size_t freeb = 0, totalb = 0;
    CU(cudaMemGetInfo(&freeb, &totalb));
    const size_t other = (size_t)ncl_of(ctx) * (nslot * ctx->nb + 4 * nbT + 2) * sizeof(double) + (2ull << 30);
    ctx->rot = 2 * ibytes + other > freeb ? 1 : 0;
    if (const char *e = getenv("BTE_ROTATE")) ctx->rot = atoi(e) ? 1 : 0;
    if (ctx->umesh) ctx->rot = 0;  // unstructured: two buffers
    if (ctx->implicit && ctx->rot)  // every iteration re-reads I^n of all octants
      return bail(fail(ctx, BTE_ENOMEM, "implicit step needs two full intensity buffers (%zu bytes each)", ibytes));
  }
  for (int sl = 0; sl < kMaxSlots; ++sl) g.slot_off[sl] = (int64_t)sl * g.slot_stride;
  g.rot = ctx->rot;
  if (ctx->rot) {
    const size_t rbytes = (size_t)g.slot_stride * (nslot + 1) * sizeof(double);
    ctx->I[0] = ctx->I[1] = (double *)dev_alloc(ctx, rbytes);
    if (!ctx->I[0]) return bail(fail(ctx, BTE_ENOMEM, "cannot allocate the intensity buffer (%zu bytes)", rbytes));
    CU(cudaMemsetAsync(ctx->I[0], 0, rbytes, ctx->stream));
    ctx->spare = nslot;
  } else {
    for (int k = 0; k < 2; ++k) {
      ctx->I[k] = (double *)dev_alloc(ctx, ibytes);
      if (!ctx->I[k]) return bail(fail(ctx, BTE_ENOMEM, "cannot allocate the intensity buffer (%zu bytes)", ibytes));
      CU(cudaMemsetAsync(ctx->I[k], 0, ibytes, ctx->stream));
    }
  }
  const int64_t ncl = ctx->ncells_local;
  ctx->I0c = (double *)dev_alloc(ctx, ncl * nbT * sizeof(double));
  ctx->beta = (double *)dev_alloc(ctx, ncl * nbT * sizeof(double));
  ctx->dI0c = (double *)dev_alloc(ctx, ncl * nbT * sizeof(double));
  ctx->I0s = ctx->I0c;
  ctx->betas = ctx->beta;
  if (ctx->band) {
    ctx->Sall = (double *)dev_alloc(ctx, (size_t)ctx->nranks * ncl * sizeof(double));
    ctx->I0s = (double *)dev_alloc(ctx, ncl * ctx->nb * sizeof(double));
    ctx->betas = (double *)dev_alloc(ctx, ncl * ctx->nb * sizeof(double));
    if (!ctx->Sall || !ctx->I0s || !ctx->betas) return bail(fail(ctx, BTE_ENOMEM, "device allocation failed"));
    CU(cudaMemsetAsync(ctx->Sall, 0, (size_t)ctx->nranks * ncl * sizeof(double), ctx->stream));
  }
  ctx->T = (double *)dev_alloc(ctx, ncl * sizeof(double));
  ctx->zbeta = (double *)dev_alloc(ctx, ncl * ctx->nb * sizeof(double));
  if (!ctx->zbeta) return bail(fail(ctx, BTE_ENOMEM, "device allocation failed"));
  CU(cudaMemsetAsync(ctx->zbeta, 0, ncl * ctx->nb * sizeof(double), ctx->stream));
  ctx->Dpart = (double *)dev_alloc(ctx, ncl * nslot * ctx->nb * sizeof(double));
  ctx->d_err = (unsigned long long *)dev_alloc(ctx, sizeof(unsigned long long));
  if (!ctx->I0c || !ctx->dI0c || !ctx->beta || !ctx->T || !ctx->Dpart || !ctx->d_err)
    return bail(fail(ctx, BTE_ENOMEM, "device allocation failed"));
  CU(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long), ctx->stream));
  // staging for host <-> device state transfers (canonical order), <= 256 MB
  const int64_t per_cell = (int64_t)ctx->nd * ctx->nb * sizeof(double);
  ctx->staging_cells = std::max<int64_t>(1, std::min<int64_t>(ncl, (256ll << 20) / per_cell));
  ctx->staging = (double *)dev_alloc(ctx, ctx->staging_cells * per_cell);
  if (!ctx->staging) return bail(fail(ctx, BTE_ENOMEM, "staging allocation failed"));
  for (int r = 0; r < 6; ++r) {
    g.kind[r] = ctx->refl_closed[r / 2] ? BC_SPEC : BC_DIFF;
    const int64_t nf = n_faces_global(ctx, r);
    ctx->gtab[r] = (double *)dev_alloc(ctx, nf * ctx->nb * sizeof(double));
    if (!ctx->gtab[r]) return bail(fail(ctx, BTE_ENOMEM, "ghost table allocation failed"));
    g.gtab[r] = ctx->gtab[r];
    // diffuse denominator: sum over incoming directions of w|s_a| (octant tree)
    const int a = r / 2;
    const double sg = (r & 1) ? 1.0 : -1.0;
    double q[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int d = 0; d < ctx->nd; ++d) {
      const double sa = ctx->s[3 * d + a];
      if (sg * sa < 0.0) q[octant_of(&ctx->s[3 * d])] += ctx->w[d] * std::fabs(sa);
    }
    g.diff_den[r] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
  }
  if (uh) {  // unstructured tables (a0)
    int64_t *d_nbr = nullptr;
    double *d_an = nullptr, *d_sw = nullptr;
    // device rows padded to 4 faces: nbr [nc][4] (32 B), an [nc][4][3] (96 B), so
    // that the pipelined sweep moves them with 16-B bulk copies
    const int KP = uh->K <= 4 ? 4 : 8;  // device face slots per cell
    std::vector<int64_t> nbr4(KP * (size_t)uh->nc, -1);
    std::vector<double> an4(3 * KP * (size_t)uh->nc, 0.0);
    for (int64_t c = 0; c < uh->nc; ++c)
      for (int f = 0; f < uh->K; ++f) {
        nbr4[KP * c + f] = uh->nbr[c * uh->K + f];
        for (int a = 0; a < 3; ++a) an4[3 * KP * c + 3 * f + a] = uh->an[(c * uh->K + f) * 3 + a];
      }
    if ((st = upload(ctx, &d_nbr, nbr4.data(), nbr4.size()))) return bail(st);
    if ((st = upload(ctx, &d_an, an4.data(), an4.size()))) return bail(st);
    if ((st = upload(ctx, &ctx->d_ucen, uh->cen.data(), uh->cen.size()))) return bail(st);
    std::vector<double> sw(4 * (size_t)ctx->nd);
    for (int sj = 0; sj < ctx->nd; ++sj) {
      const int d = ctx->canon_d[sj];
      for (int a = 0; a < 3; ++a) sw[4 * sj + a] = ctx->s[3 * d + a];
      sw[4 * sj + 3] = ctx->w[d];
    }
    if ((st = upload(ctx, &d_sw, sw.data(), sw.size()))) return bail(st);
    ctx->u.nbr = d_nbr;
    ctx->u.an = d_an;
    ctx->u.sw = d_sw;
    for (int r = 0; r < 6; ++r) {
      int64_t *d_rc = nullptr, *d_rf = nullptr;
      if ((st = upload(ctx, &d_rc, uh->rcell[r].data(), uh->rcell[r].size()))) return bail(st);
      if ((st = upload(ctx, &d_rf, uh->rface[r].data(), uh->rface[r].size()))) return bail(st);
      ctx->u.rcell[r] = d_rc;
      ctx->u.rface[r] = d_rf;
    }
    int64_t nsend = 0, nrecv = 0;
    for (const UPeer &pe : ctx->upeers) {
      int64_t *d_sc = nullptr;
      if ((st = upload(ctx, &d_sc, pe.send_cells.data(), pe.send_cells.size()))) return bail(st);
      ctx->d_usend.push_back(d_sc);
      nsend += (int64_t)pe.send_cells.size();
      nrecv += pe.recv_cnt;
    }
    if (!ctx->upeers.empty()) {
      ctx->d_usendbuf = (double *)dev_alloc(ctx, (size_t)nsend * nslot * g.Es * sizeof(double));
      ctx->d_urecvbuf = (double *)dev_alloc(ctx, (size_t)nrecv * nslot * g.Es * sizeof(double));
      if (!ctx->d_usendbuf || !ctx->d_urecvbuf) return bail(fail(ctx, BTE_ENOMEM, "halo buffer allocation failed"));
    }
  }
  if (const char *e = getenv("BTE_SWEEP")) ctx->use_tma = strcmp(e, "plain") != 0;
  if (const char *e = getenv("BTE_STAGES")) ctx->stages_override = atoi(e);
  if (const char *e = getenv("BTE_SEGS")) ctx->seg_override = atoi(e);
  if (const char *e = getenv("BTE_THREADS")) ctx->target_threads = atoi(e);
  if (const char *e = getenv("BTE_SMEM_KB")) ctx->smem_budget_kb = atoi(e);
  // segment length along the march axis (measured on B200, configs 2 and 3):
  // ~16 planes keeps the cross-axis neighbour columns' reads within L2 reach
  // (short lag between adjacent columns) while the per-segment restart costs
  // one extra upwind-plane read per 16 cells.
  // small problems: enough segments for ~8 CTAs per SM (config 1, 20 x 20
  // cells x 4 quadrants: 1 -> 15 segments, sweep 0.019 -> 0.0085 ms)
  {
    // 3-D: ~32-plane segments (ncu, round 2: config 4 17.63 -> 17.50 B/DOF, sweep
    // 6.15 -> 6.06 ms; config 3 17.66 -> 17.53 B/DOF; full columns raise the
    // y-upwind L2 misses to 18.4-20.2 B/DOF; profiles/round2_ab_seg.jsonl)
    int nseg = g.dim == 3 ? std::max(1, (int)((g.nplanes + 16) / 32)) : std::max(1, (int)((g.nplanes + 8) / 16));
    const int64_t tasks = (int64_t)g.ncross * g.nslot;
    // (>= 12 CTAs per SM: Fig. 9's 160 column tasks x 8 segments = 1.2 waves
    // of the small-block sweep -> 12 segments, 0.0405 -> 0.0371 ms; knob table
    // profiles/round2_ab_knobs.jsonl)
    const int64_t want = 12 * 148;
    if (tasks * nseg < want) nseg = (int)std::min<int64_t>(g.nplanes, (want + tasks - 1) / tasks);
    if (ctx->seg_override > 0) nseg = std::min(ctx->seg_override, g.nplanes);
    ctx->seg_len = (g.nplanes + nseg - 1) / nseg;
  }
  if (const char *e = getenv("BTE_SPARE")) ctx->no_spare = atoi(e) == 0;
  if (const char *e = getenv("BTE_PF")) ctx->pf = atoi(e);
  if (const char *e = getenv("BTE_NEWTON_LPC")) ctx->newton_lpc = atoi(e);
  // 3-D sweep column order: strips of 16 columns along x (measured on B200,
  // config 4: DRAM 20.3 -> 17.6 B/DOF per sweep launch)
  ctx->raster = g.dim == 3 ? 16 : 0;
  if (const char *e = getenv("BTE_RASTER")) ctx->raster = std::max(0, atoi(e));
  if (const char *e = getenv("BTE_GRAPH")) ctx->use_graph = atoi(e) != 0;
  if (const char *e = getenv("BTE_SC_DIRECT")) ctx->sc_direct = atoi(e) != 0;
  if (const char *e = getenv("BTE_UGENERIC")) ctx->ugeneric = atoi(e) != 0;
  if (const char *e = getenv("BTE_USINGLE")) ctx->usingle = atoi(e) != 0;
  if (const char *e = getenv("BTE_NEWTON_PREDICT")) ctx->newton_predict = atoi(e);
  if (const char *e = getenv("BTE_NEWTON_MINB")) ctx->newton_minb = atoi(e);
  if (const char *e = getenv("BTE_NEWTON_STATS"))
    if (atoi(e)) {
      ctx->d_stats = (unsigned long long *)dev_alloc(ctx, 4 * sizeof(unsigned long long));
      if (ctx->d_stats) CU(cudaMemsetAsync(ctx->d_stats, 0, 4 * sizeof(unsigned long long), ctx->stream));
    }
  if (const char *e = getenv("BTE_OVERLAP")) ctx->overlap = atoi(e);
  CU(cudaEventCreateWithFlags(&ctx->ev_bnd, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
  if (ctx->nranks > 1 && !ctx->comm_stream) CU(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));

  // ---- multi-GPU communicator
  if (ctx->nranks > 1 && run->nccl_id) {
    std::string emsg;
    if (nccl_shim_init(&ctx->nccl_comm, run->nccl_id, ctx->nranks, ctx->rank, &emsg) != 0)
      return bail(fail(ctx, BTE_ENCCL, "NCCL init failed: %s", emsg.c_str()));
    int cn = 0, cr = -1;
    if (nccl_shim_comm_info(ctx->nccl_comm, &cn, &cr, &emsg) != 0)
      return bail(fail(ctx, BTE_ENCCL, "NCCL comm query failed: %s", emsg.c_str()));
    if (cn != ctx->nranks || cr != ctx->rank)
      return bail(fail(ctx, BTE_ENCCL, "NCCL communicator is rank %d of %d, expected %d of %d", cr, cn, ctx->rank,
                       ctx->nranks));
    fprintf(stderr, "[bte] NCCL communicator: rank %d of %d (device %d, %s)\n", cr, cn, ctx->device,
            ctx->band ? "band partition" : ctx->umesh ? "cell partition" : "slab partition");
    if (!ctx->comm_stream) CU(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  }

  // ---- initial state: equilibrium at T_init
  std::vector<double> T0(ncl, ctx->T_init);
  CU(cudaMemcpyAsync(ctx->T, T0.data(), ncl * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if ((st = refresh(ctx))) return bail(st);
  CU(launch_fill_equilibrium(g, ctx->I0s, ctx->I[0], ctx->stream));
  ctx->cur = 0;
  if (ctx->nccl_comm && !ctx->band &&
      (st = ctx->umesh ? uhalo_exchange(ctx, ctx->I[0], nullptr) : halo_exchange(ctx, ctx->I[0])))
    return bail(st);
  CU(cudaStreamSynchronize(ctx->stream));
  *out = ctx;
  return BTE_OK;
}

bte_status bte_set_bc(bte_ctx *ctx, int region, int kind, const double *T_wall, double T_uniform) {
  if (!ctx) return BTE_EINVAL;
  graph_invalidate(ctx);
  const int nreg = ctx->mesh.dim == 3 ? 6 : 4;
  if (region < 0 || region >= nreg) return fail(ctx, BTE_EINVAL, "region %d out of range", region);
  if (kind == BTE_BC_SPECULAR) {
    if (!ctx->refl_closed[region / 2])
      return fail(ctx, BTE_ENOTCLOSED, "specular wall %d: direction set is not closed under the axis-%d reflection",
                  region, region / 2);
  } else if (kind == BTE_BC_ISOTHERMAL) {
    const int64_t nf = n_faces_global(ctx, region);
    std::vector<double> Tw(nf, T_uniform);
    if (T_wall) std::copy(T_wall, T_wall + nf, Tw.begin());
    double tmax = ctx->Tmax;
    for (double t : Tw) {
      if (!(t > 0)) return fail(ctx, BTE_EINVAL, "wall temperatures must be > 0");
      tmax = std::max(tmax, t);
    }
    const double old = ctx->Tmax;
    ctx->Tmax = tmax;
    bte_status st = check_dt(ctx);
    if (st) {
      ctx->Tmax = old;
      return st;
    }
    double *d_Tw = nullptr;
    CU(cudaMalloc(&d_Tw, nf * sizeof(double)));
    CU(cudaMemcpyAsync(d_Tw, Tw.data(), nf * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CU(launch_iso_table(ctx->m, d_Tw, nf, ctx->gtab[region], ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaFree(d_Tw));
  } else if (kind == BTE_BC_DIFFUSE) {
    if (!(ctx->g.diff_den[region] > 0))
      return fail(ctx, BTE_EINVAL, "diffuse wall %d: no direction crosses it", region);
  } else if (kind == BTE_BC_PARTIAL) {
    return fail(ctx, BTE_EINVAL, "partially specular wall %d: use bte_set_bc_partial", region);
  } else {
    return fail(ctx, BTE_EINVAL, "unknown boundary kind %d", kind);
  }
  ctx->g.kind[region] = kind;
  return BTE_OK;
}

bte_status bte_set_bc_partial(bte_ctx *ctx, int region, double specularity) {
  if (!ctx) return BTE_EINVAL;
  graph_invalidate(ctx);
  const int nreg = ctx->mesh.dim == 3 ? 6 : 4;
  if (region < 0 || region >= nreg) return fail(ctx, BTE_EINVAL, "region %d out of range", region);
  if (!(specularity >= 0.0 && specularity <= 1.0))
    return fail(ctx, BTE_EINVAL, "specularity must lie in [0, 1] (got %g)", specularity);
  if (!ctx->refl_closed[region / 2])
    return fail(ctx, BTE_ENOTCLOSED, "partial wall %d: direction set is not closed under the axis-%d reflection",
                region, region / 2);
  if (!(ctx->g.diff_den[region] > 0))
    return fail(ctx, BTE_EINVAL, "partial wall %d: no direction crosses it", region);
  ctx->g.spec_p[region] = specularity;
  ctx->g.spec_q[region] = 1.0 - specularity;
  ctx->g.kind[region] = BC_PART;
  return BTE_OK;
}

static bte_status transfer_I(bte_ctx *ctx, double *host, int to_device) {
  const Geometry &g = ctx->g;
  const int64_t per_cell = (int64_t)ctx->nd * ctx->nb;
  for (int64_t c0 = 0; c0 < ctx->ncells_local; c0 += ctx->staging_cells) {
    const int64_t n = std::min(ctx->staging_cells, ctx->ncells_local - c0);
    if (to_device) {
      CU(cudaMemcpyAsync(ctx->staging, host + c0 * per_cell, n * per_cell * sizeof(double), cudaMemcpyHostToDevice,
                         ctx->stream));
      CU(launch_permute(g, ctx->d_dmap, ctx->nd, ctx->staging, c0, n, ctx->I[ctx->cur], 1, ctx->stream));
    } else {
      CU(launch_permute(g, ctx->d_dmap, ctx->nd, ctx->staging, c0, n, ctx->I[ctx->cur], 0, ctx->stream));
      CU(cudaMemcpyAsync(host + c0 * per_cell, ctx->staging, n * per_cell * sizeof(double), cudaMemcpyDeviceToHost,
                         ctx->stream));
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return BTE_OK;
}

static bte_status run_newton(bte_ctx *ctx, int64_t step);

bte_status bte_set_state(bte_ctx *ctx, const double *I, const double *T) {
  if (!ctx) return BTE_EINVAL;
  if (!I && !T) return fail(ctx, BTE_EINVAL, "set_state needs I or T");
  if (ctx->band && !T) return fail(ctx, BTE_EINVAL, "band context: set_state needs T");
  const int64_t ncl = ctx->ncells_local;
  bte_status st;
  if (T) {
    double tmax = ctx->Tmax;
    for (int64_t c = 0; c < ncl; ++c) {
      if (!(T[c] > 0) || !std::isfinite(T[c])) return fail(ctx, BTE_EINVAL, "T must be finite and > 0");
      tmax = std::max(tmax, T[c]);
    }
    const double old = ctx->Tmax;
    ctx->Tmax = tmax;
    if ((st = check_dt(ctx))) {
      ctx->Tmax = old;
      return st;
    }
    CU(cudaMemcpyAsync(ctx->T, T, ncl * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  } else {
    std::vector<double> T0(ncl, ctx->T_init);
    CU(cudaMemcpyAsync(ctx->T, T0.data(), ncl * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  }
  if ((st = refresh(ctx))) return st;
  if (I) {
    if ((st = transfer_I(ctx, const_cast<double *>(I), 1))) return st;
  } else {
    CU(launch_fill_equilibrium(ctx->g, ctx->I0s, ctx->I[ctx->cur], ctx->stream));
  }
  if (ctx->nccl_comm && !ctx->band &&
      (st = ctx->umesh ? uhalo_exchange(ctx, ctx->I[ctx->cur], nullptr) : halo_exchange(ctx, ctx->I[ctx->cur])))
    return st;
  if (I && !T) {
    // T from one reduction + Newton from T_init (beta_next = beta(T_init)):
    // Dpart = sum_j w_j (I0c - I) per octant of the given I, then the Newton kernel.
    CU(launch_dpart_from_I(ctx->g, ctx->I[ctx->cur], ctx->I0c, ctx->Dpart, ctx->stream));
    // the temperature of a state is the plain balance (#2), also under the
    // semi-implicit integrator (its weights belong to its step)
    const int semi = ctx->semi;
    ctx->semi = 0;
    st = run_newton(ctx, 0);
    ctx->semi = semi;
    if (st) return st;
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return sync_check(ctx);
}

bte_status bte_init_random(bte_ctx *ctx, uint64_t seed, const double phase[3], double T_mean, double T_amp,
                           double I_amp) {
  if (!ctx || !phase) return BTE_EINVAL;
  const double old = ctx->Tmax;
  ctx->Tmax = std::max(ctx->Tmax, T_mean + std::fabs(T_amp));
  bte_status st = check_dt(ctx);
  if (st) {
    ctx->Tmax = old;
    return st;
  }
  if (!(T_mean - std::fabs(T_amp) > 0)) return fail(ctx, BTE_EINVAL, "random start would give T <= 0");
  const bte_mesh &m = ctx->mesh;
  if (ctx->umesh)
    CU(launch_random_T_u(ctx->ncells_local, m.dim, ctx->d_ucen, ctx->ulo, ctx->uL, phase, T_mean, T_amp, ctx->T,
                         ctx->stream));
  else
    CU(launch_random_T(ctx->g, 0, m.dx, m.dy, m.dz, phase, T_mean, T_amp, ctx->T, ctx->stream));
  if ((st = refresh(ctx))) return st;
  CU(launch_random_I(ctx->g, ctx->d_canon_d, ctx->nd, seed, I_amp, ctx->I0s, ctx->I[ctx->cur], ctx->stream));
  if (ctx->nccl_comm && !ctx->band &&
      (st = ctx->umesh ? uhalo_exchange(ctx, ctx->I[ctx->cur], nullptr) : halo_exchange(ctx, ctx->I[ctx->cur])))
    return st;
  CU(cudaStreamSynchronize(ctx->stream));
  return BTE_OK;
}

// ---- the step

static bte_status launch_boundary(bte_ctx *ctx, const double *Icur, cudaStream_t strm = nullptr) {
  Geometry &g = ctx->g;
  cudaStream_t stream = strm ? strm : ctx->stream;
  const int nreg = g.dim == 3 ? 6 : 4;
  int n = 0;
  for (int r = 0; r < nreg; ++r) {
    const int a = r / 2;
    if (a == g.dim - 1 && !((r & 1) ? g.has_hi_wall : g.has_lo_wall)) continue;
    if (g.kind[r] == BC_DIFF || g.kind[r] == BC_PART) {
      if (ctx->umesh)
        CU(launch_udiffuse(g, ctx->u, Icur, r, ctx->gtab[r], stream));
      else
        CU(launch_diffuse(g, Icur, r, ctx->gtab[r], stream));
      ++n;
    }
    if ((g.kind[r] == BC_SPEC || g.kind[r] == BC_PART) && ctx->rot) {
      if (!ctx->gspec[r]) {  // first use: [faces][nslot*nj][nb]
        const size_t bytes = (size_t)n_faces_global(ctx, r) * g.nslot * g.nj * g.nb * sizeof(double);
        ctx->gspec[r] = (double *)dev_alloc(ctx, bytes);
        if (!ctx->gspec[r]) return fail(ctx, BTE_ENOMEM, "specular snapshot allocation (%zu bytes) failed", bytes);
        g.gspec[r] = ctx->gspec[r];
      }
      CU(launch_spec_snapshot(g, Icur, r, ctx->gspec[r], stream));
      ++n;
    }
  }
  ctx->tacc.launches += n;
  ctx->tacc.boundary_launches += n;
  return BTE_OK;
}

// walls that need a boundary pass before the sweep: diffuse ghosts, and under
// slot rotation the specular snapshots
static int n_diffuse(const bte_ctx *ctx) {
  int n = 0;
  for (int r = 0; r < (ctx->g.dim == 3 ? 6 : 4); ++r)
    n += ctx->g.kind[r] == BC_DIFF || ctx->g.kind[r] == BC_PART ||
         (ctx->rot && ctx->g.kind[r] == BC_SPEC);
  return n;
}

static NewtonArgs newton_args(bte_ctx *ctx, int64_t step) {
  NewtonArgs a{};
  a.sc_direct = ctx->sc_direct;
  a.step_ctr = ctx->graph_capture ? ctx->d_stepctr : nullptr;
  a.m = ctx->mF;
  a.Dpart = ctx->Dpart;
  a.T = ctx->T;
  a.I0c = ctx->I0c;
  a.dI0c = ctx->dI0c;
  a.beta_next = ctx->beta;
  a.nslot = ctx->g.nslot;
  a.nb = ctx->nbT;
  a.Sall = ctx->band ? ctx->Sall : nullptr;
  a.nparts = ctx->nranks;
  a.I0s = ctx->band ? ctx->I0s : nullptr;
  a.betas = ctx->band ? ctx->betas : nullptr;
  a.b0s = ctx->b0;
  a.semi_dt = ctx->semi ? ctx->dt : 0.0;
  a.nbs = ctx->nb;
  for (int k = 0; k < kMaxSlots; ++k) a.slot_oct[k] = ctx->g.slot_oct[k];
  for (int o = 0; o < 8; ++o) a.oct_slot[o] = ctx->g.oct_slot[o];
  a.W = ctx->W;
  a.ncells = ctx->ncells_local;
  a.cell0_global = ctx->g.cell0;
  a.err = ctx->d_err;
  a.step = step;
  a.col0 = 0;
  a.ncols = ctx->g.ncross;
  a.ncross = ctx->g.ncross;
  a.nplanes = ctx->g.nplanes;
  a.predict = ctx->newton_predict;
  a.minb = ctx->newton_minb;
  a.stats = ctx->d_stats;
  // band integrals lane per channel when its 16*ceil(nb/32) node terms per lane
  // are within 1.2x of the (node group, channel) mapping's 4*ceil(nb/8) -- it
  // saves the cross-lane sums (measured: 55 channels -7 % Newton, 40 channels +3.5 %)
  {
    const int nb = ctx->nbT;
    const bool lpc_auto = 16 * ((nb + 31) / 32) * 5 <= 6 * 4 * ((nb + 7) / 8);
    a.lpc = ctx->newton_lpc >= 0 ? ctx->newton_lpc : (lpc_auto ? 1 : 0);
  }
  return a;
}

static SweepArgs sweep_args(const bte_ctx *ctx, const double *Iin, double *Iout, int p_lo, int p_hi, int seg_len) {
  SweepArgs a{};
  a.slot0 = 0;
  a.nslots = 0;
  for (int sl = 0; sl < kMaxSlots; ++sl) a.out_off[sl] = ctx->g.slot_off[sl];
  a.col0 = 0;
  a.ncols = 0;
  a.p_lo = p_lo;
  a.p_hi = p_hi;
  a.g = ctx->g;
  a.Iin = Iin;
  a.Iout = Iout;
  a.I0c = ctx->I0s;
  a.beta = ctx->semi ? ctx->zbeta : ctx->betas;
  a.Dpart = ctx->Dpart;
  a.v = ctx->m.v;
  a.dt = ctx->dt;
  a.seg_len = seg_len > 0 ? seg_len : ctx->seg_len;
  a.use_tma = ctx->use_tma;
  a.stages_override = ctx->stages_override;
  a.target_threads = ctx->target_threads;
  a.smem_budget_kb = ctx->smem_budget_kb;
  a.no_spare = ctx->no_spare;
  a.pf = ctx->pf;
  a.raster = ctx->raster;
  return a;
}

// a1 (inline ghosts) + a2 over planes [p_lo, p_hi) (all when p_hi <= p_lo)
static bte_status launch_sweep_step(bte_ctx *ctx, const double *Iin, double *Iout, int p_lo = 0, int p_hi = 0,
                                    int seg_len = 0) {
  if (ctx->umesh) {
    USweepArgs a{};
    a.g = ctx->g;
    a.u = ctx->u;
    a.Iin = Iin;
    a.Iout = Iout;
    a.I0c = ctx->I0s;
    a.beta = ctx->semi ? ctx->zbeta : ctx->betas;
    a.Dpart = ctx->Dpart;
    a.v = ctx->m.v;
    a.dt = ctx->dt;
    a.target_threads = ctx->target_threads;
    a.pipelined = ctx->use_tma;
    a.stages = ctx->stages_override;
    a.chunk = ctx->seg_override;
    a.generic = ctx->ugeneric;
    a.single_buf = ctx->usingle;
    CU(launch_usweep(a, ctx->stream));
    ctx->tacc.launches++;
    ctx->tacc.sweep_launches++;
    return BTE_OK;
  }
  if (ctx->rot) {
    // octant-slot rotation: octant k is swept from its region into the spare
    // region, whose old occupant's region becomes the next spare; the octants
    // go one launch each, in slot order (each reads only its own I^n; the
    // specular ghosts come from the boundary pass's snapshot)
    for (int k = 0; k < ctx->g.nslot; ++k) {
      SweepArgs a = sweep_args(ctx, Iin, Iout, p_lo, p_hi, seg_len);
      a.slot0 = k;
      a.nslots = 1;
      a.out_off[k] = (int64_t)ctx->spare * ctx->g.slot_stride;
      CU(launch_sweep(a, ctx->stream));
      const int freed = (int)(ctx->g.slot_off[k] / ctx->g.slot_stride);
      ctx->g.slot_off[k] = (int64_t)ctx->spare * ctx->g.slot_stride;
      ctx->spare = freed;
      ctx->tacc.launches++;
      ctx->tacc.sweep_launches++;
    }
    return BTE_OK;
  }
  SweepArgs a = sweep_args(ctx, Iin, Iout, p_lo, p_hi, seg_len);
  CU(launch_sweep(a, ctx->stream));
  ctx->tacc.launches++;
  ctx->tacc.sweep_launches++;
  return BTE_OK;
}

static bte_status run_newton(bte_ctx *ctx, int64_t step) {
  NewtonArgs a = newton_args(ctx, step);
  if (ctx->tau_mode == 1)
    CU(launch_newton_sc(a, ctx->stream));
  else
    CU(launch_newton(a, ctx->stream));
  ctx->tacc.launches++;
  ctx->tacc.newton_launches++;
  return BTE_OK;
}


static bte_status span_begin(bte_ctx *ctx, bool t, int kind, cudaStream_t s, size_t *id) {
  if (!t) return BTE_OK;
  if (ctx->ev_used + 2 > ctx->ev.size()) {  // pool exhausted: stop recording, and say so
    ctx->tacc.truncated = 1;
    return BTE_OK;
  }
  *id = ctx->ev_used;
  ctx->ev_used += 2;
  ctx->spans.push_back({kind, *id});
  CU(cudaEventRecord(ctx->ev[*id], s));
  return BTE_OK;
}
static bte_status span_end(bte_ctx *ctx, bool t, cudaStream_t s, size_t id) {
  if (!t || id == (size_t)-1) return BTE_OK;
  CU(cudaEventRecord(ctx->ev[id + 1], s));
  return BTE_OK;
}

// Launch one step (a1..a4) of ctx on its stream; the caller exchanges halos.
// split: sweep the two owned boundary planes first and record ctx->ev_bnd, so
// the halo exchange (a5) can run on the comm stream while the interior planes
// are swept (SURVEY 8(e) overlap schedule).
static bte_status step_launch(bte_ctx *ctx, bool t, bool split = false) {
  const bool has_bnd = n_diffuse(ctx) > 0;
  const int np = ctx->g.nplanes;
  bte_status st;
  double *Iin = ctx->I[ctx->cur];
  double *Iout = ctx->I[1 - ctx->cur];
  size_t id = (size_t)-1;
  nvtx_push("bte_step");
  if (has_bnd && ctx->bnd_ready) {
    // the previous step already ran this step's boundary pass on the side
    // stream, concurrently with its Newton
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side, 0));
    ctx->bnd_ready = false;
  } else if (has_bnd) {
    nvtx_push("a1 boundary");
    if ((st = span_begin(ctx, t, 2, ctx->stream, &id))) return st;
    if ((st = launch_boundary(ctx, Iin))) return st;
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    nvtx_pop();
  }
  // the semi-implicit step exchanges halos after its relaxation pass
  if (split && (ctx->rot || ctx->semi || ctx->umesh)) split = false;
  nvtx_push("a2 sweep");
  if (split) {
    id = (size_t)-1;
    if ((st = span_begin(ctx, t, 0, ctx->stream, &id))) return st;
    if ((st = launch_sweep_step(ctx, Iin, Iout, 0, 1, 1))) return st;
    if (np > 1 && (st = launch_sweep_step(ctx, Iin, Iout, np - 1, np, 1))) return st;
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    CU(cudaEventRecord(ctx->ev_bnd, ctx->stream));
    if (np > 2) {
      id = (size_t)-1;
      if ((st = span_begin(ctx, t, 0, ctx->stream, &id))) return st;
      if ((st = launch_sweep_step(ctx, Iin, Iout, 1, np - 1))) return st;
      if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    }
  } else {
    id = (size_t)-1;
    if ((st = span_begin(ctx, t, 0, ctx->stream, &id))) return st;
    if ((st = launch_sweep_step(ctx, Iin, Iout))) return st;
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
  }
  nvtx_pop();
  if (has_bnd && ctx->rot && !ctx->semi && ctx->prefetch_bnd) {
    // octant-slot rotation: the next step's boundary pass (specular
    // snapshots, diffuse tables) reads only I^{n+1}, not T: run it on a side
    // stream concurrently with this step's Newton (FP64-bound vs memory-bound)
    if (!ctx->side_stream) {
      CU(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&ctx->ev_swept, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(ctx->ev_swept, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side_stream, ctx->ev_swept, 0));
    nvtx_push("a1 boundary (next step, side stream)");
    id = (size_t)-1;
    if ((st = span_begin(ctx, t, 2, ctx->side_stream, &id))) return st;
    if ((st = launch_boundary(ctx, Iout, ctx->side_stream))) return st;
    if ((st = span_end(ctx, t, ctx->side_stream, id))) return st;
    nvtx_pop();
    CU(cudaEventRecord(ctx->ev_side, ctx->side_stream));
    ctx->bnd_ready = true;
  }
  nvtx_push("a3+a4 reduce+Newton");
  id = (size_t)-1;
  if ((st = span_begin(ctx, t, 1, ctx->stream, &id))) return st;
  if ((st = run_newton(ctx, ctx->steps_done))) return st;
  if ((st = span_end(ctx, t, ctx->stream, id))) return st;
  if (ctx->semi) {  // reading R-l: I^{n+1} = (J + dt beta I0(T^{n+1})) / (1 + dt beta)
    id = (size_t)-1;
    if ((st = span_begin(ctx, t, 1, ctx->stream, &id))) return st;
    CU(launch_relax(ctx->g, Iout, ctx->I0c, ctx->beta, ctx->dt, ctx->stream));
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    ctx->tacc.launches++;
  }
  nvtx_pop();
  if (!split) CU(cudaEventRecord(ctx->ev_bnd, ctx->stream));
  nvtx_pop();
  return BTE_OK;
}

// ---- implicit step by source iteration (reading R-n)

// the (slot, column) tasks of the implicit sweep in an upwind-topological
// order: by distance of the column from its octant's upwind corner, octants
// interleaved, so a task's upwind columns always hold smaller tickets.
// (Measured on config 3: a strip raster -- also topological, neighbours one
// and 16 tickets apart -- took 32.8 ms per iteration against 26 ms: each
// ticket then waits on the one just before it, the chains never get slack.)
static bte_status implicit_setup(bte_ctx *ctx) {
  if (ctx->d_tasks) return BTE_OK;
  const Geometry &g = ctx->g;
  const int nx = g.dim == 3 ? g.nx : g.ncross, ny = g.dim == 3 ? g.ny : 1;
  std::vector<std::pair<int64_t, int2>> key;
  key.reserve((size_t)g.nslot * g.ncross);
  for (int sl = 0; sl < g.nslot; ++sl) {
    const int oct = g.slot_oct[sl];
    const bool xneg = oct & 4, yneg = oct & 2;
    for (int c = 0; c < g.ncross; ++c) {
      const int x = c % nx, y = c / nx;
      const int64_t dist = (xneg ? nx - 1 - x : x) + (g.dim == 3 ? (yneg ? ny - 1 - y : y) : 0);
      key.push_back({(dist * g.nslot + sl) * (int64_t)g.ncross + c, make_int2(sl, c)});
    }
  }
  std::sort(key.begin(), key.end(), [](const std::pair<int64_t, int2> &a, const std::pair<int64_t, int2> &b) {
    return a.first < b.first;
  });
  std::vector<int2> tasks(key.size());
  for (size_t k = 0; k < key.size(); ++k) tasks[k] = key[k].second;
  bte_status st;
  if ((st = upload(ctx, &ctx->d_tasks, tasks.data(), tasks.size()))) return st;
  ctx->d_prog = (int *)dev_alloc(ctx, tasks.size() * 32 * sizeof(int));  // one 128-B line per counter
  ctx->d_ticket = (unsigned *)dev_alloc(ctx, 16);
  ctx->d_conv = (unsigned long long *)dev_alloc(ctx, 2 * sizeof(unsigned long long));
  if (!ctx->d_prog || !ctx->d_ticket || !ctx->d_conv) return fail(ctx, BTE_ENOMEM, "implicit-step tables");
  return BTE_OK;
}

// (a): wall data of the current iterate Icur -- diffuse tables and, for
// specular / partial walls, the snapshot of the reflected intensities -- with
// their largest relative change since the previous iterate into d_conv[1]
static bte_status implicit_boundary(bte_ctx *ctx, const double *Icur, bool t) {
  Geometry &g = ctx->g;
  const int nreg = g.dim == 3 ? 6 : 4;
  size_t id = (size_t)-1;
  bte_status st;
  if ((st = span_begin(ctx, t, 2, ctx->stream, &id))) return st;
  for (int r = 0; r < nreg; ++r) {
    if (g.kind[r] == BC_DIFF || g.kind[r] == BC_PART) {
      CU(launch_diffuse(g, Icur, r, ctx->gtab[r], ctx->stream, ctx->d_conv + 1));
      ctx->tacc.launches++;
      ctx->tacc.boundary_launches++;
    }
    if (g.kind[r] == BC_SPEC || g.kind[r] == BC_PART) {
      if (!ctx->gspec[r]) {
        const size_t bytes = (size_t)n_faces_global(ctx, r) * g.nslot * g.nj * g.nb * sizeof(double);
        ctx->gspec[r] = (double *)dev_alloc(ctx, bytes);
        if (!ctx->gspec[r]) return fail(ctx, BTE_ENOMEM, "specular snapshot allocation (%zu bytes) failed", bytes);
        g.gspec[r] = ctx->gspec[r];
      }
      CU(launch_spec_snapshot(g, Icur, r, ctx->gspec[r], ctx->stream, ctx->d_conv + 1));
      ctx->tacc.launches++;
      ctx->tacc.boundary_launches++;
    }
  }
  return span_end(ctx, t, ctx->stream, id);
}

static bte_status implicit_step(bte_ctx *ctx, bool t) {
  bte_status st;
  if ((st = implicit_setup(ctx))) return st;
  const Geometry &g = ctx->g;
  const int64_t ncl = ctx->ncells_local;
  double *In = ctx->I[ctx->cur];
  double *Iout = ctx->I[1 - ctx->cur];
  bool iter_walls = false;  // walls whose data come from the iterate
  for (int r = 0; r < (g.dim == 3 ? 6 : 4); ++r) iter_walls |= g.kind[r] != BC_ISO;
  nvtx_push("bte_step (implicit)");
  // beta(T^n) weights the whole step (lagged as #15); I0c, dI0c are at T^n already
  CU(launch_refresh(ctx->mF, ctx->T, ncl, nullptr, nullptr, ctx->beta, ctx->stream));
  ctx->tacc.launches++;
  int64_t k = 0;
  for (; k < ctx->imp_max_iter; ++k) {
    CU(cudaMemsetAsync(ctx->d_conv, 0, 2 * sizeof(unsigned long long), ctx->stream));
    nvtx_push("a1 boundary (iterate)");
    if ((st = implicit_boundary(ctx, k == 0 ? In : Iout, t))) return st;
    nvtx_pop();
    nvtx_push("a2 implicit sweep");
    CU(cudaMemsetAsync(ctx->d_prog, 0, (size_t)g.nslot * g.ncross * 32 * sizeof(int), ctx->stream));
    CU(cudaMemsetAsync(ctx->d_ticket, 0, sizeof(unsigned), ctx->stream));
    SweepArgs a = sweep_args(ctx, In, Iout, 0, 0, 0);
    a.g.rot = 1;  // wall ghosts from the snapshot of I^k (the sweep overwrites I^k)
    size_t id = (size_t)-1;
    if ((st = span_begin(ctx, t, 0, ctx->stream, &id))) return st;
    CU(launch_sweep_imp(a, ctx->d_tasks, g.nslot * g.ncross, ctx->d_prog, ctx->d_ticket, ctx->stream));
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    ctx->tacc.launches++;
    ctx->tacc.sweep_launches++;
    nvtx_pop();
    nvtx_push("a3+a4 reduce+Newton (iterate)");
    NewtonArgs na = newton_args(ctx, ctx->steps_done);
    na.beta_fixed = 1;
    na.dTmax = ctx->d_conv;
    id = (size_t)-1;
    if ((st = span_begin(ctx, t, 1, ctx->stream, &id))) return st;
    CU(launch_newton(na, ctx->stream));
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
    ctx->tacc.launches++;
    ctx->tacc.newton_launches++;
    nvtx_pop();
    if (ctx->imp_tol > 0.0) {  // stop when both inputs of the last sweep had settled
      unsigned long long h[2];
      CU(cudaMemcpyAsync(h, ctx->d_conv, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      double dT, dg;
      std::memcpy(&dT, &h[0], 8);
      std::memcpy(&dg, &h[1], 8);
      if (iter_walls && k == 0) dg = INFINITY;
      if (dT <= ctx->imp_tol && dg <= ctx->imp_tol) {
        ++k;
        break;
      }
    }
  }
  ctx->imp_iters.push_back(k);
  nvtx_pop();
  return BTE_OK;
}

static void graph_invalidate(bte_ctx *ctx) {
  for (auto &e : ctx->gexec)
    if (e) {
      cudaGraphExecDestroy(e);
      e = nullptr;
    }
}

// One explicit step by replaying its captured graph (one context, two
// buffers, no timing): the launches of step_launch for this buffer parity,
// plus k_step_tick for the device step index the Newton's error key reads.
static bte_status graph_step(bte_ctx *ctx) {
  const int par = ctx->cur;
  if (!ctx->gexec[par]) {
    if (!ctx->d_stepctr) {
      ctx->d_stepctr = (unsigned long long *)dev_alloc(ctx, sizeof(unsigned long long));
      if (!ctx->d_stepctr) return fail(ctx, BTE_ENOMEM, "graph step counter");
    }
    const int64_t l0 = ctx->tacc.launches;
    cudaGraph_t graph = nullptr;
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on ctx->stream
    if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->cap_stream;
    cudaError_t e0 = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed);
    if (e0 != cudaSuccess) {
      ctx->stream = user;
      CU(e0);
    }
    ctx->graph_capture = true;
    bte_status st = step_launch(ctx, false);
    cudaError_t e = st ? cudaSuccess : launch_step_tick(ctx->d_stepctr, ctx->stream);
    ctx->graph_capture = false;
    cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &graph);
    ctx->stream = user;
    if (st) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    CU(e);
    CU(e2);
    e = cudaGraphInstantiate(&ctx->gexec[par], graph, 0);
    cudaGraphDestroy(graph);
    CU(e);
    ctx->graph_launches = ctx->tacc.launches - l0 + 1;
    ctx->tacc.launches = l0;
  }
  ctx->h_stepctr = (unsigned long long)ctx->steps_done;
  CU(cudaMemcpyAsync(ctx->d_stepctr, &ctx->h_stepctr, sizeof ctx->h_stepctr, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaGraphLaunch(ctx->gexec[par], ctx->stream));
  ctx->tacc.launches += ctx->graph_launches;
  return BTE_OK;
}

// Band partition, first half of a step: boundary + sweep of this part's
// channels, then its partial S_r = sum_{b in part} c_b D_b into row `rank`
// of Sall (the bands couple only through this reduction).
static bte_status band_sweep_launch(bte_ctx *ctx, bool t) {
  bte_status st;
  double *Iin = ctx->I[ctx->cur];
  double *Iout = ctx->I[1 - ctx->cur];
  size_t id = (size_t)-1;
  if (n_diffuse(ctx) > 0) {
    if ((st = span_begin(ctx, t, 2, ctx->stream, &id))) return st;
    if ((st = launch_boundary(ctx, Iin))) return st;
    if ((st = span_end(ctx, t, ctx->stream, id))) return st;
  }
  id = (size_t)-1;
  if ((st = span_begin(ctx, t, 0, ctx->stream, &id))) return st;
  if ((st = launch_sweep_step(ctx, Iin, Iout))) return st;
  if ((st = span_end(ctx, t, ctx->stream, id))) return st;
  id = (size_t)-1;
  if ((st = span_begin(ctx, t, 1, ctx->stream, &id))) return st;
  CU(launch_band_partial(ctx->g, ctx->mF, ctx->Dpart, ctx->T, ctx->ncells_local,
                         ctx->Sall + (int64_t)ctx->rank * ctx->ncells_local, ctx->stream));
  ctx->tacc.launches++;
  ctx->tacc.newton_launches++;
  return span_end(ctx, t, ctx->stream, id);
}

// Band partition, second half: the Newton over all channels from the gathered
// partials (identical inputs, hence identical T, on every part).
static bte_status band_newton_launch(bte_ctx *ctx, bool t) {
  bte_status st;
  size_t id = (size_t)-1;
  if ((st = span_begin(ctx, t, 1, ctx->stream, &id))) return st;
  if ((st = run_newton(ctx, ctx->steps_done))) return st;
  return span_end(ctx, t, ctx->stream, id);
}


// One step = [diffuse ghosts] + for each column chunk k: sweep(k) on the
// context stream and, on the Newton stream once sweep(k) is done, Newton(k)
// (one chunk by default) + [halo exchange (NCCL)].
bte_status bte_step(bte_ctx *ctx, int64_t nsteps) {
  if (!ctx) return BTE_EINVAL;
  if (nsteps < 0) return fail(ctx, BTE_EINVAL, "nsteps < 0");
  if (ctx->nranks > 1 && !ctx->nccl_comm)
    return fail(ctx, BTE_EINVAL, "local-mode (slab or band) context: advance the group with bte_group_step");
  bte_status st;
  if (ctx->band) {
    const int64_t ncl = ctx->ncells_local;
    for (int64_t s = 0; s < nsteps; ++s) {
      const bool t = ctx->timing && ctx->timing_used < ctx->timing_max;
      if ((st = band_sweep_launch(ctx, t))) return st;
      if (ctx->nranks > 1 && !ctx->dbg_skip_exchange) {  // AllGather of the per-cell partials, in place
        size_t id = (size_t)-1;
        if ((st = span_begin(ctx, t, 3, ctx->stream, &id))) return st;
        std::string emsg;
        if (nccl_shim_allgather(ctx->nccl_comm, ctx->Sall + (int64_t)ctx->rank * ncl, ctx->Sall, (size_t)ncl,
                                ctx->stream, &emsg))
          return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
        if ((st = span_end(ctx, t, ctx->stream, id))) return st;
      }
      if ((st = band_newton_launch(ctx, t))) return st;
      if (t) ctx->timing_used++;
      ctx->cur = 1 - ctx->cur;
      ctx->steps_done++;
    }
    return sync_check(ctx);
  }
  if (ctx->implicit) {  // reading R-n
    ctx->imp_iters.clear();
    for (int64_t s = 0; s < nsteps; ++s) {
      const bool t = ctx->timing && ctx->timing_used < ctx->timing_max;
      if ((st = implicit_step(ctx, t))) return st;
      if (t) ctx->timing_used++;
      ctx->cur = 1 - ctx->cur;
      ctx->steps_done++;
    }
    return sync_check(ctx);
  }
  for (int64_t s = 0; s < nsteps; ++s) {
    const bool t = ctx->timing && ctx->timing_used < ctx->timing_max;
    // graph replay for repeated steps of a single two-buffer context (the
    // rotated layout changes its slot map every step; groups exchange halos)
    const bool graph = ctx->use_graph && nsteps > 1 && !t && ctx->nranks == 1 && !ctx->rot && !ctx->band;
    if (graph) {
      if ((st = graph_step(ctx))) return st;
      ctx->cur = 1 - ctx->cur;
      ctx->steps_done++;
      continue;
    }
    ctx->prefetch_bnd = s + 1 < nsteps;
    st = step_launch(ctx, t, ctx->nranks > 1 && ctx->overlap);
    ctx->prefetch_bnd = 0;
    if (st) {
      if (ctx->bnd_ready) {  // keep the stream order simple after an error
        cudaStreamWaitEvent(ctx->stream, ctx->ev_side, 0);
        ctx->bnd_ready = false;
      }
      return st;
    }
    if (ctx->nranks > 1) {
      // a5 on the comm stream once the boundary planes are swept; the next
      // step's sweeps wait for it (the wait sits after this step's Newton)
      CU(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_bnd, 0));
      size_t id = (size_t)-1;
      nvtx_push("a5 halo exchange");
      if ((st = span_begin(ctx, t, 3, ctx->comm_stream, &id))) return st;
      if ((st = ctx->umesh ? uhalo_exchange(ctx, ctx->I[1 - ctx->cur], ctx->comm_stream)
                           : halo_exchange(ctx, ctx->I[1 - ctx->cur], ctx->comm_stream)))
        return st;
      if ((st = span_end(ctx, t, ctx->comm_stream, id))) return st;
      nvtx_pop();
      CU(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
      CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    }
    if (t) ctx->timing_used++;
    ctx->cur = 1 - ctx->cur;
    ctx->steps_done++;
  }
  if (ctx->d_stats) {
    unsigned long long h[4];
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(h, ctx->d_stats, sizeof h, cudaMemcpyDeviceToHost));
    fprintf(stderr, "[bte] Newton stats after %lld steps: evaluations %llu, final re-evaluations %llu, cells solved %llu\n",
            (long long)ctx->steps_done, h[0], h[1], h[2]);
  }
  return sync_check(ctx);
}

// Local-mode halo exchange of a whole group on buffers I[which] of every
// context: each sender copies its owned boundary planes straight into the
// receiver's halo planes (the receives of the plan are implied), after both
// sides' previous work, and the receivers wait for those copies.
// Priming exchange of a local group on the current buffers (before the first
// step of a bte_group_step call): senders copy owned planes into halos.
static bte_status group_exchange(bte_ctx **ctxs, int n, bool output_buffers) {
  bte_ctx *ctx = ctxs[0];
  if (ctxs[0]->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  std::vector<cudaEvent_t> done(n), put(n);
  for (int r = 0; r < n; ++r) {
    CU(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&put[r], cudaEventDisableTiming));
    CU(cudaEventRecord(done[r], ctxs[r]->stream));
  }
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    const Geometry &g = c->g;
    double *src = c->I[output_buffers ? 1 - c->cur : c->cur];
    for (int k = 0; k < c->plan.n_msgs; ++k) {
      const bte_msg &m = c->plan.msg[k];
      if (!m.send) continue;
      bte_ctx *q = ctxs[m.peer];
      CU(cudaStreamWaitEvent(c->stream, done[m.peer], 0));
      double *dst = q->I[output_buffers ? 1 - q->cur : q->cur];
      const double *sp = src + g.slot_off[m.slot] + (m.plane - g.m0 + g.plane_off) * g.plane_stride;
      double *dp = dst + q->g.slot_off[m.slot] + (m.plane - q->g.m0 + q->g.plane_off) * q->g.plane_stride;
      CU(cudaMemcpyAsync(dp, sp, (size_t)m.count * sizeof(double), cudaMemcpyDefault, c->stream));
    }
    CU(cudaEventRecord(put[r], c->stream));
  }
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    for (int k = 0; k < c->plan.n_msgs; ++k)
      if (!c->plan.msg[k].send) CU(cudaStreamWaitEvent(c->stream, put[c->plan.msg[k].peer], 0));
  }
  for (int r = 0; r < n; ++r) {
    cudaEventDestroy(done[r]);
    cudaEventDestroy(put[r]);
  }
  return BTE_OK;
}

// Per-step local exchange, overlapped: on each sender's comm stream, once the
// sender's boundary planes and the receiver's previous step are done (both
// ev_bnd), copy the planes into the receiver's halo; each receiver's compute
// stream waits for its senders' copies after this step's Newton.
static bte_status group_exchange_overlap(bte_ctx **ctxs, int n) {
  if (ctxs[0]->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  bte_ctx *ctx = ctxs[0];
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    const Geometry &g = c->g;
    CU(cudaStreamWaitEvent(c->comm_stream, c->ev_bnd, 0));
    const double *src = c->I[1 - c->cur];
    for (int k = 0; k < c->plan.n_msgs; ++k) {
      const bte_msg &m = c->plan.msg[k];
      if (!m.send) continue;
      bte_ctx *q = ctxs[m.peer];
      CU(cudaStreamWaitEvent(c->comm_stream, q->ev_bnd, 0));
      double *dst = q->I[1 - q->cur];
      const double *sp = src + g.slot_off[m.slot] + (m.plane - g.m0 + g.plane_off) * g.plane_stride;
      double *dp = dst + q->g.slot_off[m.slot] + (m.plane - q->g.m0 + q->g.plane_off) * q->g.plane_stride;
      CU(cudaMemcpyAsync(dp, sp, (size_t)m.count * sizeof(double), cudaMemcpyDefault, c->comm_stream));
    }
    CU(cudaEventRecord(c->ev_halo, c->comm_stream));
  }
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    for (int k = 0; k < c->plan.n_msgs; ++k)
      if (!c->plan.msg[k].send) CU(cudaStreamWaitEvent(c->stream, ctxs[c->plan.msg[k].peer]->ev_halo, 0));
  }
  return BTE_OK;
}

// Local-mode band exchange: every part's row of Sall is copied into the same
// row of every other part's Sall, after the receiver's previous Newton (which
// read its Sall) and the sender's partial.
static bte_status band_exchange(bte_ctx **ctxs, int n) {
  bte_ctx *ctx = ctxs[0];
  if (ctxs[0]->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  const int64_t ncl = ctx->ncells_local;
  std::vector<cudaEvent_t> done(n), put(n);
  for (int r = 0; r < n; ++r) {
    CU(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&put[r], cudaEventDisableTiming));
    CU(cudaEventRecord(done[r], ctxs[r]->stream));
  }
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      CU(cudaStreamWaitEvent(c->stream, done[q], 0));
      CU(cudaMemcpyAsync(ctxs[q]->Sall + r * ncl, c->Sall + r * ncl, (size_t)ncl * sizeof(double),
                         cudaMemcpyDefault, c->stream));
    }
    CU(cudaEventRecord(put[r], c->stream));
  }
  for (int q = 0; q < n; ++q)
    for (int r = 0; r < n; ++r)
      if (r != q) CU(cudaStreamWaitEvent(ctxs[q]->stream, put[r], 0));
  for (int r = 0; r < n; ++r) {
    cudaEventDestroy(done[r]);
    cudaEventDestroy(put[r]);
  }
  return BTE_OK;
}

// ---- partitioned unstructured meshes: halo cells
// Where peer q's cells sit in my halo: block position n_own + recv_off of every slot region.
static double *uhalo_dst(bte_ctx *q, double *Ibuf, int slot, int64_t recv_off) {
  return Ibuf + q->g.slot_off[slot] + (q->ncells_local + recv_off) * (int64_t)q->g.Es;
}

// In-process group: every rank packs the cells its peers hold as halo copies
// (buffer `output` ? I[1-cur] : I[cur]) once its step is done, then copies each
// peer's segment slot by slot into the peer's halo blocks; receivers wait.
static bte_status ugroup_exchange(bte_ctx **ctxs, int n, bool output) {
  bte_ctx *ctx = ctxs[0];
  if (ctxs[0]->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  std::vector<cudaEvent_t> done(n), put(n);
  for (int r = 0; r < n; ++r) {
    CU(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&put[r], cudaEventDisableTiming));
    CU(cudaEventRecord(done[r], ctxs[r]->stream));
  }
  for (int r = 0; r < n; ++r) {
    bte_ctx *c = ctxs[r];
    const Geometry &g = c->g;
    const double *src = c->I[output ? 1 - c->cur : c->cur];
    int64_t off = 0;
    for (size_t k = 0; k < c->upeers.size(); ++k) {
      const UPeer &pe = c->upeers[k];
      const int64_t cnt = (int64_t)pe.send_cells.size();
      if (cnt == 0) continue;
      bte_ctx *q = ctxs[pe.peer];
      double *seg = c->d_usendbuf + off * g.nslot * g.Es;
      CU(launch_pack_cells(g, c->d_usend[k], cnt, src, seg, c->stream));
      CU(cudaStreamWaitEvent(c->stream, done[pe.peer], 0));
      // where q keeps my cells
      int64_t roff = -1;
      for (const UPeer &qe : q->upeers)
        if (qe.peer == r) roff = qe.recv_off;
      if (roff < 0) return fail(ctx, BTE_EINVAL, "inconsistent unstructured halo plan (rank %d -> %d)", r, pe.peer);
      double *dstb = q->I[output ? 1 - q->cur : q->cur];
      for (int sl = 0; sl < g.nslot; ++sl)
        CU(cudaMemcpyAsync(uhalo_dst(q, dstb, sl, roff), seg + (int64_t)sl * cnt * g.Es,
                           (size_t)cnt * g.Es * sizeof(double), cudaMemcpyDefault, c->stream));
      off += cnt;
    }
    CU(cudaEventRecord(put[r], c->stream));
  }
  for (int r = 0; r < n; ++r)
    for (const UPeer &pe : ctxs[r]->upeers)
      if (pe.recv_cnt) CU(cudaStreamWaitEvent(ctxs[r]->stream, put[pe.peer], 0));
  for (int r = 0; r < n; ++r) {
    cudaEventDestroy(done[r]);
    cudaEventDestroy(put[r]);
  }
  return BTE_OK;
}

// NCCL: pack, grouped send/recv of the packed segments, scatter into the halo.
static bte_status uhalo_exchange(bte_ctx *ctx, double *Ibuf, cudaStream_t stream) {
  if (ctx->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  const Geometry &g = ctx->g;
  if (!stream) stream = ctx->stream;
  std::string emsg;
  int64_t soff = 0;
  for (size_t k = 0; k < ctx->upeers.size(); ++k) {
    const int64_t cnt = (int64_t)ctx->upeers[k].send_cells.size();
    CU(launch_pack_cells(g, ctx->d_usend[k], cnt, Ibuf, ctx->d_usendbuf + soff * g.nslot * g.Es, stream));
    soff += cnt;
  }
  if (nccl_shim_group_start(&emsg)) return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
  soff = 0;
  int64_t roff = 0;
  for (const UPeer &pe : ctx->upeers) {
    const int64_t cnt = (int64_t)pe.send_cells.size();
    if (cnt && nccl_shim_send(ctx->nccl_comm, ctx->d_usendbuf + soff * g.nslot * g.Es, (size_t)(cnt * g.nslot * g.Es),
                              pe.peer, stream, &emsg))
      return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
    if (pe.recv_cnt && nccl_shim_recv(ctx->nccl_comm, ctx->d_urecvbuf + roff * g.nslot * g.Es,
                                      (size_t)(pe.recv_cnt * g.nslot * g.Es), pe.peer, stream, &emsg))
      return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
    soff += cnt;
    roff += pe.recv_cnt;
  }
  if (nccl_shim_group_end(&emsg)) return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
  roff = 0;
  for (const UPeer &pe : ctx->upeers) {
    for (int sl = 0; sl < g.nslot && pe.recv_cnt; ++sl)
      CU(cudaMemcpyAsync(uhalo_dst(ctx, Ibuf, sl, pe.recv_off), ctx->d_urecvbuf + (roff * g.nslot + sl * pe.recv_cnt) * g.Es,
                         (size_t)pe.recv_cnt * g.Es * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    roff += pe.recv_cnt;
  }
  return BTE_OK;
}

bte_status bte_group_step(bte_ctx **ctxs, int n, int64_t nsteps) {
  if (!ctxs || n < 1 || nsteps < 0) return BTE_EINVAL;
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r]) return BTE_EINVAL;
    if (ctxs[r]->rank != r || ctxs[r]->nranks != n || ctxs[r]->nccl_comm)
      return fail(ctxs[r], BTE_EINVAL, "bte_group_step: ctxs[%d] must be local-mode rank %d of %d", r, r, n);
    if (ctxs[r]->steps_done != ctxs[0]->steps_done)
      return fail(ctxs[r], BTE_EINVAL, "bte_group_step: contexts are at different steps");
    if (ctxs[r]->band != ctxs[0]->band || (ctxs[0]->band && ctxs[r]->ncells_local != ctxs[0]->ncells_local))
      return fail(ctxs[r], BTE_EINVAL, "bte_group_step: mixed band/slab contexts or different meshes");
  }
  bte_status st;
  if (ctxs[0]->band) {
    for (int64_t s = 0; s < nsteps; ++s) {
      for (int r = 0; r < n; ++r) {
        const bool t = ctxs[r]->timing && ctxs[r]->timing_used < ctxs[r]->timing_max;
        if ((st = band_sweep_launch(ctxs[r], t))) return st;
      }
      if (n > 1 && (st = band_exchange(ctxs, n))) return st;
      for (int r = 0; r < n; ++r) {
        bte_ctx *c = ctxs[r];
        const bool t = c->timing && c->timing_used < c->timing_max;
        if ((st = band_newton_launch(c, t))) return st;
        if (t) c->timing_used++;
        c->cur = 1 - c->cur;
        c->steps_done++;
      }
    }
    for (int r = 0; r < n; ++r)
      if ((st = sync_check(ctxs[r]))) return st;
    return BTE_OK;
  }
  const bool um = ctxs[0]->umesh;
  if (n > 1 && (st = um ? ugroup_exchange(ctxs, n, false) : group_exchange(ctxs, n, false)))
    return st;  // prime halos from the current state
  for (int64_t s = 0; s < nsteps; ++s) {
    for (int r = 0; r < n; ++r) {
      const bool t = ctxs[r]->timing && ctxs[r]->timing_used < ctxs[r]->timing_max;
      if ((st = step_launch(ctxs[r], t, n > 1 && ctxs[r]->overlap))) return st;
    }
    if (n > 1 && (st = um ? ugroup_exchange(ctxs, n, true) : group_exchange_overlap(ctxs, n))) return st;
    for (int r = 0; r < n; ++r) {
      bte_ctx *c = ctxs[r];
      if (c->timing && c->timing_used < c->timing_max) c->timing_used++;
      c->cur = 1 - c->cur;
      c->steps_done++;
    }
  }
  for (int r = 0; r < n; ++r)
    if ((st = sync_check(ctxs[r]))) return st;
  return BTE_OK;
}

static bte_status halo_exchange(bte_ctx *ctx, double *Ibuf, cudaStream_t stream) {
  // a5: execute this rank's halo plan (bte_plan_slab) as one NCCL group on
  // `stream` (default: the context stream); plane p (global) lives at local
  // index p - m0 + plane_off.
  if (ctx->dbg_skip_exchange) return BTE_OK;  // mutation tests (bte_set_debug)
  const Geometry &g = ctx->g;
  if (!stream) stream = ctx->stream;
  std::string emsg;
  if (nccl_shim_group_start(&emsg)) return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
  for (int k = 0; k < ctx->plan.n_msgs; ++k) {
    const bte_msg &m = ctx->plan.msg[k];
    double *ptr = Ibuf + g.slot_off[m.slot] + (m.plane - g.m0 + g.plane_off) * g.plane_stride;
    const int rc = m.send ? nccl_shim_send(ctx->nccl_comm, ptr, (size_t)m.count, m.peer, stream, &emsg)
                          : nccl_shim_recv(ctx->nccl_comm, ptr, (size_t)m.count, m.peer, stream, &emsg);
    if (rc) return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
  }
  if (nccl_shim_group_end(&emsg)) return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
  return BTE_OK;
}

bte_status bte_get_intensity(bte_ctx *ctx, double *out, size_t count) {
  if (!ctx || !out) return BTE_EINVAL;
  if (count != (size_t)ctx->ncells_local * ctx->nd * ctx->nb)
    return fail(ctx, BTE_EINVAL, "intensity count %zu != %lld", count,
                (long long)(ctx->ncells_local * ctx->nd * ctx->nb));
  return transfer_I(ctx, out, 0);
}

bte_status bte_get_intensity_cells(bte_ctx *ctx, const int64_t *cells, int64_t n, double *out) {
  if (!ctx || (n > 0 && (!cells || !out)) || n < 0) return BTE_EINVAL;
  for (int64_t k = 0; k < n; ++k)
    if (cells[k] < 0 || cells[k] >= ctx->ncells_local)
      return fail(ctx, BTE_EINVAL, "cell index %lld out of range", (long long)cells[k]);
  const int64_t per_cell = (int64_t)ctx->nd * ctx->nb;
  // staging holds staging_cells * per_cell doubles: the index list goes at its
  // end (8 B per cell), the gathered rows at its start
  const int64_t chunk = std::max<int64_t>(1, (ctx->staging_cells * per_cell) / (per_cell + 1));
  for (int64_t k0 = 0; k0 < n; k0 += chunk) {
    const int64_t m = std::min(chunk, n - k0);
    int64_t *d_idx = reinterpret_cast<int64_t *>(ctx->staging + ctx->staging_cells * per_cell) - m;
    CU(cudaMemcpyAsync(d_idx, cells + k0, m * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    CU(launch_gather_cells(ctx->g, ctx->d_dmap, ctx->nd, d_idx, m, ctx->I[ctx->cur], ctx->staging, ctx->stream));
    CU(cudaMemcpyAsync(out + k0 * per_cell, ctx->staging, m * per_cell * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return BTE_OK;
}

bte_status bte_get_temperature(bte_ctx *ctx, double *out, size_t count) {
  if (!ctx || !out) return BTE_EINVAL;
  if (count != (size_t)ctx->ncells_local) return fail(ctx, BTE_EINVAL, "temperature count mismatch");
  CU(cudaMemcpyAsync(out, ctx->T, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return BTE_OK;
}

bte_status bte_get_energy(bte_ctx *ctx, double *E) {
  if (!ctx || !E) return BTE_EINVAL;
  const int64_t ncl = ctx->ncells_local;
  if (!ctx->d_energy) {  // per-cell energies [ncl] + the gathered rank sums [nranks], kept for later calls
    ctx->d_energy = (double *)dev_alloc(ctx, (size_t)(ncl + ctx->nranks) * sizeof(double));
    if (!ctx->d_energy) return fail(ctx, BTE_ENOMEM, "energy buffer allocation failed");
  }
  CU(launch_energy(ctx->g, ctx->I[ctx->cur], ctx->m.v, ctx->d_energy, ctx->stream));
  std::vector<double> h(ncl);
  CU(cudaMemcpyAsync(h.data(), ctx->d_energy, ncl * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  const bte_mesh &m = ctx->mesh;
  const double V = ctx->umesh ? 1.0 : m.dx * m.dy * m.dz;
  if (ctx->umesh)
    for (int64_t c = 0; c < ncl; ++c) h[c] *= ctx->uvol[c];
  double s = 0, comp = 0;  // Kahan
  for (double x : h) {
    const double y = x - comp;
    const double t = s + y;
    comp = (t - s) - y;
    s = t;
  }
  double e = V * s;
  if (ctx->nccl_comm) {
    // all ranks' partial sums (AllGather), added in rank order: the same total,
    // bit for bit, on every rank (an AllReduce does not fix its order)
    double *d_all = ctx->d_energy + ncl;
    CU(cudaMemcpyAsync(d_all + ctx->rank, &e, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    std::string emsg;
    if (nccl_shim_allgather(ctx->nccl_comm, d_all + ctx->rank, d_all, 1, ctx->stream, &emsg))
      return fail(ctx, BTE_ENCCL, "%s", emsg.c_str());
    std::vector<double> parts(ctx->nranks);
    CU(cudaMemcpyAsync(parts.data(), d_all, ctx->nranks * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    e = 0.0;
    for (double x : parts) e += x;
  }
  *E = e;
  return BTE_OK;
}

bte_status bte_set_debug(bte_ctx *ctx, int what, int value) {
  if (!ctx) return BTE_EINVAL;
  if (what != BTE_DEBUG_SKIP_EXCHANGE) return fail(ctx, BTE_EINVAL, "unknown debug switch %d", what);
  ctx->dbg_skip_exchange = value != 0;
  return BTE_OK;
}

bte_status bte_debug_substep(bte_ctx *ctx, int which, double *out, size_t count) {
  if (!ctx || !out) return BTE_EINVAL;
  const int64_t ncl = ctx->ncells_local;
  bte_status st;
  if (which == 2 || which == 3) {
    if (count != (size_t)(ncl * ctx->nbT)) return fail(ctx, BTE_EINVAL, "count mismatch");
    CU(cudaMemcpy(out, which == 2 ? ctx->I0c : ctx->beta, count * sizeof(double), cudaMemcpyDeviceToHost));
    return BTE_OK;
  }
  if (which != 0 && which != 1) return fail(ctx, BTE_EINVAL, "which must be 0..3");
  if (ctx->rot) return fail(ctx, BTE_EINVAL, "sub-step 0/1 would overwrite the state under octant-slot rotation");
  const size_t want = which == 0 ? (size_t)ncl * ctx->nd * ctx->nb : (size_t)ncl * ctx->nb;
  if (count != want) return fail(ctx, BTE_EINVAL, "count mismatch");
  double *Iin = ctx->I[ctx->cur];
  double *Iout = ctx->I[1 - ctx->cur];
  if (n_diffuse(ctx) && (st = launch_boundary(ctx, Iin))) return st;
  if ((st = launch_sweep_step(ctx, Iin, Iout))) return st;
  if (which == 0) {
    ctx->cur = 1 - ctx->cur;  // read the swept buffer, then restore
    st = transfer_I(ctx, out, 0);
    ctx->cur = 1 - ctx->cur;
    return st;
  }
  double *d_D = nullptr;
  CU(cudaMalloc(&d_D, want * sizeof(double)));
  CU(launch_octant_tree_g(ctx->g, ctx->Dpart, ncl, d_D, ctx->stream));
  CU(cudaMemcpyAsync(out, d_D, want * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaFree(d_D));
  return BTE_OK;
}

bte_status bte_timing_enable(bte_ctx *ctx, int enable, int64_t max_steps) {
  if (!ctx) return BTE_EINVAL;
  CU(cudaStreamSynchronize(ctx->stream));
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  ctx->ev.clear();
  ctx->spans.clear();
  ctx->ev_used = 0;
  ctx->tacc = bte_timing{};
  ctx->timing = enable != 0;
  ctx->timing_used = 0;
  ctx->timing_max = enable ? max_steps : 0;
  if (enable) {
    // spans per step at most: boundary, 2 sweeps (split), Newton, relax, halo;
    // implicit (R-n): boundary + sweep + Newton per iteration
    const int64_t per_step = ctx->implicit ? 2 * (3 * (int64_t)ctx->imp_max_iter) : 2 * 6;
    ctx->ev.resize((size_t)(per_step * max_steps));
    for (auto &e : ctx->ev) CU(cudaEventCreate(&e));
  }
  return BTE_OK;
}

bte_status bte_timing_read(bte_ctx *ctx, bte_timing *out) {
  if (!ctx || !out) return BTE_EINVAL;
  CU(cudaStreamSynchronize(ctx->stream));
  bte_timing t = ctx->tacc;
  t.steps = ctx->timing_used;
  t.sweep_ms = t.newton_ms = t.boundary_ms = t.halo_ms = 0;
  for (const auto &sp : ctx->spans) {
    float ms;
    CU(cudaEventElapsedTime(&ms, ctx->ev[sp.second], ctx->ev[sp.second + 1]));
    double *dst = sp.first == 0 ? &t.sweep_ms : sp.first == 1 ? &t.newton_ms : sp.first == 2 ? &t.boundary_ms : &t.halo_ms;
    *dst += ms;
  }
  *out = t;
  return BTE_OK;
}

bte_status bte_get_info(const bte_ctx *ctx, bte_info *out) {
  if (!ctx || !out) return BTE_EINVAL;
  out->ncells_local = ctx->ncells_local;
  out->ncells_global = ctx->ncells_global;
  out->z0 = ctx->g.m0;
  out->nz_local = ctx->g.nplanes;
  out->nd = ctx->nd;
  out->nb = ctx->nb;
  out->n_octants = ctx->g.nslot;
  out->nj = ctx->g.nj;
  out->bytes_state = ctx->bytes;
  out->b0 = ctx->b0;
  out->b1 = ctx->b0 + ctx->nb;
  out->nb_total = ctx->nbT;
  out->band = ctx->band;
  out->rotate = ctx->rot;
  out->cell0 = ctx->g.cell0;
  out->step_mode = ctx->implicit ? 2 : ctx->semi ? 1 : 0;
  out->newton_kernel = ctx->band ? "k_newton (warp per cell, band partials)"
                       : ctx->tau_mode == 1 ? (ctx->mF.uniform && !ctx->sc_direct ? "k_newton_scu (self-consistent tau)"
                                                                                  : "k_newton_sc (self-consistent tau)")
                                            : "k_newton (warp per cell)";
  if (ctx->umesh) {
    out->sweep_kernel = "k_usweep_tma (face-list upwind flux + relaxation on m-sided cells)";
  } else {
    SweepArgs a = sweep_args(ctx, ctx->I[0], ctx->I[1], 0, 0, 0);
    out->sweep_kernel = ctx->implicit ? "k_sweep_imp (implicit wavefront sweep, reading R-n)" : sweep_kernel_name(a);
  }
  return BTE_OK;
}

void bte_destroy(bte_ctx *ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  graph_invalidate(ctx);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
  }
  if (ctx->ev_swept) cudaEventDestroy(ctx->ev_swept);
  if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  if (ctx->ev_bnd) cudaEventDestroy(ctx->ev_bnd);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
  if (ctx->nccl_comm) nccl_shim_destroy(ctx->nccl_comm);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  for (void *p : ctx->allocs) {
    if (ctx->dealloc)
      ctx->dealloc(p, ctx->alloc_ctx);
    else
      cudaFree(p);
  }
  delete ctx;
}

}  // extern "C"
