/*
 * bte_oracle.c -- plain, slow, fp64 CPU ORACLE for the explicit finite-volume
 * phonon-BTE time step of arXiv 2305.19400.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no source with the CUDA path (paper_2305_19400_b200/csrc) and
 * includes none of its headers.
 *
 * Citations: P:L<a>-<b> = /root/reference/PAPER.md; S:L = SPEC.md;
 * "reading #n" = DESIGN.md section "Readings of the paper".
 *
 *   Eq. 4  dI/dt + v_g . grad I = (I0 - I)/tau
 *   Eq. 5  FV form: volume relaxation - |v_g|_b * surface integral
 *                        of I_{d,b} s_d . n  (first-order upwind, P:L150-157,
 *                        P:L476-479)
 *   Eqs. 2-3 forward Euler, cell-average discretisation
 *   Eq. 6  ghost intensities: I0_b at isothermal, I_{r,b} at
 *                        symmetric walls; diffuse-adiabatic walls per reading #11
 *   temperature update, readings #2,#14,
 *                        #15,#18: deviation-form reduction + Newton.
 *
 * Layout: canonical I[(c*nd + d)*nb + b], c = x + nx*(y + ny*z).
 * Loop nest: cell -> direction -> band.
 * Build: gcc -O2 -ffp-contract=off -fopenmp (no fast-math): every cell's
 * arithmetic is in a fixed order, so results do not depend on thread count.
 *
 * parity pins: see tests/test_oracle_pins.py (all functions pinned; the
 * silicon material constants themselves are paper-silent data -- "parity
 * unpinned" applies only to the physical realism of those constants, not to
 * any function here).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_OK 0
#define ORA_EINVAL 1
#define ORA_ENOMEM 2
#define ORA_ENOTCLOSED 6
#define ORA_ENEWTON 7
#define ORA_ENONFINITE 8

#define BC_ISO 0
#define BC_SPEC 1
#define BC_DIFF 2
#define BC_PART 3 /* partially specular (reading R-i) */

#define HBAR 1.054571817e-34
#define KB 1.380649e-23
#define NGL 16
#define T_LO 1.0
#define T_HI 5000.0
#define NEWTON_MAXIT 50
#define NEWTON_RTOL 1e-13

typedef struct {
  int dim;
  long nx, ny, nz;
  double dx, dy, dz;
  int nd;
  const double *s; /* [nd][3] */
  const double *w; /* [nd] */
  int nb;
  const double *v; /* [nb] */
  int mode;        /* 0 linear, 1 Bose-Einstein */
  const double *I_ref, *slope;
  double T_ref;
  const double *w_lo, *w_hi, *vs, *c2, *g;
  const double *beta_coef; /* [nb][5] */
  double dt;
  int bc_kind[6];
  const double *T_wall[6]; /* per face or NULL */
  double T_uniform[6];
  int nthreads;
  double specularity[6]; /* BC_PART: fraction p of specular reflection */
  int tau_mode;          /* 0: lagged tau (reading #15); 1: self-consistent tau(T^{n+1}) (reading R-k) */
  int semi;              /* 1: semi-implicit step, implicit relaxation (reading R-l) */
  int implicit;          /* 1: implicit step solved by source iteration (reading R-n) */
  int imp_max_iter;      /* R-n: iterations per step (the count when imp_tol == 0) */
  double imp_tol;        /* R-n: stop when max_c |T^{k+1} - T^k| <= imp_tol * T^k (0: fixed count) */
} ora_problem;

/* ---------------------------------------------------------------- quadrature */

/* Gauss-Legendre nodes/weights on [-1,1], ascending nodes: Newton iteration on
 * the three-term Legendre recurrence (textbook construction). */
void ora_gauss_legendre(int n, double *x, double *wt) {
  for (int i = 0; i < n; i++) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5));
    double p1 = 0, p0 = 0, dp = 0;
    for (int it = 0; it < 100; it++) {
      p0 = 1.0;
      p1 = z;
      for (int k = 2; k <= n; k++) {
        double pk = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = pk;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (fabs(dz) < 1e-17) break;
    }
    p0 = 1.0;
    p1 = z;
    for (int k = 2; k <= n; k++) {
      double pk = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = pk;
    }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    /* cos(...) runs from ~1 downward: store ascending */
    x[n - 1 - i] = z;
    wt[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

static double GLX[NGL], GLW[NGL];
static int gl_ready = 0;
static void gl_init(void) {
  if (!gl_ready) {
    ora_gauss_legendre(NGL, GLX, GLW);
    gl_ready = 1;
  }
}

/* ------------------------------------------------------------ material model */

/* wavenumber on the quadratic dispersion omega = vs*k + c2*k^2 (reading #1):
 * k = (-vs + sqrt(vs^2 + 4 c2 w)) / (2 c2), written in the algebraically equal
 * rationalised form 2w / (vs + sqrt(vs^2 + 4 c2 w)) to avoid cancellation. */
static double k_of_omega(double vs, double c2, double w) {
  if (c2 == 0.0) return w / vs;
  return 2.0 * w / (vs + sqrt(vs * vs + 4.0 * c2 * w));
}

/* Equilibrium intensity of channel b at temperature T and its T-derivative.
 * LINEAR: I_ref + a (T - T_ref).
 * BOSE_EINSTEIN (reading #1): g hbar/(8 pi^3) int_{wlo}^{whi} w k(w)^2 /
 *   (exp(hbar w / kB T) - 1) dw with 16-point Gauss-Legendre;
 *   dI0/dT integrand = integrand * (x/T) * e^x/(e^x - 1), x = hbar w/(kB T). */
double ora_I0(const ora_problem *p, int b, double T, double *dI0dT) {
  if (p->mode == 0) {
    if (dI0dT) *dI0dT = p->slope[b];
    return p->I_ref[b] + p->slope[b] * (T - p->T_ref);
  }
  gl_init();
  double half = 0.5 * (p->w_hi[b] - p->w_lo[b]);
  double mid = 0.5 * (p->w_hi[b] + p->w_lo[b]);
  double sum = 0.0, dsum = 0.0;
  for (int j = 0; j < NGL; j++) {
    double w = mid + half * GLX[j];
    double k = k_of_omega(p->vs[b], p->c2[b], w);
    double x = HBAR * w / (KB * T);
    double em1 = expm1(x);
    double f = w * k * k / em1;
    sum += GLW[j] * f;
    dsum += GLW[j] * (f * (x / T) * (1.0 + 1.0 / em1));
  }
  double pref = p->g[b] * HBAR / (8.0 * M_PI * M_PI * M_PI) * half;
  if (dI0dT) *dI0dT = pref * dsum;
  return pref * sum;
}

/* inverse relaxation time beta_b(T) = 1/tau_b(T) (readings #3, #15) */
double ora_beta(const ora_problem *p, int b, double T) {
  const double *q = p->beta_coef + 5 * b;
  double r = q[0] + q[1] * T * T * T + q[2] * T * T * T * T;
  if (q[3] != 0.0) r += q[3] / sinh(q[4] / T);
  return r;
}

/* d beta_b / dT of the expression above, term by term:
 * 3 p3 T^2 + 4 p4 T^3 + pu theta cosh(theta/T) / (T^2 sinh^2(theta/T)) */
double ora_dbeta(const ora_problem *p, int b, double T) {
  const double *q = p->beta_coef + 5 * b;
  double r = 3.0 * q[1] * T * T + 4.0 * q[2] * T * T * T;
  if (q[3] != 0.0) {
    double x = q[4] / T, sh = sinh(x);
    r += q[3] * q[4] * cosh(x) / (T * T * sh * sh);
  }
  return r;
}

/* ---------------------------------------------------------------- directions */

int ora_octant(const double *s) {
  return (s[0] < 0.0 ? 4 : 0) | (s[1] < 0.0 ? 2 : 0) | (s[2] < 0.0 ? 1 : 0);
}

/* r_axis(d): the direction whose vector equals s_d with component `axis`
 * negated, bit-exactly ("r is the direction vector index
 * corresponding to a reflection"). Returns 0, or ORA_ENOTCLOSED. */
int ora_reflection(const ora_problem *p, int axis, int *r) {
  for (int d = 0; d < p->nd; d++) {
    double t[3] = {p->s[3 * d], p->s[3 * d + 1], p->s[3 * d + 2]};
    t[axis] = -t[axis];
    r[d] = -1;
    for (int e = 0; e < p->nd; e++) {
      if (p->s[3 * e] == t[0] && p->s[3 * e + 1] == t[1] && p->s[3 * e + 2] == t[2] &&
          p->w[e] == p->w[d]) {
        r[d] = e;
        break;
      }
    }
    if (r[d] < 0) return ORA_ENOTCLOSED;
  }
  return ORA_OK;
}

static double octant_tree(const double *q) {
  return ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
}

/* ---------------------------------------------------------------- geometry */

static long n_axis(const ora_problem *p, int a) { return a == 0 ? p->nx : (a == 1 ? p->ny : p->nz); }
static double d_axis(const ora_problem *p, int a) { return a == 0 ? p->dx : (a == 1 ? p->dy : p->dz); }

static long face_index(const ora_problem *p, int axis, long x, long y, long z) {
  if (axis == 0) return y + p->ny * z;
  if (axis == 1) return x + p->nx * z;
  return x + p->nx * y;
}

long ora_n_faces(const ora_problem *p, int region) {
  int a = region / 2;
  if (a == 0) return p->ny * p->nz;
  if (a == 1) return p->nx * p->nz;
  return p->nx * p->ny;
}

/* Largest admissible explicit step check (reading #9): returns
 * min over (d,b) of 1 - dt*beta_b(Tmax) - dt*v_b*sum_a |s_da|/D_a. */
double ora_dt_margin(const ora_problem *p, double Tmax) {
  double m = 1e300;
  int na = p->dim == 3 ? 3 : 2;
  for (int b = 0; b < p->nb; b++) {
    double be = ora_beta(p, b, Tmax);
    for (int d = 0; d < p->nd; d++) {
      double k = 0.0;
      for (int a = 0; a < na; a++) k += fabs(p->s[3 * d + a]) / d_axis(p, a);
      double mm = 1.0 - (p->semi ? 0.0 : p->dt * be) - p->dt * p->v[b] * k;
      if (mm < m) m = mm;
    }
  }
  return m;
}

/* ---------------------------------------------------------------- state init */

/* I_{c,d,b} = I0_b(T_c) for all d ("initial(I, [I_init[b] ...])") */
void ora_equilibrium(const ora_problem *p, const double *T, double *I) {
  long nc = p->nx * p->ny * p->nz;
  int nd = p->nd, nb = p->nb;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1)
  for (long c = 0; c < nc; c++)
    for (int b = 0; b < nb; b++) {
      double i0 = ora_I0(p, b, T[c], NULL);
      for (int d = 0; d < nd; d++) I[(c * nd + d) * nb + b] = i0;
    }
}

/* I0c = I0(T), betac = beta(T) per cell/channel */
void ora_refresh(const ora_problem *p, const double *T, double *I0c, double *betac) {
  long nc = p->nx * p->ny * p->nz;
  for (long c = 0; c < nc; c++)
    for (int b = 0; b < p->nb; b++) {
      I0c[c * p->nb + b] = ora_I0(p, b, T[c], NULL);
      betac[c * p->nb + b] = ora_beta(p, b, T[c]);
    }
}

/* ------------------------------------------------------------ step pieces */

/* Isothermal ghost table g[f][b] = I0_b(T_wall(f)) (Eq. 6 first case) */
static void iso_table(const ora_problem *p, int region, double *g) {
  long nf = ora_n_faces(p, region);
  for (long f = 0; f < nf; f++) {
    double Tw = p->T_wall[region] ? p->T_wall[region][f] : p->T_uniform[region];
    for (int b = 0; b < p->nb; b++) g[f * p->nb + b] = ora_I0(p, b, Tw, NULL);
  }
}

/* Diffuse-adiabatic ghost (reading #11): for outward sign sg of the wall on
 * axis a, g_b = [sum over outgoing d' (sg*s_a > 0) of w|s_a| I_{d'}] /
 *               [sum over incoming d'' (sg*s_a < 0) of w|s_a|],
 * both sums within-octant ascending, then the octant sign-bit tree. */
static double diffuse_den(const ora_problem *p, int region) {
  int a = region / 2;
  double sg = (region & 1) ? 1.0 : -1.0;
  double q[8] = {0};
  for (int d = 0; d < p->nd; d++) {
    double sa = p->s[3 * d + a];
    if (sg * sa < 0.0) q[ora_octant(p->s + 3 * d)] += p->w[d] * fabs(sa);
  }
  return octant_tree(q);
}

static void diffuse_table(const ora_problem *p, int region, const double *I, double den, double *g) {
  int a = region / 2;
  double sg = (region & 1) ? 1.0 : -1.0;
  long n0 = p->nx, n1 = p->ny, n2 = p->nz;
  long nf = ora_n_faces(p, region);
  int nd = p->nd, nb = p->nb;
  for (long f = 0; f < nf; f++) {
    long x, y, z;
    /* cell adjacent to face f of this wall */
    if (a == 0) {
      y = f % n1; z = f / n1; x = (region & 1) ? n0 - 1 : 0;
    } else if (a == 1) {
      x = f % n0; z = f / n0; y = (region & 1) ? n1 - 1 : 0;
    } else {
      x = f % n0; y = f / n0; z = (region & 1) ? n2 - 1 : 0;
    }
    long c = x + n0 * (y + n1 * z);
    for (int b = 0; b < nb; b++) {
      double q[8] = {0};
      for (int d = 0; d < nd; d++) {
        double sa = p->s[3 * d + a];
        if (sg * sa > 0.0) q[ora_octant(p->s + 3 * d)] += p->w[d] * fabs(sa) * I[(c * nd + d) * nb + b];
      }
      g[f * nb + b] = octant_tree(q) / den;
    }
  }
}

typedef struct {
  double *giso[6];
  double *gdiff[6];
  double den[6];
  int *refl[3];
} ora_bcdata;

static int bc_prepare(const ora_problem *p, ora_bcdata *bd) {
  memset(bd, 0, sizeof(*bd));
  int nreg = p->dim == 3 ? 6 : 4;
  for (int a = 0; a < 3; a++) {
    bd->refl[a] = (int *)malloc(sizeof(int) * p->nd);
    if (!bd->refl[a]) return ORA_ENOMEM;
  }
  for (int r = 0; r < nreg; r++) {
    long nf = ora_n_faces(p, r);
    if (p->bc_kind[r] == BC_ISO) {
      bd->giso[r] = (double *)malloc(sizeof(double) * nf * p->nb);
      if (!bd->giso[r]) return ORA_ENOMEM;
      iso_table(p, r, bd->giso[r]);
    } else if (p->bc_kind[r] == BC_DIFF) {
      bd->gdiff[r] = (double *)malloc(sizeof(double) * nf * p->nb);
      if (!bd->gdiff[r]) return ORA_ENOMEM;
      bd->den[r] = diffuse_den(p, r);
      if (!(bd->den[r] > 0.0)) return ORA_EINVAL;
    } else if (p->bc_kind[r] == BC_SPEC) {
      if (ora_reflection(p, r / 2, bd->refl[r / 2]) != ORA_OK) return ORA_ENOTCLOSED;
    } else if (p->bc_kind[r] == BC_PART) {
      if (!(p->specularity[r] >= 0.0 && p->specularity[r] <= 1.0)) return ORA_EINVAL;
      if (ora_reflection(p, r / 2, bd->refl[r / 2]) != ORA_OK) return ORA_ENOTCLOSED;
      bd->gdiff[r] = (double *)malloc(sizeof(double) * nf * p->nb);
      if (!bd->gdiff[r]) return ORA_ENOMEM;
      bd->den[r] = diffuse_den(p, r);
      if (!(bd->den[r] > 0.0)) return ORA_EINVAL;
    } else {
      return ORA_EINVAL;
    }
  }
  return ORA_OK;
}

static void bc_free(ora_bcdata *bd) {
  for (int r = 0; r < 6; r++) {
    free(bd->giso[r]);
    free(bd->gdiff[r]);
  }
  for (int a = 0; a < 3; a++) free(bd->refl[a]);
}

/* upwind ghost for wall `region` at face f, cell c, direction d, channel b (Eq. 6) */
static double ghost(const ora_problem *p, const ora_bcdata *bd, int region, long f, long c, int d, int b,
                    const double *I) {
  int k = p->bc_kind[region];
  if (k == BC_ISO) return bd->giso[region][f * p->nb + b];
  if (k == BC_DIFF) return bd->gdiff[region][f * p->nb + b];
  double spec = I[(c * p->nd + bd->refl[region / 2][d]) * p->nb + b];
  if (k == BC_PART) {
    /* reading R-i: Ziman/Soffer specularity mixing of the two adiabatic ghosts */
    double sp = p->specularity[region];
    return sp * spec + (1.0 - sp) * bd->gdiff[region][f * p->nb + b];
  }
  return spec;
}

/* Sweep (Eq. 5 with forward Euler, Eqs. 2-3):
 *   I'_{c,d,b} = I + dt*( beta_c,b (I0c_c,b - I) - v_b * flux ),
 *   flux = sum over axes a (x, y, z order) of (|s_da|/D_a)(I_c - I_up_a),
 * the per-axis difference form of the face sum sum_f (A_f/V)(s.n_f) I_up
 * (upwind: I_up = I_c if s.n > 0, else the neighbour/ghost across f). */
void ora_sweep_bd(const ora_problem *p, const ora_bcdata *bd, const double *I, const double *I0c,
                  const double *betac, double *Iout) {
  long nx = p->nx, ny = p->ny, nz = p->nz;
  long nc = nx * ny * nz;
  int nd = p->nd, nb = p->nb;
  int na = p->dim == 3 ? 3 : 2;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1)
  for (long c = 0; c < nc; c++) {
    long ix[3] = {c % nx, (c / nx) % ny, c / (nx * ny)};
    long stride[3] = {1, nx, nx * ny};
    for (int d = 0; d < nd; d++) {
      for (int b = 0; b < nb; b++) {
        double Ic = I[(c * nd + d) * nb + b];
        double flux = 0.0;
        for (int a = 0; a < na; a++) {
          double sa = p->s[3 * d + a];
          double up;
          if (sa > 0.0) {
            if (ix[a] > 0)
              up = I[((c - stride[a]) * nd + d) * nb + b];
            else
              up = ghost(p, bd, 2 * a, face_index(p, a, ix[0], ix[1], ix[2]), c, d, b, I);
          } else if (sa < 0.0) {
            if (ix[a] < n_axis(p, a) - 1)
              up = I[((c + stride[a]) * nd + d) * nb + b];
            else
              up = ghost(p, bd, 2 * a + 1, face_index(p, a, ix[0], ix[1], ix[2]), c, d, b, I);
          } else {
            continue;
          }
          flux += (fabs(sa) / d_axis(p, a)) * (Ic - up);
        }
        Iout[(c * nd + d) * nb + b] =
            Ic + p->dt * (betac[c * nb + b] * (I0c[c * nb + b] - Ic) - p->v[b] * flux);
      }
    }
  }
}

/* Reduction (reading #18/#19): D_{c,b} = sum_d w_d (I0c_{c,b} - I_{c,d,b}),
 * within-octant ascending d, then the octant sign-bit tree. */
void ora_reduce(const ora_problem *p, const double *I, const double *I0c, double *D) {
  long nc = p->nx * p->ny * p->nz;
  int nd = p->nd, nb = p->nb;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1)
  for (long c = 0; c < nc; c++)
    for (int b = 0; b < nb; b++) {
      double q[8] = {0};
      for (int d = 0; d < nd; d++)
        q[ora_octant(p->s + 3 * d)] += p->w[d] * (I0c[c * nb + b] - I[(c * nd + d) * nb + b]);
      D[c * nb + b] = octant_tree(q);
    }
}

/* Per-cell Newton (readings #2, #18): solve
 *   F(T) = sum_b c_b [ W (I0_b(T) - I0c_b) + D_b ] = 0,   c_b = beta_next_b / v_b,
 * from T = Tn; F(Tn) == 0.0 exactly keeps Tn.  Bracket [1, 5000] K updated by
 * the sign of F (F increasing); bisect when a Newton step leaves it; stop when
 * |dT| <= 1e-13 T or F == 0; more than 50 iterations is an error. */
int ora_newton(const ora_problem *p, double Tn, const double *D, const double *I0c, const double *bnext,
               double *Tout, int *iters) {
  double W = 0.0;
  for (int d = 0; d < p->nd; d++) W += p->w[d];
  int nb = p->nb;
  double T = Tn, lo = T_LO, hi = T_HI;
  *iters = 0;
  for (int it = 0; it <= NEWTON_MAXIT; it++) {
    double F = 0.0, Fp = 0.0;
    for (int b = 0; b < nb; b++) {
      double dI0;
      double i0 = ora_I0(p, b, T, &dI0);
      double cb = bnext[b] / p->v[b];
      F += cb * (W * (i0 - I0c[b]) + D[b]);
      Fp += cb * W * dI0;
    }
    if (!isfinite(F) || !isfinite(Fp)) return ORA_ENONFINITE;
    if (F == 0.0) {
      *Tout = T;
      return ORA_OK;
    }
    if (it == NEWTON_MAXIT) break;
    if (F < 0.0)
      lo = T;
    else
      hi = T;
    double step = F / Fp;
    double Tn1 = T - step;
    *iters = it + 1;
    /* converged on the Newton step itself (before any bracket test: a step
     * below one ulp of T must not be mistaken for leaving the bracket) */
    if (fabs(step) <= NEWTON_RTOL * T) {
      *Tout = Tn1;
      return ORA_OK;
    }
    if (!(Tn1 > lo && Tn1 < hi)) Tn1 = 0.5 * (lo + hi);
    T = Tn1;
  }
  *Tout = T;
  return ORA_ENEWTON;
}

/* Self-consistent tau (reading R-k, SURVEY f4 "non-lagged tau(T) inside the
 * Newton"): solve
 *   F(T) = sum_b (beta_b(T)/v_b) [ W (I0_b(T) - I0c_b) + D_b ] = 0
 * with F'(T) = sum_b [ (beta_b'(T)/v_b)(W (I0_b - I0c_b) + D_b) + (beta_b/v_b) W dI0_b/dT ],
 * the same bracket / step rules as ora_newton (F(Tn) == 0.0 keeps Tn). */
int ora_newton_sc(const ora_problem *p, double Tn, const double *D, const double *I0c, double *Tout, int *iters) {
  double W = 0.0;
  for (int d = 0; d < p->nd; d++) W += p->w[d];
  int nb = p->nb;
  double T = Tn, lo = T_LO, hi = T_HI;
  *iters = 0;
  for (int it = 0; it <= NEWTON_MAXIT; it++) {
    double F = 0.0, Fp = 0.0;
    for (int b = 0; b < nb; b++) {
      double dI0;
      double i0 = ora_I0(p, b, T, &dI0);
      double h = W * (i0 - I0c[b]) + D[b];
      F += ora_beta(p, b, T) / p->v[b] * h;
      Fp += ora_dbeta(p, b, T) / p->v[b] * h + ora_beta(p, b, T) / p->v[b] * W * dI0;
    }
    if (!isfinite(F) || !isfinite(Fp)) return ORA_ENONFINITE;
    if (F == 0.0) {
      *Tout = T;
      return ORA_OK;
    }
    if (it == NEWTON_MAXIT) break;
    if (F < 0.0)
      lo = T;
    else
      hi = T;
    double step = F / Fp;
    double Tn1 = T - step;
    *iters = it + 1;
    if (fabs(step) <= NEWTON_RTOL * T) {
      *Tout = Tn1;
      return ORA_OK;
    }
    if (!(Tn1 > lo && Tn1 < hi) || !(Fp > 0.0)) Tn1 = 0.5 * (lo + hi);
    T = Tn1;
  }
  *Tout = T;
  return ORA_ENEWTON;
}

/* Temperature update over all cells: beta_next = beta(Tn) (lagged tau, reading
 * #15), Newton, then refresh I0c <- I0(T^{n+1}), betac <- beta_next (P:L277-281,
 * P:L498-500).  Returns first failing cell in *bad (or -1). */
int ora_temperature_update(const ora_problem *p, const double *D, double *T, double *I0c, double *betac,
                           long *bad, int *max_iters) {
  long nc = p->nx * p->ny * p->nz;
  int nb = p->nb;
  long first_bad = -1;
  int status = ORA_OK, mit = 0;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1) reduction(max : mit)
  for (long c = 0; c < nc; c++) {
    double bn[512];
    for (int b = 0; b < nb; b++) bn[b] = ora_beta(p, b, T[c]);
    double Tnew;
    int it;
    double bw[512]; /* Newton weights times v_b: beta_b, or beta_b/(1 + dt beta_b) in the semi-implicit step (R-l) */
    for (int b = 0; b < nb; b++) bw[b] = p->semi ? bn[b] / (1.0 + p->dt * bn[b]) : bn[b];
    int st = p->tau_mode == 1 ? ora_newton_sc(p, T[c], D + c * nb, I0c + c * nb, &Tnew, &it)
                              : ora_newton(p, T[c], D + c * nb, I0c + c * nb, bw, &Tnew, &it);
    if (it > mit) mit = it;
    if (st != ORA_OK) {
#pragma omp critical
      {
        if (first_bad < 0 || c < first_bad) {
          first_bad = c;
          status = st;
        }
      }
      continue;
    }
    T[c] = Tnew;
    for (int b = 0; b < nb; b++) {
      I0c[c * nb + b] = ora_I0(p, b, Tnew, NULL);
      betac[c * nb + b] = p->tau_mode == 1 ? ora_beta(p, b, Tnew) : bn[b];
    }
  }
  if (bad) *bad = first_bad;
  if (max_iters) *max_iters = mit;
  return status;
}

/* --------------------------------------------------------------- public API */

int ora_sweep(const ora_problem *p, const double *I, const double *I0c, const double *betac, double *Iout) {
  ora_bcdata bd;
  int st = bc_prepare(p, &bd);
  if (st) {
    bc_free(&bd);
    return st;
  }
  int nreg = p->dim == 3 ? 6 : 4;
  for (int r = 0; r < nreg; r++)
    if (p->bc_kind[r] == BC_DIFF || p->bc_kind[r] == BC_PART) diffuse_table(p, r, I, bd.den[r], bd.gdiff[r]);
  ora_sweep_bd(p, &bd, I, I0c, betac, Iout);
  bc_free(&bd);
  return ORA_OK;
}

/* ghost table of one wall for the current I (tests): iso or diffuse */
int ora_ghost_table(const ora_problem *p, int region, const double *I, double *g) {
  ora_bcdata bd;
  int st = bc_prepare(p, &bd);
  if (!st) {
    if (p->bc_kind[region] == BC_ISO)
      memcpy(g, bd.giso[region], sizeof(double) * ora_n_faces(p, region) * p->nb);
    else if (p->bc_kind[region] == BC_DIFF)
      diffuse_table(p, region, I, bd.den[region], g);
    else
      st = ORA_EINVAL;
  }
  bc_free(&bd);
  return st;
}

/* Semi-implicit step (reading R-l), last part: with J the advected field and
 * (I0c, betac) refreshed at T^{n+1} (betac = beta(T^n), lagged),
 *   I^{n+1}_{c,d,b} = (J + dt beta_b I0_b(T^{n+1})) / (1 + dt beta_b). */
void ora_relax(const ora_problem *p, long nc, const double *J, const double *I0c, const double *betac, double *I) {
  int nd = p->nd, nb = p->nb;
  for (long c = 0; c < nc; c++)
    for (int d = 0; d < nd; d++)
      for (int b = 0; b < nb; b++) {
        double db = p->dt * betac[c * nb + b];
        I[(c * nd + d) * nb + b] = (J[(c * nd + d) * nb + b] + db * I0c[c * nb + b]) / (1.0 + db);
      }
}

/* Run nsteps explicit steps in place on (I, T, I0c, betac).
 * Order within a step (reading #14): ghosts from I^n -> sweep -> reduce ->
 * Newton -> refresh.  On error: *err_step = failing step, *err_cell = cell. */
int ora_run(const ora_problem *p, double *I, double *T, double *I0c, double *betac, long nsteps,
            long *err_step, long *err_cell, int *max_iters) {
  long nc = p->nx * p->ny * p->nz;
  size_t n = (size_t)nc * p->nd * p->nb;
  ora_bcdata bd;
  int st = bc_prepare(p, &bd);
  if (st) {
    bc_free(&bd);
    return st;
  }
  double *J = (double *)malloc(sizeof(double) * n);
  double *D = (double *)malloc(sizeof(double) * nc * p->nb);
  double *Z = (double *)calloc((size_t)nc * p->nb, sizeof(double));
  if (!J || !D || !Z) {
    free(J);
    free(D);
    free(Z);
    bc_free(&bd);
    return ORA_ENOMEM;
  }
  if (p->semi && p->tau_mode == 1) {
    free(J);
    free(D);
    free(Z);
    bc_free(&bd);
    return ORA_EINVAL;
  }
  int nreg = p->dim == 3 ? 6 : 4;
  int mit = 0;
  if (err_step) *err_step = -1;
  if (err_cell) *err_cell = -1;
  for (long s = 0; s < nsteps && st == ORA_OK; s++) {
    for (int r = 0; r < nreg; r++)
      if (p->bc_kind[r] == BC_DIFF || p->bc_kind[r] == BC_PART) diffuse_table(p, r, I, bd.den[r], bd.gdiff[r]);
    /* semi-implicit (R-l): advection only (beta = 0 in the sweep), then the
     * temperature with weights beta/(1 + dt beta), then the implicit relaxation */
    ora_sweep_bd(p, &bd, I, I0c, p->semi ? Z : betac, J);
    ora_reduce(p, J, I0c, D);
    long bad;
    int it;
    st = ora_temperature_update(p, D, T, I0c, betac, &bad, &it);
    if (it > mit) mit = it;
    if (p->semi)
      ora_relax(p, nc, J, I0c, betac, I);
    else
      memcpy(I, J, sizeof(double) * n);
    if (st != ORA_OK) {
      if (err_step) *err_step = s;
      if (err_cell) *err_cell = bad;
    }
  }
  if (max_iters) *max_iters = mit;
  free(J);
  free(D);
  free(Z);
  bc_free(&bd);
  return st;
}

/* ---------------------------------------------------------- implicit step (R-n)
 *
 * "solvers take 10-20 iterations (depending on the time
 * step size) to attain 3-4 orders of convergence within each time step".
 * Reading R-n: the backward-Euler step of Eq. 4 in the finite-volume form of
 * Eq. 5, every term at the new time level,
 *   I' - I^n = dt [ beta_{c,b} (I0_b(T') - I') - v_b sum_a (|s_a|/D_a)(I' - I'_up,a) ],
 * beta = beta(T^n) (lagged as #15), ghosts of I' (Eq. 6), and T' from the
 * scattering balance (#2) of I'.  Solved by source iteration, k = 0, 1, ...
 * from I^0 = I^n, T^0 = T^n:
 *   (a) wall ghosts from I^k (diffuse tables, specular partners);
 *   (b) for every direction, a transport sweep in upwind order -- each cell
 *       after its upwind neighbours, so I'_up is this sweep's own value
 *       (exact inversion of the upwind operator for the source I0(T^k)):
 *         I^{k+1} = I^n + [dt beta (I0c^k - I^n) + sum_a kk_a (I^{k+1}_up,a - I^n)]
 *                         / (1 + dt beta + sum_a kk_a),     kk_a = dt v_b |s_a| / D_a,
 *       axis terms in x, y, z order (the deviation form keeps a uniform
 *       equilibrium exact, like #19);
 *   (c) D = sum_d w_d (I0c^k - I^{k+1}) (step-3 order), Newton for T^{k+1}
 *       from T^k with weights beta/v_b (the step's beta), I0c^{k+1} = I0(T^{k+1});
 * until k = imp_max_iter, or earlier when imp_tol > 0 and both inputs of the
 * last sweep had settled: max_c |T^{k+1} - T^k| <= imp_tol T^k and the wall
 * data of (a) changed by at most imp_tol relative from the previous
 * iteration's (the outgoing intensities of specular/partial wall cells, the
 * diffuse ghost tables; at k = 0 there is no previous, so no early stop while
 * such walls exist).  The step ends with I^{n+1} = I^K, T^{n+1} = T^K,
 * I0c = I0(T^K), betac = beta(T^n). */

/* largest relative change of the wall data (a) between iterates Ik and Ikm1:
 * outgoing intensities of the cells on specular / partial walls, and the
 * diffuse tables gd vs gdm1 (diffuse / partial walls) */
static double wall_change(const ora_problem *p, const ora_bcdata *bd, const double *Ik, const double *Ikm1,
                          double *const *gdm1) {
  int nreg = p->dim == 3 ? 6 : 4;
  int nd = p->nd, nb = p->nb;
  double m = 0.0;
  for (int r = 0; r < nreg; r++) {
    int k = p->bc_kind[r];
    int a = r / 2;
    double sg = (r & 1) ? 1.0 : -1.0;
    long nf = ora_n_faces(p, r);
    if (k == BC_SPEC || k == BC_PART) {
      for (long f = 0; f < nf; f++) {
        long x, y, z;
        if (a == 0) {
          y = f % p->ny; z = f / p->ny; x = (r & 1) ? p->nx - 1 : 0;
        } else if (a == 1) {
          x = f % p->nx; z = f / p->nx; y = (r & 1) ? p->ny - 1 : 0;
        } else {
          x = f % p->nx; y = f / p->nx; z = (r & 1) ? p->nz - 1 : 0;
        }
        long c = x + p->nx * (y + p->ny * z);
        for (int d = 0; d < nd; d++) {
          if (!(sg * p->s[3 * d + a] > 0.0)) continue; /* outgoing through this wall */
          for (int b = 0; b < nb; b++) {
            long e = (c * nd + d) * nb + b;
            double rel = fabs(Ik[e] - Ikm1[e]) / fabs(Ikm1[e]);
            if (rel > m) m = rel;
          }
        }
      }
    }
    if (k == BC_DIFF || k == BC_PART) {
      for (long e = 0; e < nf * nb; e++) {
        double rel = fabs(bd->gdiff[r][e] - gdm1[r][e]) / fabs(gdm1[r][e]);
        if (rel > m) m = rel;
      }
    }
  }
  return m;
}

/* one upwind-ordered transport sweep (b) for all directions */
static void implicit_sweep(const ora_problem *p, const ora_bcdata *bd, const double *In, const double *Ik,
                           const double *I0c, const double *beta, double *Inew) {
  long nx = p->nx, ny = p->ny, nz = p->nz;
  int nd = p->nd, nb = p->nb;
  int na = p->dim == 3 ? 3 : 2;
  long n[3] = {nx, ny, nz};
  long stride[3] = {1, nx, nx * ny};
#pragma omp parallel for schedule(dynamic, 1) num_threads(p->nthreads > 0 ? p->nthreads : 1)
  for (int d = 0; d < nd; d++) {
    const double *sd = p->s + 3 * d;
    /* per axis: march from the upwind side (any order where s_a == 0) */
    long lo[3], st[3];
    for (int a = 0; a < 3; a++) {
      int neg = a < na && sd[a] < 0.0;
      lo[a] = neg ? n[a] - 1 : 0;
      st[a] = neg ? -1 : 1;
    }
    for (long kz = 0; kz < nz; kz++)
      for (long ky = 0; ky < ny; ky++)
        for (long kx = 0; kx < nx; kx++) {
          long ix[3] = {lo[0] + st[0] * kx, lo[1] + st[1] * ky, lo[2] + st[2] * kz};
          long c = ix[0] + nx * (ix[1] + ny * ix[2]);
          for (int b = 0; b < nb; b++) {
            double Ic = In[(c * nd + d) * nb + b];
            double db = p->dt * beta[c * nb + b];
            double num = db * (I0c[c * nb + b] - Ic);
            double den = 1.0 + db;
            for (int a = 0; a < na; a++) {
              double sa = sd[a];
              if (sa == 0.0) continue;
              double up;
              if (sa > 0.0) {
                if (ix[a] > 0)
                  up = Inew[((c - stride[a]) * nd + d) * nb + b];
                else
                  up = ghost(p, bd, 2 * a, face_index(p, a, ix[0], ix[1], ix[2]), c, d, b, Ik);
              } else {
                if (ix[a] < n[a] - 1)
                  up = Inew[((c + stride[a]) * nd + d) * nb + b];
                else
                  up = ghost(p, bd, 2 * a + 1, face_index(p, a, ix[0], ix[1], ix[2]), c, d, b, Ik);
              }
              double kk = p->dt * p->v[b] * (fabs(sa) / d_axis(p, a));
              num += kk * (up - Ic);
              den += kk;
            }
            Inew[(c * nd + d) * nb + b] = Ic + num / den;
          }
        }
  }
}

/* nsteps implicit steps (R-n) in place; iters[s] = iterations of step s (optional) */
int ora_run_implicit(const ora_problem *p, double *I, double *T, double *I0c, double *betac, long nsteps,
                     long *iters, long *err_step, long *err_cell) {
  long nc = p->nx * p->ny * p->nz;
  int nb = p->nb;
  size_t n = (size_t)nc * p->nd * nb;
  if (p->imp_max_iter < 1 || p->tau_mode != 0 || p->semi) return ORA_EINVAL;
  ora_bcdata bd;
  int st = bc_prepare(p, &bd);
  if (st) {
    bc_free(&bd);
    return st;
  }
  int nreg = p->dim == 3 ? 6 : 4;
  double *In = (double *)malloc(sizeof(double) * n);
  double *J = (double *)malloc(sizeof(double) * n);
  double *Ip = (double *)malloc(sizeof(double) * n); /* I^{k-1}: the wall-data change */
  double *D = (double *)malloc(sizeof(double) * nc * nb);
  double *beta = (double *)malloc(sizeof(double) * nc * nb);
  double *gdm1[6] = {NULL, NULL, NULL, NULL, NULL, NULL};
  int ok = In && J && Ip && D && beta;
  int walls = 0; /* walls whose data (a) come from the iterate */
  for (int r = 0; r < nreg && ok; r++) {
    if (p->bc_kind[r] != BC_ISO) walls = 1;
    if (p->bc_kind[r] == BC_DIFF || p->bc_kind[r] == BC_PART) {
      gdm1[r] = (double *)malloc(sizeof(double) * ora_n_faces(p, r) * nb);
      ok = gdm1[r] != NULL;
    }
  }
  if (!ok) {
    free(In);
    free(J);
    free(Ip);
    free(D);
    free(beta);
    for (int r = 0; r < 6; r++) free(gdm1[r]);
    bc_free(&bd);
    return ORA_ENOMEM;
  }
  if (err_step) *err_step = -1;
  if (err_cell) *err_cell = -1;
  for (long s = 0; s < nsteps && st == ORA_OK; s++) {
    memcpy(In, I, sizeof(double) * n);
    for (long c = 0; c < nc; c++)
      for (int b = 0; b < nb; b++) beta[c * nb + b] = ora_beta(p, b, T[c]); /* beta(T^n) for the whole step */
    long k = 0;
    for (; k < p->imp_max_iter; k++) {
      for (int r = 0; r < nreg; r++) /* (a) ghosts of I^k */
        if (p->bc_kind[r] == BC_DIFF || p->bc_kind[r] == BC_PART) {
          if (k > 0) memcpy(gdm1[r], bd.gdiff[r], sizeof(double) * ora_n_faces(p, r) * nb);
          diffuse_table(p, r, I, bd.den[r], bd.gdiff[r]);
        }
      double gch = walls ? (k > 0 ? wall_change(p, &bd, I, Ip, gdm1) : INFINITY) : 0.0;
      implicit_sweep(p, &bd, In, I, I0c, beta, J); /* (b) */
      ora_reduce(p, J, I0c, D);                    /* (c) */
      double dmax = 0.0;
      long first_bad = -1;
      int cst = ORA_OK;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1) reduction(max : dmax)
      for (long c = 0; c < nc; c++) {
        double Tnew;
        int it;
        int r = ora_newton(p, T[c], D + c * nb, I0c + c * nb, beta + c * nb, &Tnew, &it);
        if (r != ORA_OK) {
#pragma omp critical
          {
            if (first_bad < 0 || c < first_bad) {
              first_bad = c;
              cst = r;
            }
          }
          continue;
        }
        double rel = fabs(Tnew - T[c]) / T[c];
        if (rel > dmax) dmax = rel;
        T[c] = Tnew;
        for (int b = 0; b < nb; b++) I0c[c * nb + b] = ora_I0(p, b, Tnew, NULL);
      }
      memcpy(Ip, I, sizeof(double) * n);
      memcpy(I, J, sizeof(double) * n);
      if (cst != ORA_OK) {
        st = cst;
        if (err_step) *err_step = s;
        if (err_cell) *err_cell = first_bad;
        k++;
        break;
      }
      if (p->imp_tol > 0.0 && dmax <= p->imp_tol && gch <= p->imp_tol) {
        k++;
        break;
      }
    }
    if (iters) iters[s] = k;
    memcpy(betac, beta, sizeof(double) * nc * nb);
  }
  free(In);
  free(J);
  free(Ip);
  free(D);
  free(beta);
  for (int r = 0; r < 6; r++) free(gdm1[r]);
  bc_free(&bd);
  return st;
}

/* Set-state with I only: T from one reduce-and-Newton solve starting at
 * T_guess with beta_next = beta(T_guess) and I0c = I0(T_guess). */
int ora_solve_T(const ora_problem *p, const double *I, const double *T_guess, double *T, double *I0c,
                double *betac) {
  long nc = p->nx * p->ny * p->nz;
  memcpy(T, T_guess, sizeof(double) * nc);
  ora_refresh(p, T, I0c, betac);
  double *D = (double *)malloc(sizeof(double) * nc * p->nb);
  if (!D) return ORA_ENOMEM;
  ora_reduce(p, I, I0c, D);
  long bad;
  int it;
  /* the temperature of a given state is the plain scattering balance (#2),
   * whatever the integrator (the semi-implicit weights belong to its step) */
  ora_problem q = *p;
  q.semi = 0;
  int st = ora_temperature_update(&q, D, T, I0c, betac, &bad, &it);
  free(D);
  return st;
}

/* Diagnostic energy E = sum_c V sum_b (1/v_b) sum_d w_d I_{c,d,b} */
double ora_energy(const ora_problem *p, const double *I) {
  long nc = p->nx * p->ny * p->nz;
  double V = p->dx * p->dy * p->dz; /* dim 2: dz is the unit depth */
  double E = 0.0;
  for (long c = 0; c < nc; c++) {
    double ec = 0.0;
    for (int b = 0; b < p->nb; b++) {
      double G = 0.0;
      for (int d = 0; d < p->nd; d++) G += p->w[d] * I[(c * p->nd + d) * p->nb + b];
      ec += G / p->v[b];
    }
    E += V * ec;
  }
  return E;
}

int ora_sizeof_problem(void) { return (int)sizeof(ora_problem); }
