/*
 * bte_oracle_umesh.c -- plain fp64 CPU ORACLE of the explicit BTE step on an
 * UNSTRUCTURED simplex mesh.  TEST INFRASTRUCTURE ONLY (same
 * rules as bte_oracle.c: only tests/, smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it; it shares no source with the CUDA path).
 *
 * The finite-volume step is Eq. 3 written out literally for
 * m-sided cells, with the upwind face value of P:L150-157:
 *
 *   I'_{c,d,b} = I + dt*( beta_{c,b} (I0c_{c,b} - I)
 *                         - v_b * sum_{f in faces(c)} (A_f / V_c) (s_d . n_f) I_up(f,d,b) )
 *
 *   I_up = I_c                       if s_d . n_f > 0   ("CELL1")
 *        = I of the neighbour across f, or the wall ghost (Eq. 6), otherwise
 *                                                       ("CELL2")
 *
 * The face sum runs over the cell's faces in local order (face k is opposite
 * local vertex k); s.n = s_x n_x + s_y n_y + s_z n_z in that order.
 * Geometry (a0, written from the definitions):
 *   triangle (2-D): V = |(p1-p0) x (p2-p0)|/2 * depth, face k = edge
 *     (p_{k+1}, p_{k+2}) of length L, A = L * depth, n = the unit
 *     perpendicular of the edge pointing away from p_k;
 *   convex m-gon (2-D, "a polygonal/polyhedral cell with m sides",
 *     P:L176-181): V = |shoelace sum|/2 * depth, face k = edge
 *     (p_{k+1 mod m}, p_{k+2 mod m}), n pointing away from the vertex mean;
 *   tetrahedron (3-D): V = |det(p1-p0, p2-p0, p3-p0)|/6, face k = triangle
 *     of the other three vertices (ascending local order) a, b, c,
 *     A = |(b-a) x (c-a)|/2, n = (b-a) x (c-a) / |.| pointing away from p_k;
 *   hexahedron (3-D, "polyhedral cell with m sides"; Gmsh vertex
 *     order, bottom 0-1-2-3, top 4-5-6-7): faces 0 (0,1,2,3), 1 (4,5,6,7),
 *     2 (0,1,5,4), 3 (1,2,6,5), 4 (2,3,7,6), 5 (3,0,4,7), each the bilinear
 *     patch through its four corners (planar when the corners are coplanar):
 *     area vector S = (q2-q0) x (q3-q1) / 2 (the integral of the normal over
 *     the patch), A = |S|, n = S/|S| pointing away from the cell's vertex
 *     mean; V = (1/3) sum_f qbar_f . S_f (divergence theorem with the face
 *     vertex mean qbar_f, exact for bilinear faces).
 * Boundary faces (no neighbour) must lie on a wall of the vertices' bounding
 * box: all vertices at x = xmin -> region 0, x = xmax -> 1, y -> 2/3, z -> 4/5
 * (tested in that order).  A wall face's normal is the outward axis vector,
 * and its ghosts are the structured ones (Eq. 6; readings #11, #12, R-i).
 * Wall faces are numbered per region in (cell, local face) ascending order.
 *
 * The temperature update (reduction, Newton, refresh) is the same per-cell
 * operation as on the structured grid and is taken from bte_oracle.c with
 * the problem's nx = ncells, ny = nz = 1.
 *
 * parity pins: tests/test_oracle_pins.py (unstructured section).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_EINVAL 1
#define ORA_ENOMEM 2
#define ORA_ENOTCLOSED 6
#define BC_ISO 0
#define BC_SPEC 1
#define BC_DIFF 2
#define BC_PART 3

/* must match bte_oracle.c */
typedef struct {
  int dim;
  long nx, ny, nz;
  double dx, dy, dz;
  int nd;
  const double *s;
  const double *w;
  int nb;
  const double *v;
  int mode;
  const double *I_ref, *slope;
  double T_ref;
  const double *w_lo, *w_hi, *vs, *c2, *g;
  const double *beta_coef;
  double dt;
  int bc_kind[6];
  const double *T_wall[6];
  double T_uniform[6];
  int nthreads;
  double specularity[6];
  int tau_mode;
  int semi;
} ora_problem;

double ora_I0(const ora_problem *p, int b, double T, double *dI0dT);
int ora_octant(const double *s);
int ora_reflection(const ora_problem *p, int axis, int *r);
void ora_reduce(const ora_problem *p, const double *I, const double *I0c, double *D);
int ora_temperature_update(const ora_problem *p, const double *D, double *T, double *I0c, double *betac,
                           long *bad, int *max_iters);
void ora_relax(const ora_problem *p, long nc, const double *J, const double *I0c, const double *betac, double *I);

typedef struct {
  int dim;
  long nverts;
  const double *verts; /* [nverts][3] */
  long ncells;
  const long *cells;   /* [ncells][nvc] */
  double depth;
  int nvc;             /* vertices per cell: dim 2 -> 3 (triangles) or m (convex polygons), dim 3 -> 4 or 8 */
} ora_umesh;

typedef struct {
  long nc;
  int K;          /* faces per cell = dim + 1 */
  double *vol;    /* [nc] */
  double *area;   /* [nc][K] */
  double *nrm;    /* [nc][K][3] */
  long *nbr;      /* [nc][K] neighbour or -1 */
  int *region;    /* [nc][K] wall region of a boundary face, else -1 */
  long *bface;    /* [nc][K] index of the face in its region's list */
  long nrf[6];    /* faces per region */
  long *rcell[6]; /* region face -> cell */
} ora_ugeom;

typedef struct {
  long key[4];
  long cell;
  int k;
} face_rec;

/* hexahedron faces as cycles of local vertices (Gmsh order) */
static const int HEXF[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};

static int face_cmp(const void *a, const void *b) {
  const face_rec *x = (const face_rec *)a, *y = (const face_rec *)b;
  for (int i = 0; i < 4; i++)
    if (x->key[i] != y->key[i]) return x->key[i] < y->key[i] ? -1 : 1;
  if (x->cell != y->cell) return x->cell < y->cell ? -1 : 1;
  return x->k - y->k;
}

static void sort3(long *v, int n) {
  for (int i = 1; i < n; i++)
    for (int j = i; j > 0 && v[j - 1] > v[j]; j--) {
      long t = v[j];
      v[j] = v[j - 1];
      v[j - 1] = t;
    }
}

void ora_ugeom_free(ora_ugeom *g) {
  if (!g) return;
  free(g->vol);
  free(g->area);
  free(g->nrm);
  free(g->nbr);
  free(g->region);
  free(g->bface);
  for (int r = 0; r < 6; r++) free(g->rcell[r]);
  free(g);
}

/* geometry precompute (a0): volumes, face areas, outward normals, face
 * matching, wall classification.  Returns ORA_EINVAL for a degenerate cell, a
 * face shared by more than two cells, or a boundary face off the box walls. */
int ora_ugeom_build(const ora_umesh *m, ora_ugeom **out) {
  *out = NULL;
  if (m->dim != 2 && m->dim != 3) return ORA_EINVAL;
  const int nvc = m->nvc > 0 ? m->nvc : m->dim + 1;
  if ((m->dim == 3 && nvc != 4 && nvc != 8) || (m->dim == 2 && (nvc < 3 || nvc > 8))) return ORA_EINVAL;
  const int hexa = m->dim == 3 && nvc == 8;
  const int K = hexa ? 6 : nvc, nfv = hexa ? 4 : m->dim; /* faces per cell, vertices per face */
  const long nc = m->ncells;
  ora_ugeom *g = (ora_ugeom *)calloc(1, sizeof(ora_ugeom));
  if (!g) return ORA_ENOMEM;
  g->nc = nc;
  g->K = K;
  g->vol = (double *)malloc(sizeof(double) * nc);
  g->area = (double *)malloc(sizeof(double) * nc * K);
  g->nrm = (double *)malloc(sizeof(double) * nc * K * 3);
  g->nbr = (long *)malloc(sizeof(long) * nc * K);
  g->region = (int *)malloc(sizeof(int) * nc * K);
  g->bface = (long *)malloc(sizeof(long) * nc * K);
  face_rec *fr = (face_rec *)malloc(sizeof(face_rec) * nc * K);
  if (!g->vol || !g->area || !g->nrm || !g->nbr || !g->region || !g->bface || !fr) {
    free(fr);
    ora_ugeom_free(g);
    return ORA_ENOMEM;
  }
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (long i = 0; i < m->nverts; i++)
    for (int a = 0; a < 3; a++) {
      double x = m->verts[3 * i + a];
      if (x < lo[a]) lo[a] = x;
      if (x > hi[a]) hi[a] = x;
    }
  for (long c = 0; c < nc; c++) {
    const long *cv = m->cells + c * nvc;
    for (int k = 0; k < nvc; k++)
      if (cv[k] < 0 || cv[k] >= m->nverts) {
        free(fr);
        ora_ugeom_free(g);
        return ORA_EINVAL;
      }
    const double *P[8];
    for (int k = 0; k < nvc; k++) P[k] = m->verts + 3 * cv[k];
    if (hexa) {
      double cm[3] = {0.0, 0.0, 0.0};
      for (int k = 0; k < 8; k++)
        for (int t = 0; t < 3; t++) cm[t] += P[k][t];
      for (int t = 0; t < 3; t++) cm[t] /= 8.0;
      double vol = 0.0;
      for (int k = 0; k < 6; k++) {
        const double *q0 = P[HEXF[k][0]], *q1 = P[HEXF[k][1]], *q2 = P[HEXF[k][2]], *q3 = P[HEXF[k][3]];
        double d1[3], d2[3], S[3], qb[3];
        for (int t = 0; t < 3; t++) {
          d1[t] = q2[t] - q0[t];
          d2[t] = q3[t] - q1[t];
          qb[t] = (q0[t] + q1[t] + q2[t] + q3[t]) / 4.0;
        }
        S[0] = (d1[1] * d2[2] - d1[2] * d2[1]) / 2.0;
        S[1] = (d1[2] * d2[0] - d1[0] * d2[2]) / 2.0;
        S[2] = (d1[0] * d2[1] - d1[1] * d2[0]) / 2.0;
        if (S[0] * (qb[0] - cm[0]) + S[1] * (qb[1] - cm[1]) + S[2] * (qb[2] - cm[2]) < 0.0)
          for (int t = 0; t < 3; t++) S[t] = -S[t];
        double A = sqrt(S[0] * S[0] + S[1] * S[1] + S[2] * S[2]);
        g->area[c * K + k] = A;
        for (int t = 0; t < 3; t++) g->nrm[(c * K + k) * 3 + t] = S[t] / A;
        vol += qb[0] * S[0] + qb[1] * S[1] + qb[2] * S[2];
      }
      g->vol[c] = vol / 3.0;
    } else if (m->dim == 2 && K > 3) {
      double sh = 0.0, cx = 0.0, cy = 0.0;
      for (int k = 0; k < K; k++) {
        const double *a = P[k], *b = P[(k + 1) % K];
        sh += a[0] * b[1] - b[0] * a[1];
        cx += a[0];
        cy += a[1];
      }
      cx /= K;
      cy /= K;
      g->vol[c] = fabs(sh) / 2.0 * m->depth;
      for (int k = 0; k < K; k++) {
        const double *a = P[(k + 1) % K], *b = P[(k + 2) % K];
        double ex = b[0] - a[0], ey = b[1] - a[1];
        double L = sqrt(ex * ex + ey * ey);
        double nx = ey / L, ny = -ex / L;
        if (nx * (cx - a[0]) + ny * (cy - a[1]) > 0.0) {
          nx = -nx;
          ny = -ny;
        }
        g->area[c * K + k] = L * m->depth;
        g->nrm[(c * K + k) * 3 + 0] = nx;
        g->nrm[(c * K + k) * 3 + 1] = ny;
        g->nrm[(c * K + k) * 3 + 2] = 0.0;
      }
    } else if (m->dim == 2) {
      double ux = P[1][0] - P[0][0], uy = P[1][1] - P[0][1];
      double vx = P[2][0] - P[0][0], vy = P[2][1] - P[0][1];
      g->vol[c] = fabs(ux * vy - uy * vx) / 2.0 * m->depth;
      for (int k = 0; k < K; k++) {
        const double *a = P[(k + 1) % 3], *b = P[(k + 2) % 3], *o = P[k];
        double ex = b[0] - a[0], ey = b[1] - a[1];
        double L = sqrt(ex * ex + ey * ey);
        double nx = ey / L, ny = -ex / L;
        if (nx * (o[0] - a[0]) + ny * (o[1] - a[1]) > 0.0) {
          nx = -nx;
          ny = -ny;
        }
        g->area[c * K + k] = L * m->depth;
        g->nrm[(c * K + k) * 3 + 0] = nx;
        g->nrm[(c * K + k) * 3 + 1] = ny;
        g->nrm[(c * K + k) * 3 + 2] = 0.0;
      }
    } else {
      double u[3], v[3], w[3];
      for (int a = 0; a < 3; a++) {
        u[a] = P[1][a] - P[0][a];
        v[a] = P[2][a] - P[0][a];
        w[a] = P[3][a] - P[0][a];
      }
      double det = u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0]) +
                   u[2] * (v[0] * w[1] - v[1] * w[0]);
      g->vol[c] = fabs(det) / 6.0;
      for (int k = 0; k < K; k++) {
        int q[3], n = 0;
        for (int i = 0; i < 4; i++)
          if (i != k) q[n++] = i;
        const double *a = P[q[0]], *b = P[q[1]], *cc = P[q[2]], *o = P[k];
        double e1[3], e2[3], cr[3];
        for (int t = 0; t < 3; t++) {
          e1[t] = b[t] - a[t];
          e2[t] = cc[t] - a[t];
        }
        cr[0] = e1[1] * e2[2] - e1[2] * e2[1];
        cr[1] = e1[2] * e2[0] - e1[0] * e2[2];
        cr[2] = e1[0] * e2[1] - e1[1] * e2[0];
        double len = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        double nn[3] = {cr[0] / len, cr[1] / len, cr[2] / len};
        if (nn[0] * (o[0] - a[0]) + nn[1] * (o[1] - a[1]) + nn[2] * (o[2] - a[2]) > 0.0)
          for (int t = 0; t < 3; t++) nn[t] = -nn[t];
        g->area[c * K + k] = len / 2.0;
        for (int t = 0; t < 3; t++) g->nrm[(c * K + k) * 3 + t] = nn[t];
      }
    }
    if (!(g->vol[c] > 0.0)) {
      free(fr);
      ora_ugeom_free(g);
      return ORA_EINVAL;
    }
    for (int k = 0; k < K; k++) {
      face_rec *f = fr + c * K + k;
      int n = 0;
      f->key[2] = -1;
      f->key[3] = -1;
      if (hexa) {
        for (int i = 0; i < 4; i++) f->key[i] = cv[HEXF[k][i]];
      } else if (m->dim == 2) { /* edge (v_{k+1}, v_{k+2}) (for triangles: the face opposite v_k) */
        f->key[0] = cv[(k + 1) % K];
        f->key[1] = cv[(k + 2) % K];
      } else {
        for (int i = 0; i < K; i++)
          if (i != k) f->key[n++] = cv[i];
      }
      sort3(f->key, nfv);
      f->cell = c;
      f->k = k;
      g->nbr[c * K + k] = -1;
      g->region[c * K + k] = -1;
      g->bface[c * K + k] = -1;
    }
  }
  /* face matching: equal sorted vertex keys */
  qsort(fr, (size_t)nc * K, sizeof(face_rec), face_cmp);
  long nf = nc * K;
  for (long i = 0; i < nf;) {
    long j = i + 1;
    while (j < nf && fr[j].key[0] == fr[i].key[0] && fr[j].key[1] == fr[i].key[1] &&
           fr[j].key[2] == fr[i].key[2] && fr[j].key[3] == fr[i].key[3])
      j++;
    if (j - i > 2) {
      free(fr);
      ora_ugeom_free(g);
      return ORA_EINVAL;
    }
    if (j - i == 2) {
      g->nbr[fr[i].cell * K + fr[i].k] = fr[i + 1].cell;
      g->nbr[fr[i + 1].cell * K + fr[i + 1].k] = fr[i].cell;
    }
    i = j;
  }
  free(fr);
  /* walls, numbered in (cell, local face) order */
  for (long c = 0; c < nc; c++)
    for (int k = 0; k < K; k++) {
      if (g->nbr[c * K + k] >= 0) continue;
      const long *cv = m->cells + c * nvc;
      int reg = -1;
      for (int r = 0; r < 2 * m->dim && reg < 0; r++) {
        int a = r / 2;
        double wall = (r & 1) ? hi[a] : lo[a];
        int all = 1;
        if (hexa) {
          for (int i = 0; i < 4; i++)
            if (m->verts[3 * cv[HEXF[k][i]] + a] != wall) all = 0;
        } else if (m->dim == 2) {
          if (m->verts[3 * cv[(k + 1) % K] + a] != wall || m->verts[3 * cv[(k + 2) % K] + a] != wall) all = 0;
        } else {
          for (int i = 0; i < K; i++)
            if (i != k && m->verts[3 * cv[i] + a] != wall) all = 0;
        }
        if (all) reg = r;
      }
      if (reg < 0) {
        ora_ugeom_free(g);
        return ORA_EINVAL;
      }
      g->region[c * K + k] = reg;
      g->bface[c * K + k] = g->nrf[reg]++;
      double *n = g->nrm + (c * K + k) * 3;
      n[0] = n[1] = n[2] = 0.0;
      n[reg / 2] = (reg & 1) ? 1.0 : -1.0;
    }
  for (int r = 0; r < 6; r++) {
    g->rcell[r] = (long *)malloc(sizeof(long) * (g->nrf[r] > 0 ? g->nrf[r] : 1));
    if (!g->rcell[r]) {
      ora_ugeom_free(g);
      return ORA_ENOMEM;
    }
  }
  for (long c = 0; c < nc; c++)
    for (int k = 0; k < K; k++)
      if (g->region[c * K + k] >= 0) g->rcell[g->region[c * K + k]][g->bface[c * K + k]] = c;
  *out = g;
  return ORA_OK;
}

long ora_ugeom_nfaces(const ora_ugeom *g, int region) { return g->nrf[region]; }

void ora_ugeom_export(const ora_ugeom *g, double *vol, double *area, double *nrm, long *nbr, int *region) {
  long n = g->nc * g->K;
  if (vol) memcpy(vol, g->vol, sizeof(double) * g->nc);
  if (area) memcpy(area, g->area, sizeof(double) * n);
  if (nrm) memcpy(nrm, g->nrm, sizeof(double) * n * 3);
  if (nbr) memcpy(nbr, g->nbr, sizeof(long) * n);
  if (region) memcpy(region, g->region, sizeof(int) * n);
}

/* ------------------------------------------------------------ wall ghosts */

typedef struct {
  double *giso[6];
  double *gdiff[6];
  double den[6];
  int *refl[3];
} ubc;

static double octant_tree(const double *q) {
  return ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
}

/* diffuse denominator of wall r: sum over incoming d of w|s_a| (reading #11) */
static double udiffuse_den(const ora_problem *p, int r) {
  int a = r / 2;
  double sg = (r & 1) ? 1.0 : -1.0;
  double q[8] = {0};
  for (int d = 0; d < p->nd; d++) {
    double sa = p->s[3 * d + a];
    if (sg * sa < 0.0) q[ora_octant(p->s + 3 * d)] += p->w[d] * fabs(sa);
  }
  return octant_tree(q);
}

static void udiffuse_table(const ora_problem *p, const ora_ugeom *g, int r, const double *I, double den,
                           double *out) {
  int a = r / 2;
  double sg = (r & 1) ? 1.0 : -1.0;
  int nd = p->nd, nb = p->nb;
  for (long f = 0; f < g->nrf[r]; f++) {
    long c = g->rcell[r][f];
    for (int b = 0; b < nb; b++) {
      double q[8] = {0};
      for (int d = 0; d < nd; d++) {
        double sa = p->s[3 * d + a];
        if (sg * sa > 0.0) q[ora_octant(p->s + 3 * d)] += p->w[d] * fabs(sa) * I[(c * nd + d) * nb + b];
      }
      out[f * nb + b] = octant_tree(q) / den;
    }
  }
}

static void ubc_free(ubc *bd) {
  for (int r = 0; r < 6; r++) {
    free(bd->giso[r]);
    free(bd->gdiff[r]);
  }
  for (int a = 0; a < 3; a++) free(bd->refl[a]);
}

static int ubc_prepare(const ora_problem *p, const ora_ugeom *g, ubc *bd) {
  memset(bd, 0, sizeof(*bd));
  for (int a = 0; a < 3; a++) {
    bd->refl[a] = (int *)malloc(sizeof(int) * p->nd);
    if (!bd->refl[a]) return ORA_ENOMEM;
  }
  int nreg = p->dim == 3 ? 6 : 4;
  for (int r = 0; r < nreg; r++) {
    long nf = g->nrf[r];
    int k = p->bc_kind[r];
    if (k == BC_ISO) {
      bd->giso[r] = (double *)malloc(sizeof(double) * (nf > 0 ? nf : 1) * p->nb);
      if (!bd->giso[r]) return ORA_ENOMEM;
      for (long f = 0; f < nf; f++) {
        double Tw = p->T_wall[r] ? p->T_wall[r][f] : p->T_uniform[r];
        for (int b = 0; b < p->nb; b++) bd->giso[r][f * p->nb + b] = ora_I0(p, b, Tw, NULL);
      }
    } else if (k == BC_SPEC || k == BC_DIFF || k == BC_PART) {
      if (k != BC_DIFF && ora_reflection(p, r / 2, bd->refl[r / 2]) != ORA_OK) return ORA_ENOTCLOSED;
      if (k == BC_PART && !(p->specularity[r] >= 0.0 && p->specularity[r] <= 1.0)) return ORA_EINVAL;
      if (k != BC_SPEC) {
        bd->gdiff[r] = (double *)malloc(sizeof(double) * (nf > 0 ? nf : 1) * p->nb);
        if (!bd->gdiff[r]) return ORA_ENOMEM;
        bd->den[r] = udiffuse_den(p, r);
        if (!(bd->den[r] > 0.0)) return ORA_EINVAL;
      }
    } else {
      return ORA_EINVAL;
    }
  }
  return ORA_OK;
}

static void ubc_update(const ora_problem *p, const ora_ugeom *g, ubc *bd, const double *I) {
  int nreg = p->dim == 3 ? 6 : 4;
  for (int r = 0; r < nreg; r++)
    if (p->bc_kind[r] == BC_DIFF || p->bc_kind[r] == BC_PART) udiffuse_table(p, g, r, I, bd->den[r], bd->gdiff[r]);
}

static double ughost(const ora_problem *p, const ubc *bd, int r, long f, long c, int d, int b, const double *I) {
  int k = p->bc_kind[r];
  if (k == BC_ISO) return bd->giso[r][f * p->nb + b];
  if (k == BC_DIFF) return bd->gdiff[r][f * p->nb + b];
  double spec = I[(c * p->nd + bd->refl[r / 2][d]) * p->nb + b];
  if (k == BC_PART) {
    double sp = p->specularity[r];
    return sp * spec + (1.0 - sp) * bd->gdiff[r][f * p->nb + b];
  }
  return spec;
}

/* ------------------------------------------------------------ the sweep */

static void usweep_bd(const ora_problem *p, const ora_ugeom *g, const ubc *bd, const double *I, const double *I0c,
                      const double *betac, double *Iout) {
  const long nc = g->nc;
  const int K = g->K, nd = p->nd, nb = p->nb;
#pragma omp parallel for schedule(static) num_threads(p->nthreads > 0 ? p->nthreads : 1)
  for (long c = 0; c < nc; c++) {
    for (int d = 0; d < nd; d++) {
      const double *s = p->s + 3 * d;
      for (int b = 0; b < nb; b++) {
        double Ic = I[(c * nd + d) * nb + b];
        double flux = 0.0;
        for (int k = 0; k < K; k++) {
          const double *n = g->nrm + (c * K + k) * 3;
          double sn = s[0] * n[0] + s[1] * n[1] + s[2] * n[2];
          double up;
          if (sn > 0.0) {
            up = Ic;
          } else {
            long e = g->nbr[c * K + k];
            if (e >= 0)
              up = I[(e * nd + d) * nb + b];
            else
              up = ughost(p, bd, g->region[c * K + k], g->bface[c * K + k], c, d, b, I);
          }
          flux += (g->area[c * K + k] / g->vol[c]) * sn * up;
        }
        Iout[(c * nd + d) * nb + b] =
            Ic + p->dt * (betac[c * nb + b] * (I0c[c * nb + b] - Ic) - p->v[b] * flux);
      }
    }
  }
}

int ora_usweep(const ora_problem *p, const ora_ugeom *g, const double *I, const double *I0c, const double *betac,
               double *Iout) {
  ubc bd;
  int st = ubc_prepare(p, g, &bd);
  if (!st) {
    ubc_update(p, g, &bd, I);
    usweep_bd(p, g, &bd, I, I0c, betac, Iout);
  }
  ubc_free(&bd);
  return st;
}

/* Run nsteps explicit steps in place (reading #14 order): ghosts from I^n ->
 * sweep -> reduce -> Newton -> refresh.  p->nx must equal the cell count. */
int ora_urun(const ora_problem *p, const ora_ugeom *g, double *I, double *T, double *I0c, double *betac,
             long nsteps, long *err_step, long *err_cell, int *max_iters) {
  if (p->nx * p->ny * p->nz != g->nc) return ORA_EINVAL;
  size_t n = (size_t)g->nc * p->nd * p->nb;
  ubc bd;
  int st = ubc_prepare(p, g, &bd);
  if (st) {
    ubc_free(&bd);
    return st;
  }
  double *J = (double *)malloc(sizeof(double) * n);
  double *D = (double *)malloc(sizeof(double) * g->nc * p->nb);
  double *Z = (double *)calloc((size_t)g->nc * p->nb, sizeof(double));
  if (!J || !D || !Z || (p->semi && p->tau_mode == 1)) {
    free(J);
    free(D);
    free(Z);
    ubc_free(&bd);
    return (J && D && Z) ? ORA_EINVAL : ORA_ENOMEM;
  }
  int mit = 0;
  if (err_step) *err_step = -1;
  if (err_cell) *err_cell = -1;
  for (long s = 0; s < nsteps && st == ORA_OK; s++) {
    ubc_update(p, g, &bd, I);
    usweep_bd(p, g, &bd, I, I0c, p->semi ? Z : betac, J);  /* semi-implicit (R-l): advection only */
    ora_reduce(p, J, I0c, D);
    long bad;
    int it;
    st = ora_temperature_update(p, D, T, I0c, betac, &bad, &it);
    if (it > mit) mit = it;
    if (p->semi)
      ora_relax(p, g->nc, J, I0c, betac, I);
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
  ubc_free(&bd);
  return st;
}

/* E = sum_c V_c sum_b (1/v_b) sum_d w_d I_{c,d,b} */
double ora_uenergy(const ora_problem *p, const ora_ugeom *g, const double *I) {
  double E = 0.0;
  for (long c = 0; c < g->nc; c++) {
    double ec = 0.0;
    for (int b = 0; b < p->nb; b++) {
      double G = 0.0;
      for (int d = 0; d < p->nd; d++) G += p->w[d] * I[(c * p->nd + d) * p->nb + b];
      ec += G / p->v[b];
    }
    E += g->vol[c] * ec;
  }
  return E;
}

/* positivity margin of the explicit update (reading #9 on a general mesh):
 * min over c, d, b of 1 - dt*beta_b(Tmax) - dt*v_b * sum_{f: s.n > 0} (A_f/V_c) s.n */
double ora_udt_margin(const ora_problem *p, const ora_ugeom *g, double beta_max_b0, int b) {
  double worst = 1e300;
  for (long c = 0; c < g->nc; c++)
    for (int d = 0; d < p->nd; d++) {
      double out = 0.0;
      for (int k = 0; k < g->K; k++) {
        const double *n = g->nrm + (c * g->K + k) * 3;
        double sn = p->s[3 * d] * n[0] + p->s[3 * d + 1] * n[1] + p->s[3 * d + 2] * n[2];
        if (sn > 0.0) out += (g->area[c * g->K + k] / g->vol[c]) * sn;
      }
      double m = 1.0 - p->dt * beta_max_b0 - p->dt * p->v[b] * out;
      if (m < worst) worst = m;
    }
  return worst;
}
