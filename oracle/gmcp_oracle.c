/* Plain-C restatement of the GMCP contact hot path. TEST INFRASTRUCTURE ONLY.
 *
 * This is the CPU oracle the CUDA path is differential-tested against. It is
 * a restatement (SoA, C99, no Eigen) of the reference algorithm, written to
 * reproduce the reference's IEEE operation order so results are bitwise equal
 * to oracle/_ref (the unmodified reference headers) -- tests/test_oracle.py
 * pins that. Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj/include/gmcp/).
 *
 * Build: oracle/Makefile (-O3, -ffp-contract=off: no FMA contraction).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "gmcp_oracle_api.h"

/* ------------------------------------------------------------------------ */
/* errors                                                                     */

static __thread char g_err[256];

static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }
int orc_is_reference(void) { return 0; }

/* ------------------------------------------------------------------------ */
/* small vector algebra in the reference's evaluation order                   */

typedef struct { double v[3]; } v3;
typedef struct { double x, y; } v2;

static inline v3 mk3(double a, double b, double c) { v3 r = {{a, b, c}}; return r; }
static inline v3 ld3(const double* x, int64_t vid) { return mk3(x[3 * vid], x[3 * vid + 1], x[3 * vid + 2]); }
static inline v3 add3(v3 a, v3 b) { return mk3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static inline v3 sub3(v3 a, v3 b) { return mk3(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static inline v3 scl3(double s, v3 a) { return mk3(s * a.v[0], s * a.v[1], s * a.v[2]); }
static inline v3 div3(v3 a, double s) { return mk3(a.v[0] / s, a.v[1] / s, a.v[2] / s); }
static inline double dot3(v3 a, v3 b) { return (a.v[0] * b.v[0] + a.v[1] * b.v[1]) + a.v[2] * b.v[2]; }
static inline double nrm3(v3 a) { return sqrt(dot3(a, a)); }
static inline v3 crs3(v3 a, v3 b) {
  return mk3(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
             a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static inline v3 unit3(v3 a) { /* Eigen normalized(): divide by sqrt(squaredNorm) */
  const double z = dot3(a, a);
  return z > 0 ? div3(a, sqrt(z)) : a;
}
static inline double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

static inline v2 mk2(double x, double y) { v2 r = {x, y}; return r; }
static inline v2 sub2(v2 a, v2 b) { return mk2(a.x - b.x, a.y - b.y); }
static inline v2 add2(v2 a, v2 b) { return mk2(a.x + b.x, a.y + b.y); }
static inline v2 scl2(double s, v2 a) { return mk2(s * a.x, s * a.y); }
static inline double nrm2(v2 a) { return sqrt(a.x * a.x + a.y * a.y); }
static inline double cross2(v2 a, v2 b) { return a.x * b.y - a.y * b.x; } /* contact_sampling.hpp:35 */

/* ------------------------------------------------------------------------ */
/* geometry.hpp                                                                */

/* geometry.hpp:14-21 (triangle_aabb core.hpp:92-98, Aabb::diagonal core.hpp:84) */
static int triangle_normal(v3 a, v3 b, v3 c, v3* n) {
  const v3 cr = crs3(sub3(b, a), sub3(c, a));
  v3 lo = mk3(DBL_MAX, DBL_MAX, DBL_MAX), hi = mk3(-DBL_MAX, -DBL_MAX, -DBL_MAX);
  const v3 p[3] = {a, b, c};
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      lo.v[k] = dmin(lo.v[k], p[i].v[k]);
      hi.v[k] = dmax(hi.v[k], p[i].v[k]);
    }
  const double diag2 = nrm3(sub3(hi, lo));
  const double area_eps = 1e-12 * diag2 * diag2;
  if (0.5 * nrm3(cr) <= area_eps)
    return set_err(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle (area below cutoff)");
  *n = unit3(cr);
  return GMCP_OK;
}

/* geometry.hpp:101-103 */
static inline double signed_area_2d(v2 a, v2 b, v2 c) {
  return 0.5 * ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x));
}

/* geometry.hpp:106-114 */
static int barycentric_2d(v2 p, v2 a, v2 b, v2 c, v3* out) {
  const double area = signed_area_2d(a, b, c);
  const double d0 = nrm2(sub2(b, a)), d1 = nrm2(sub2(c, a)), d2 = nrm2(sub2(c, b));
  const double diag = dmax(dmax(d0, d1), d2);
  if (fabs(area) <= 1e-14 * diag * diag)
    return set_err(GMCP_ERR_DEGENERATE, "barycentric_2d: degenerate 2D triangle");
  const double u = signed_area_2d(p, b, c) / area;
  const double v = signed_area_2d(a, p, c) / area;
  *out = mk3(u, v, 1.0 - u - v);
  return GMCP_OK;
}

/* geometry.hpp:118-134 */
typedef struct { v3 origin, t1, t2, n; } frame_t;

static int tangent_frame(v3 a, v3 b, v3 c, frame_t* f) {
  int rc = triangle_normal(a, b, c, &f->n);
  if (rc) return rc;
  f->origin = a;
  f->t1 = unit3(sub3(b, a));
  f->t2 = crs3(f->n, f->t1);
  return GMCP_OK;
}
static inline v2 to_plane(const frame_t* f, v3 p) {
  const v3 d = sub3(p, f->origin);
  return mk2(dot3(d, f->t1), dot3(d, f->t2));
}

/* ------------------------------------------------------------------------ */
/* quadrature.hpp:20-81                                                        */

typedef struct { double b0, b1, b2, w; } triq_t;
typedef struct { double t, w; } segq_t;

static int triangle_quadrature(int order, triq_t* q) {
  switch (order) {
    case 1:
      q[0] = (triq_t){1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 1.0};
      return 1;
    case 2: {
      const double a = 2.0 / 3.0, b = 1.0 / 6.0, w = 1.0 / 3.0;
      q[0] = (triq_t){a, b, b, w};
      q[1] = (triq_t){b, a, b, w};
      q[2] = (triq_t){b, b, a, w};
      return 3;
    }
    case 3: {
      const double a = 0.659027622374092, b = 0.231933368553031, c = 0.109039009072877, w = 1.0 / 6.0;
      q[0] = (triq_t){a, b, c, w};
      q[1] = (triq_t){a, c, b, w};
      q[2] = (triq_t){b, a, c, w};
      q[3] = (triq_t){b, c, a, w};
      q[4] = (triq_t){c, a, b, w};
      q[5] = (triq_t){c, b, a, w};
      return 6;
    }
    case 4: {
      const double a1 = 0.108103018168070, b1 = 0.445948490915965, w1 = 0.223381589678011;
      const double a2 = 0.816847572980459, b2 = 0.091576213509771, w2 = 0.109951743655322;
      q[0] = (triq_t){a1, b1, b1, w1};
      q[1] = (triq_t){b1, a1, b1, w1};
      q[2] = (triq_t){b1, b1, a1, w1};
      q[3] = (triq_t){a2, b2, b2, w2};
      q[4] = (triq_t){b2, a2, b2, w2};
      q[5] = (triq_t){b2, b2, a2, w2};
      return 6;
    }
    default:
      return -1;
  }
}

static int segment_quadrature(int points, segq_t* q) {
  static const double x2[] = {-0.5773502691896257, 0.5773502691896257}, w2[] = {1.0, 1.0};
  static const double x3[] = {-0.7745966692414834, 0.0, 0.7745966692414834};
  const double w3[] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  static const double x4[] = {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563, 0.8611363115940526};
  static const double w4[] = {0.3478548451374538, 0.6521451548625461, 0.6521451548625461, 0.3478548451374538};
  static const double x5[] = {-0.9061798459386640, -0.5384693101056831, 0.0, 0.5384693101056831, 0.9061798459386640};
  static const double w5[] = {0.2369268850561891, 0.4786286704993665, 0.5688888888888889, 0.4786286704993665,
                              0.2369268850561891};
  const double *xs, *ws;
  switch (points) {
    case 1:
      q[0] = (segq_t){0.5, 1.0};
      return 1;
    case 2: xs = x2; ws = w2; break;
    case 3: xs = x3; ws = w3; break;
    case 4: xs = x4; ws = w4; break;
    case 5: xs = x5; ws = w5; break;
    default: return -1;
  }
  for (int i = 0; i < points; ++i) q[i] = (segq_t){0.5 * (1.0 + xs[i]), 0.5 * ws[i]};
  return points;
}

/* ------------------------------------------------------------------------ */
/* barrier.hpp                                                                 */

/* barrier.hpp:55-66 */
static int barrier_eval(double g, double eps, double* B, double* dB, double* ddB) {
  if (!(g > 0)) return set_err(GMCP_ERR_INFEASIBLE, "barrier: non-positive gap");
  if (!(eps > 0)) return set_err(GMCP_ERR_INFEASIBLE, "barrier: non-positive support radius");
  *B = *dB = *ddB = 0;
  if (g >= eps) return GMCP_OK;
  const double d = g - eps;
  const double ln = log(g / eps);
  *B = -d * d * ln;
  *dB = -2.0 * d * ln - d * d / g;
  *ddB = -2.0 * ln - 4.0 * d / g + d * d / (g * g);
  return GMCP_OK;
}

/* barrier.hpp:69-74 */
static inline double hermite_step(double x, double delta) {
  if (x <= 0) return 0;
  if (x >= delta) return 1;
  const double t = x / delta;
  return t * t * (3.0 - 2.0 * t);
}
/* barrier.hpp:78-81 (callers guarantee g_ref > 0) */
static inline double adaptive_eps(double g_ref, double eps_max) { return dmin(0.9 * g_ref, eps_max); }
static inline double min3(v3 a) { return dmin(dmin(a.v[0], a.v[1]), a.v[2]); }

int orc_resolve_barrier_params(gmcp_barrier_params* p, double m) {
  /* barrier.hpp:25-46 */
  if (!(m > 0)) return set_err(GMCP_ERR_CONFIG, "barrier params: mean slave edge length must be positive");
  if (!(p->kappa_face > 0)) return set_err(GMCP_ERR_CONFIG, "barrier params: kappa_face must be positive");
  if (p->kappa_edge < 0) p->kappa_edge = 1e-3 * p->kappa_face * m;
  if (p->kappa_point < 0) p->kappa_point = 1e-3 * p->kappa_face * m * m;
  if (!(p->kappa_edge > 0) || !(p->kappa_point > 0))
    return set_err(GMCP_ERR_CONFIG, "barrier params: per-type stiffnesses must be positive");
  if (!(p->eps_max > 0)) return set_err(GMCP_ERR_CONFIG, "barrier params: eps_max must be positive");
  if (!(p->delta_face > 0) || p->delta_face > 1.0 / 3.0)
    return set_err(GMCP_ERR_CONFIG, "barrier params: delta_face must lie in (0, 1/3]");
  if (!(p->delta_edge > 0) || p->delta_edge > 0.5)
    return set_err(GMCP_ERR_CONFIG, "barrier params: delta_edge must lie in (0, 1/2]");
  if (p->detection_radius < 0) p->detection_radius = 10.0 * p->eps_max;
  if (!(p->detection_radius > 0)) return set_err(GMCP_ERR_CONFIG, "barrier params: detection_radius must be positive");
  if (p->quad_order_face < 1 || p->quad_order_face > 4)
    return set_err(GMCP_ERR_CONFIG, "barrier params: quad_order_face must lie in 1..4");
  if (p->quad_order_edge < 1 || p->quad_order_edge > 5)
    return set_err(GMCP_ERR_CONFIG, "barrier params: quad_order_edge must lie in 1..5");
  return GMCP_OK;
}

int orc_barrier(double g, double eps, double* out) { return barrier_eval(g, eps, &out[0], &out[1], &out[2]); }

int orc_mean_edge_length(const gmcp_surface* s, const double* x, double* out) {
  /* contact_sampling.hpp:257-263 */
  if (s->n_edges == 0) return set_err(GMCP_ERR_CONFIG, "contact surface has no edges");
  double sum = 0;
  for (int e = 0; e < s->n_edges; ++e) sum += nrm3(sub3(ld3(x, s->edges[2 * e]), ld3(x, s->edges[2 * e + 1])));
  *out = sum / (double)s->n_edges;
  return GMCP_OK;
}

/* ------------------------------------------------------------------------ */
/* growable arrays                                                            */

typedef struct { int32_t* a; int64_t n, cap; } ivec;
static void ipush(ivec* v, int32_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 16;
    v->a = (int32_t*)realloc(v->a, (size_t)v->cap * sizeof(int32_t));
  }
  v->a[v->n++] = x;
}
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}
static int64_t sort_unique(int32_t* a, int64_t n) {
  if (n == 0) return 0;
  qsort(a, (size_t)n, sizeof(int32_t), cmp_i32);
  int64_t k = 1;
  for (int64_t i = 1; i < n; ++i)
    if (a[i] != a[k - 1]) a[k++] = a[i];
  return k;
}

/* ------------------------------------------------------------------------ */
/* broadphase: contact_sampling.hpp:281-340 (brute-force definition; the     */
/* reference tree returns the same sorted set, test_sampling.cpp:390-397)     */

struct orc_pairs {
  int32_t n_st;
  int64_t* off[3];
  int32_t* ids[3];
};

typedef struct { v3 lo, hi; } box_t;

static box_t tri_box(const double* x, const int32_t* t) {
  box_t b = {mk3(DBL_MAX, DBL_MAX, DBL_MAX), mk3(-DBL_MAX, -DBL_MAX, -DBL_MAX)};
  for (int i = 0; i < 3; ++i) {
    const v3 p = ld3(x, t[i]);
    for (int k = 0; k < 3; ++k) {
      b.lo.v[k] = dmin(b.lo.v[k], p.v[k]);
      b.hi.v[k] = dmax(b.hi.v[k], p.v[k]);
    }
  }
  return b;
}
static inline int box_overlaps(const box_t* a, const box_t* b) { /* core.hpp:71-73 */
  for (int k = 0; k < 3; ++k)
    if (!(a->lo.v[k] <= b->hi.v[k]) || !(b->lo.v[k] <= a->hi.v[k])) return 0;
  return 1;
}

static int32_t lower_bound_i32(const int32_t* a, int32_t n, int32_t x) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

int orc_build_candidate_pairs(const gmcp_surface* slave, const gmcp_surface* master, const double* x,
                              double r, int use_tree, orc_pairs** out) {
  (void)use_tree;
  if (!(r > 0)) return set_err(GMCP_ERR_CONFIG, "build_candidate_pairs: detection radius must be positive");
  { /* shared-vertex check, contact_sampling.hpp:286-294 */
    int32_t i = 0, j = 0;
    while (i < slave->n_verts && j < master->n_verts) {
      if (slave->verts[i] == master->verts[j])
        return set_err(GMCP_ERR_CONFIG, "build_candidate_pairs: slave and master share vertices "
                                        "(self-contact is not supported)");
      if (slave->verts[i] < master->verts[j]) ++i; else ++j;
    }
  }
  box_t* mb = (box_t*)malloc(sizeof(box_t) * (size_t)(master->n_tris > 0 ? master->n_tris : 1));
  for (int32_t t = 0; t < master->n_tris; ++t) mb[t] = tri_box(x, master->tris + 3 * t);
  orc_pairs* p = (orc_pairs*)calloc(1, sizeof(orc_pairs));
  p->n_st = slave->n_tris;
  ivec all[3] = {{0}, {0}, {0}};
  for (int k = 0; k < 3; ++k) p->off[k] = (int64_t*)calloc((size_t)slave->n_tris + 1, sizeof(int64_t));
  ivec tmp = {0};
  for (int32_t st = 0; st < slave->n_tris; ++st) {
    box_t q = tri_box(x, slave->tris + 3 * st);
    for (int k = 0; k < 3; ++k) {
      q.lo.v[k] = q.lo.v[k] - r; /* Aabb::inflated, core.hpp:77-82 */
      q.hi.v[k] = q.hi.v[k] + r;
    }
    const int64_t t0 = all[0].n;
    for (int32_t mt = 0; mt < master->n_tris; ++mt)
      if (box_overlaps(&q, &mb[mt])) ipush(&all[0], mt);
    tmp.n = 0;
    for (int64_t i = t0; i < all[0].n; ++i)
      for (int e = 0; e < 3; ++e) ipush(&tmp, master->tri_edges[3 * all[0].a[i] + e]);
    int64_t ne = sort_unique(tmp.a, tmp.n);
    for (int64_t i = 0; i < ne; ++i) ipush(&all[1], tmp.a[i]);
    tmp.n = 0;
    for (int64_t i = t0; i < all[0].n; ++i)
      for (int e = 0; e < 3; ++e)
        ipush(&tmp, lower_bound_i32(master->verts, master->n_verts, master->tris[3 * all[0].a[i] + e]));
    int64_t nv = sort_unique(tmp.a, tmp.n);
    for (int64_t i = 0; i < nv; ++i) ipush(&all[2], tmp.a[i]);
    for (int k = 0; k < 3; ++k) p->off[k][st + 1] = all[k].n;
  }
  for (int k = 0; k < 3; ++k) p->ids[k] = all[k].a;
  free(tmp.a);
  free(mb);
  *out = p;
  return GMCP_OK;
}

int orc_pairs_from_csr(int32_t n_st, const int64_t* to, const int32_t* ti, const int64_t* eo, const int32_t* ei,
                       const int64_t* vo, const int32_t* vi, orc_pairs** out) {
  orc_pairs* p = (orc_pairs*)calloc(1, sizeof(orc_pairs));
  p->n_st = n_st;
  const int64_t* offs[3] = {to, eo, vo};
  const int32_t* idss[3] = {ti, ei, vi};
  for (int k = 0; k < 3; ++k) {
    p->off[k] = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n_st + 1));
    memcpy(p->off[k], offs[k], sizeof(int64_t) * ((size_t)n_st + 1));
    const int64_t n = offs[k][n_st];
    p->ids[k] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (n) memcpy(p->ids[k], idss[k], sizeof(int32_t) * (size_t)n);
  }
  *out = p;
  return GMCP_OK;
}

int64_t orc_pairs_size(const orc_pairs* p, int which) { return p->off[which][p->n_st]; }
int32_t orc_pairs_slave_tris(const orc_pairs* p) { return p->n_st; }
void orc_pairs_copy(const orc_pairs* p, int which, int64_t* offsets, int32_t* ids) {
  const int64_t n = p->off[which][p->n_st];
  if (offsets) memcpy(offsets, p->off[which], sizeof(int64_t) * ((size_t)p->n_st + 1));
  if (ids && n) memcpy(ids, p->ids[which], sizeof(int32_t) * (size_t)n);
}
void orc_pairs_free(orc_pairs* p) {
  if (!p) return;
  for (int k = 0; k < 3; ++k) {
    free(p->off[k]);
    free(p->ids[k]);
  }
  free(p);
}

/* ------------------------------------------------------------------------ */
/* samples                                                                     */

typedef struct {
  int8_t type;
  int32_t slave[3], master[3];
  double beta_s[3], beta_m[3], eta, weight, gamma, eps, g_ref;
} sample_t;

struct orc_state {
  sample_t* s;
  int64_t n, cap;
  double* ref_x;
  int64_t n_dof;
};

static void spush(struct orc_state* st, const sample_t* s) {
  if (st->n == st->cap) {
    st->cap = st->cap ? 2 * st->cap : 256;
    st->s = (sample_t*)realloc(st->s, (size_t)st->cap * sizeof(sample_t));
  }
  st->s[st->n++] = *s;
}

/* contact_sampling.hpp:80-83 */
static v3 clamp_bary(v3 b) {
  for (int k = 0; k < 3; ++k) b.v[k] = dmax(b.v[k], 0.0);
  const double s = b.v[0] + b.v[1] + b.v[2];
  return div3(b, s);
}
/* contact_sampling.hpp:88-90 */
static double local_scale(const v3* s) {
  return (nrm3(sub3(s[1], s[0])) + nrm3(sub3(s[2], s[0])) + nrm3(sub3(s[2], s[1]))) / 3.0;
}
static inline v3 interp3(const double* w, const v3* p) {
  return add3(add3(scl3(w[0], p[0]), scl3(w[1], p[1])), scl3(w[2], p[2]));
}

/* Sutherland-Hodgman clip, contact_sampling.hpp:39-58. Polygons stay <= 9. */
static int clip_polygon(v2* poly, int n, const v2* tri) {
  v2 out[12];
  for (int e = 0; e < 3; ++e) {
    if (n < 3) break;
    const v2 a = tri[e];
    const v2 dir = sub2(tri[(e + 1) % 3], a);
    int m = 0;
    for (int i = 0; i < n; ++i) {
      const v2 p = poly[i], q = poly[(i + 1) % n];
      const double dp = cross2(dir, sub2(p, a));
      const double dq = cross2(dir, sub2(q, a));
      if (dp >= 0) out[m++] = p;
      if ((dp >= 0) != (dq >= 0)) out[m++] = add2(p, scl2(dp / (dp - dq), sub2(q, p)));
    }
    memcpy(poly, out, sizeof(v2) * (size_t)m);
    n = m;
  }
  return n;
}
/* contact_sampling.hpp:60-66 */
static int merge_close(v2* poly, int n, double tol) {
  v2 out[12];
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || nrm2(sub2(poly[i], out[m - 1])) > tol) out[m++] = poly[i];
  while (m >= 2 && nrm2(sub2(out[0], out[m - 1])) <= tol) --m;
  memcpy(poly, out, sizeof(v2) * (size_t)m);
  return m;
}
/* contact_sampling.hpp:68-76 */
static double polygon_area(const v2* poly, int n) {
  double twice = 0;
  for (int i = 0; i < n; ++i) twice += cross2(poly[i], poly[(i + 1) % n]);
  return 0.5 * twice;
}

/* sample_face, contact_sampling.hpp:97-141. Appends to st. */
static int sample_face(const v3* s, const v3* m, const gmcp_barrier_params* P, const int32_t* sid,
                       const int32_t* mid, struct orc_state* out) {
  frame_t f;
  int rc = tangent_frame(s[0], s[1], s[2], &f);
  if (rc) return rc;
  const v2 s2[3] = {to_plane(&f, s[0]), to_plane(&f, s[1]), to_plane(&f, s[2])};
  const v2 m2[3] = {to_plane(&f, m[0]), to_plane(&f, m[1]), to_plane(&f, m[2])};
  const double scale = local_scale(s);
  const double merge_tol = 1e-12 * scale;
  const double area_tol = 1e-14 * scale * scale;
  const double m_area = signed_area_2d(m2[0], m2[1], m2[2]);
  if (fabs(m_area) <= area_tol) return GMCP_OK;
  v2 poly[12] = {m2[0], m2[1], m2[2]};
  if (m_area < 0) {
    const v2 t = poly[1];
    poly[1] = poly[2];
    poly[2] = t;
  }
  int n = clip_polygon(poly, 3, s2);
  n = merge_close(poly, n, merge_tol);
  if (n < 3 || polygon_area(poly, n) <= area_tol) return GMCP_OK;
  triq_t quad[6];
  const int nq = triangle_quadrature(P->quad_order_face, quad);
  for (int i = 1; i + 1 < n; ++i) {
    const v2 p0 = poly[0], p1 = poly[i], p2 = poly[i + 1];
    const double sub_area = signed_area_2d(p0, p1, p2);
    if (sub_area <= area_tol) continue;
    for (int q = 0; q < nq; ++q) {
      const v2 pt = add2(add2(scl2(quad[q].b0, p0), scl2(quad[q].b1, p1)), scl2(quad[q].b2, p2));
      sample_t smp;
      memset(&smp, 0, sizeof smp);
      smp.type = GMCP_FACE;
      v3 bs, bm;
      if ((rc = barycentric_2d(pt, s2[0], s2[1], s2[2], &bs))) return rc;
      bs = clamp_bary(bs);
      if ((rc = barycentric_2d(pt, m2[0], m2[1], m2[2], &bm))) return rc;
      memcpy(smp.beta_s, bs.v, sizeof bs.v);
      memcpy(smp.beta_m, bm.v, sizeof bm.v);
      smp.weight = quad[q].w * sub_area;
      smp.gamma = hermite_step(min3(bm), P->delta_face);
      const v3 xs = interp3(smp.beta_s, s), xm = interp3(smp.beta_m, m);
      const double g = dot3(f.n, sub3(xm, xs));
      smp.g_ref = g;
      smp.eps = g > 0 ? adaptive_eps(g, P->eps_max) : 0.0;
      for (int k = 0; k < 3; ++k) {
        smp.slave[k] = sid[k];
        smp.master[k] = mid[k];
      }
      spush(out, &smp);
    }
  }
  return GMCP_OK;
}

/* sample_edge, contact_sampling.hpp:146-192 */
static int sample_edge(const v3* s, const v3* e, const gmcp_barrier_params* P, const int32_t* sid,
                       const int32_t* eid, struct orc_state* out) {
  frame_t f;
  int rc = tangent_frame(s[0], s[1], s[2], &f);
  if (rc) return rc;
  const v2 s2[3] = {to_plane(&f, s[0]), to_plane(&f, s[1]), to_plane(&f, s[2])};
  const double scale = local_scale(s);
  const v2 q0 = to_plane(&f, e[0]);
  const v2 dq = sub2(to_plane(&f, e[1]), q0);
  if (nrm2(dq) <= 1e-12 * scale) return GMCP_OK;
  double t0 = 0, t1 = 1;
  for (int k = 0; k < 3; ++k) {
    const v2 a = s2[k];
    const v2 dir = sub2(s2[(k + 1) % 3], a);
    const double ca = cross2(dir, sub2(q0, a));
    const double dc = cross2(dir, dq);
    if (fabs(dc) <= 1e-14 * scale * scale) {
      if (ca < 0) return GMCP_OK;
    } else if (dc > 0) {
      t0 = dmax(t0, -ca / dc);
    } else {
      t1 = dmin(t1, -ca / dc);
    }
  }
  if (!(t1 - t0 > 1e-12)) return GMCP_OK;
  const double len3 = nrm3(sub3(e[1], e[0])) * (t1 - t0);
  segq_t quad[5];
  const int nq = segment_quadrature(P->quad_order_edge, quad);
  for (int q = 0; q < nq; ++q) {
    const double eta = t0 + (t1 - t0) * quad[q].t;
    sample_t smp;
    memset(&smp, 0, sizeof smp);
    smp.type = GMCP_EDGE;
    smp.eta = eta;
    v3 bs;
    if ((rc = barycentric_2d(add2(q0, scl2(eta, dq)), s2[0], s2[1], s2[2], &bs))) return rc;
    bs = clamp_bary(bs);
    memcpy(smp.beta_s, bs.v, sizeof bs.v);
    smp.weight = quad[q].w * len3;
    smp.gamma = hermite_step(eta, P->delta_edge) * hermite_step(1.0 - eta, P->delta_edge);
    const v3 xs = interp3(smp.beta_s, s);
    const v3 xm = add3(scl3(1.0 - eta, e[0]), scl3(eta, e[1]));
    const double g = dot3(f.n, sub3(xm, xs));
    smp.g_ref = g;
    smp.eps = g > 0 ? adaptive_eps(g, P->eps_max) : 0.0;
    for (int k = 0; k < 3; ++k) smp.slave[k] = sid[k];
    smp.master[0] = eid[0];
    smp.master[1] = eid[1];
    smp.master[2] = -1;
    spush(out, &smp);
  }
  return GMCP_OK;
}

/* sample_point, contact_sampling.hpp:196-215 */
static int sample_point(const v3* s, v3 v, const gmcp_barrier_params* P, const int32_t* sid, int32_t vid,
                        struct orc_state* out) {
  frame_t f;
  int rc = tangent_frame(s[0], s[1], s[2], &f);
  if (rc) return rc;
  v3 bary;
  if ((rc = barycentric_2d(to_plane(&f, v), to_plane(&f, s[0]), to_plane(&f, s[1]), to_plane(&f, s[2]), &bary)))
    return rc;
  if (min3(bary) < -1e-12) return GMCP_OK;
  sample_t smp;
  memset(&smp, 0, sizeof smp);
  smp.type = GMCP_POINT;
  const v3 bs = clamp_bary(bary);
  memcpy(smp.beta_s, bs.v, sizeof bs.v);
  smp.weight = 1;
  smp.gamma = 1;
  const v3 xs = interp3(smp.beta_s, s);
  const double g = dot3(f.n, sub3(v, xs));
  smp.g_ref = g;
  smp.eps = g > 0 ? adaptive_eps(g, P->eps_max) : 0.0;
  for (int k = 0; k < 3; ++k) smp.slave[k] = sid[k];
  smp.master[0] = vid;
  smp.master[1] = smp.master[2] = -1;
  spush(out, &smp);
  return GMCP_OK;
}

/* sample_gap, contact_sampling.hpp:350-372 */
static int sample_gap_(const sample_t* s, const double* x, double* g) {
  const v3 a0 = ld3(x, s->slave[0]), a1 = ld3(x, s->slave[1]), a2 = ld3(x, s->slave[2]);
  v3 n;
  int rc = triangle_normal(a0, a1, a2, &n);
  if (rc) return rc;
  const v3 xs = add3(add3(scl3(s->beta_s[0], a0), scl3(s->beta_s[1], a1)), scl3(s->beta_s[2], a2));
  v3 xm;
  if (s->type == GMCP_FACE)
    xm = add3(add3(scl3(s->beta_m[0], ld3(x, s->master[0])), scl3(s->beta_m[1], ld3(x, s->master[1]))),
              scl3(s->beta_m[2], ld3(x, s->master[2])));
  else if (s->type == GMCP_EDGE)
    xm = add3(scl3(1.0 - s->eta, ld3(x, s->master[0])), scl3(s->eta, ld3(x, s->master[1])));
  else
    xm = ld3(x, s->master[0]);
  *g = dot3(n, sub3(xm, xs));
  return GMCP_OK;
}

static void slave_pts(const gmcp_surface* sl, const double* x, int32_t st, v3* s) {
  for (int k = 0; k < 3; ++k) s[k] = ld3(x, sl->tris[3 * st + k]);
}

/* build_contact_state, contact_sampling.hpp:382-487 */
int orc_build_contact_state(const gmcp_surface* slave, const gmcp_surface* master, const orc_pairs* pairs,
                            const double* x, int64_t n_dof, const gmcp_barrier_params* P,
                            const double* eps_reference, orc_state** out) {
  if (pairs->n_st != slave->n_tris)
    return set_err(GMCP_ERR_CONFIG, "build_contact_state: pair set does not match slave surface");
  struct orc_state* S = (struct orc_state*)calloc(1, sizeof(struct orc_state));
  S->n_dof = n_dof;
  S->ref_x = (double*)malloc(sizeof(double) * (size_t)n_dof);
  memcpy(S->ref_x, x, sizeof(double) * (size_t)n_dof);
  int rc = GMCP_OK;

  /* point-sample ownership, contact_sampling.hpp:403-436 */
  const int32_t nmv = master->n_verts;
  ivec* by_vert = (ivec*)calloc((size_t)nmv + 1, sizeof(ivec));
  ivec* by_tri = (ivec*)calloc((size_t)slave->n_tris + 1, sizeof(ivec));
  for (int32_t st = 0; st < slave->n_tris; ++st)
    for (int64_t k = pairs->off[2][st]; k < pairs->off[2][st + 1]; ++k) ipush(&by_vert[pairs->ids[2][k]], st);
  const double boundary_tol = 1e-9;
  for (int32_t mv = 0; mv < nmv && rc == GMCP_OK; ++mv) {
    const v3 v = ld3(x, master->verts[mv]);
    int32_t first_boundary = -1;
    int any_interior = 0;
    for (int64_t k = 0; k < by_vert[mv].n; ++k) {
      const int32_t st = by_vert[mv].a[k];
      v3 s[3];
      slave_pts(slave, x, st, s);
      frame_t f;
      if ((rc = tangent_frame(s[0], s[1], s[2], &f))) break;
      v3 bary;
      if ((rc = barycentric_2d(to_plane(&f, v), to_plane(&f, s[0]), to_plane(&f, s[1]), to_plane(&f, s[2]), &bary)))
        break;
      const double mn = min3(bary);
      if (mn < -1e-12) continue;
      if (mn > boundary_tol) {
        any_interior = 1;
      } else if (first_boundary < 0) {
        first_boundary = st;
      }
    }
    if (rc) break;
    if (any_interior) {
      /* second pass re-derives the interior set (same decisions as the
         reference's interior_tris list, which keeps st ascending) */
      for (int64_t k = 0; k < by_vert[mv].n; ++k) {
        const int32_t st = by_vert[mv].a[k];
        v3 s[3];
        slave_pts(slave, x, st, s);
        frame_t f;
        tangent_frame(s[0], s[1], s[2], &f);
        v3 bary;
        barycentric_2d(to_plane(&f, v), to_plane(&f, s[0]), to_plane(&f, s[1]), to_plane(&f, s[2]), &bary);
        const double mn = min3(bary);
        if (mn >= -1e-12 && mn > boundary_tol) ipush(&by_tri[st], mv);
      }
    } else if (first_boundary >= 0) {
      ipush(&by_tri[first_boundary], mv);
    }
  }

  /* emission, contact_sampling.hpp:438-468 */
  for (int32_t st = 0; st < slave->n_tris && rc == GMCP_OK; ++st) {
    v3 s[3];
    slave_pts(slave, x, st, s);
    const int32_t* sid = slave->tris + 3 * st;
    for (int64_t k = pairs->off[0][st]; k < pairs->off[0][st + 1] && !rc; ++k) {
      const int32_t* mid = master->tris + 3 * pairs->ids[0][k];
      const v3 m[3] = {ld3(x, mid[0]), ld3(x, mid[1]), ld3(x, mid[2])};
      rc = sample_face(s, m, P, sid, mid, S);
    }
    for (int64_t k = pairs->off[1][st]; k < pairs->off[1][st + 1] && !rc; ++k) {
      const int32_t* eid = master->edges + 2 * pairs->ids[1][k];
      const v3 e[2] = {ld3(x, eid[0]), ld3(x, eid[1])};
      rc = sample_edge(s, e, P, sid, eid, S);
    }
    for (int64_t k = 0; k < by_tri[st].n && !rc; ++k) {
      const int32_t vid = master->verts[by_tri[st].a[k]];
      rc = sample_point(s, ld3(x, vid), P, sid, vid, S);
    }
  }
  for (int32_t i = 0; i <= nmv; ++i) free(by_vert[i].a);
  for (int32_t i = 0; i <= slave->n_tris; ++i) free(by_tri[i].a);
  free(by_vert);
  free(by_tri);
  if (rc) {
    orc_state_free(S);
    return rc;
  }

  /* freeze, contact_sampling.hpp:471-485 */
  int64_t kept = 0;
  for (int64_t i = 0; i < S->n; ++i) {
    sample_t smp = S->s[i];
    double g_now;
    if ((rc = sample_gap_(&smp, x, &g_now))) break;
    if (!(g_now > 0)) continue;
    double g_ref = g_now;
    if (eps_reference) {
      double g_stored;
      if ((rc = sample_gap_(&smp, eps_reference, &g_stored))) break;
      if (g_stored > 0) g_ref = g_stored;
    }
    smp.g_ref = g_ref;
    smp.eps = adaptive_eps(g_ref, P->eps_max);
    S->s[kept++] = smp;
  }
  if (rc) {
    orc_state_free(S);
    return rc;
  }
  S->n = kept;
  *out = S;
  return GMCP_OK;
}

int orc_state_from_samples(const gmcp_samples* in, const double* ref_x, int64_t n_dof, orc_state** out) {
  struct orc_state* S = (struct orc_state*)calloc(1, sizeof(struct orc_state));
  S->n_dof = n_dof;
  S->ref_x = (double*)malloc(sizeof(double) * (size_t)(n_dof > 0 ? n_dof : 1));
  if (n_dof) memcpy(S->ref_x, ref_x, sizeof(double) * (size_t)n_dof);
  for (int64_t i = 0; i < in->n; ++i) {
    sample_t s;
    s.type = in->type[i];
    for (int k = 0; k < 3; ++k) {
      s.slave[k] = in->slave[3 * i + k];
      s.master[k] = in->master[3 * i + k];
      s.beta_s[k] = in->beta_s[3 * i + k];
      s.beta_m[k] = in->beta_m[3 * i + k];
    }
    s.eta = in->eta[i];
    s.weight = in->weight[i];
    s.gamma = in->gamma[i];
    s.eps = in->eps[i];
    s.g_ref = in->g_ref[i];
    spush(S, &s);
  }
  *out = S;
  return GMCP_OK;
}

int64_t orc_state_size(const orc_state* S) { return S->n; }

void orc_state_copy(const orc_state* S, gmcp_samples* o) {
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    o->type[i] = s->type;
    for (int k = 0; k < 3; ++k) {
      o->slave[3 * i + k] = s->slave[k];
      o->master[3 * i + k] = s->master[k];
      o->beta_s[3 * i + k] = s->beta_s[k];
      o->beta_m[3 * i + k] = s->beta_m[k];
    }
    o->eta[i] = s->eta;
    o->weight[i] = s->weight;
    o->gamma[i] = s->gamma;
    o->eps[i] = s->eps;
    o->g_ref[i] = s->g_ref;
  }
}

void orc_state_free(orc_state* S) {
  if (!S) return;
  free(S->s);
  free(S->ref_x);
  free(S);
}

int orc_sample_gap(const orc_state* S, int64_t i, const double* x, double* g) {
  if (i < 0 || i >= S->n) return set_err(GMCP_ERR_ARG, "sample index out of range");
  return sample_gap_(&S->s[i], x, g);
}

/* ------------------------------------------------------------------------ */
/* contact_energy.hpp                                                          */

typedef struct {
  double g;
  v3 n, xs, xm;
  int nv;
  int32_t ids[6];
  v3 dg[6];
} kin_t;

/* sample_kinematics, contact_energy.hpp:26-73 */
static int kinematics(const sample_t* s, const double* x, int with_gradient, kin_t* k) {
  const v3 a0 = ld3(x, s->slave[0]), a1 = ld3(x, s->slave[1]), a2 = ld3(x, s->slave[2]);
  const v3 e1 = sub3(a1, a0), e2 = sub3(a2, a0);
  const v3 c = crs3(e1, e2);
  const double cn = nrm3(c);
  if (!(cn > 0)) return set_err(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle");
  k->n = div3(c, cn);
  k->xs = add3(add3(scl3(s->beta_s[0], a0), scl3(s->beta_s[1], a1)), scl3(s->beta_s[2], a2));
  int nm;
  double wm[3];
  if (s->type == GMCP_FACE) {
    nm = 3;
    wm[0] = s->beta_m[0];
    wm[1] = s->beta_m[1];
    wm[2] = s->beta_m[2];
  } else if (s->type == GMCP_EDGE) {
    nm = 2;
    wm[0] = 1.0 - s->eta;
    wm[1] = s->eta;
    wm[2] = 0;
  } else {
    nm = 1;
    wm[0] = 1;
    wm[1] = wm[2] = 0;
  }
  k->xm = mk3(0, 0, 0);
  for (int j = 0; j < nm; ++j) k->xm = add3(k->xm, scl3(wm[j], ld3(x, s->master[j])));
  const v3 d = sub3(k->xm, k->xs);
  k->g = dot3(k->n, d);
  k->nv = 3 + nm;
  for (int i = 0; i < 3; ++i) k->ids[i] = s->slave[i];
  for (int j = 0; j < nm; ++j) k->ids[3 + j] = s->master[j];
  if (!with_gradient) return GMCP_OK;
  const v3 r = div3(sub3(d, scl3(k->g, k->n)), cn);
  k->dg[0] = add3(scl3(-s->beta_s[0], k->n), crs3(r, sub3(e2, e1)));
  k->dg[1] = add3(scl3(-s->beta_s[1], k->n), crs3(e2, r));
  k->dg[2] = add3(scl3(-s->beta_s[2], k->n), crs3(r, e1));
  for (int j = 0; j < nm; ++j) k->dg[3 + j] = scl3(wm[j], k->n);
  return GMCP_OK;
}

/* contact_energy.hpp:75-84 */
static inline double sample_kappa(int type, const gmcp_barrier_params* P) {
  return type == GMCP_FACE ? P->kappa_face : type == GMCP_EDGE ? P->kappa_edge : P->kappa_point;
}

int orc_kinematics(const orc_state* S, const double* x, double* g, int32_t* nv, int32_t* ids, double* dg) {
  for (int64_t i = 0; i < S->n; ++i) {
    kin_t k;
    const int rc = kinematics(&S->s[i], x, 1, &k);
    if (rc) return rc;
    g[i] = k.g;
    nv[i] = k.nv;
    for (int v = 0; v < 6; ++v) {
      ids[6 * i + v] = v < k.nv ? k.ids[v] : -1;
      for (int a = 0; a < 3; ++a) dg[18 * i + 3 * v + a] = v < k.nv ? k.dg[v].v[a] : 0.0;
    }
  }
  return GMCP_OK;
}

/* contact_energy.hpp:95-108 */
int orc_try_contact_energy(const orc_state* S, const gmcp_barrier_params* P, const double* x, double* energy,
                           double* min_gap, int32_t* feasible) {
  double e = 0, mg = DBL_MAX;
  *feasible = 1;
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    double g, B, dB, ddB;
    int rc = sample_gap_(s, x, &g);
    if (rc) return rc;
    mg = dmin(mg, g);
    if (!(g > 0)) {
      *feasible = 0;
      break;
    }
    if ((rc = barrier_eval(g, s->eps, &B, &dB, &ddB))) return rc;
    e += sample_kappa(s->type, P) * s->weight * s->gamma * B;
  }
  *energy = e;
  *min_gap = mg;
  return GMCP_OK;
}

static int infeasible(int64_t i, double g, int64_t* bad) {
  char msg[160];
  snprintf(msg, sizeof msg, "contact sample %lld has non-positive gap %.17g", (long long)i, g);
  *bad = i;
  return set_err(GMCP_ERR_INFEASIBLE, msg);
}

/* contact_energy.hpp:110-123 */
int orc_contact_energy(const orc_state* S, const gmcp_barrier_params* P, const double* x, double* energy,
                       int64_t* bad) {
  double e = 0;
  *bad = -1;
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    double g, B, dB, ddB;
    int rc = sample_gap_(s, x, &g);
    if (rc) return rc;
    if (!(g > 0)) return infeasible(i, g, bad);
    if ((rc = barrier_eval(g, s->eps, &B, &dB, &ddB))) return rc;
    e += sample_kappa(s->type, P) * s->weight * s->gamma * B;
  }
  *energy = e;
  return GMCP_OK;
}

/* contact_energy.hpp:126-142 */
int orc_add_contact_gradient(const orc_state* S, const gmcp_barrier_params* P, const double* x, double* grad,
                             double* energy, int64_t* bad) {
  double e = 0;
  *bad = -1;
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    kin_t k;
    double B, dB, ddB;
    int rc = kinematics(s, x, 1, &k);
    if (rc) return rc;
    if (!(k.g > 0)) return infeasible(i, k.g, bad);
    if ((rc = barrier_eval(k.g, s->eps, &B, &dB, &ddB))) return rc;
    const double coef = sample_kappa(s->type, P) * s->weight * s->gamma;
    e += coef * B;
    for (int v = 0; v < k.nv; ++v) {
      const double f = coef * dB;
      for (int a = 0; a < 3; ++a) grad[3 * k.ids[v] + a] = grad[3 * k.ids[v] + a] + f * k.dg[v].v[a];
    }
  }
  *energy = e;
  return GMCP_OK;
}

/* 3x3 block accumulator keyed by (row, col): open addressing, insertion
 * order of first appearance kept so sums follow the triplet order. */
typedef struct {
  int64_t* key;
  int64_t* slot;
  int64_t cap, n;
  int32_t *row, *col;
  double* val;
  int64_t vcap;
} blockmap;

static int64_t bm_get(blockmap* m, int32_t r, int32_t c) {
  if (2 * (m->n + 1) > m->cap) {
    const int64_t oc = m->cap;
    int64_t* ok = m->key;
    int64_t* os = m->slot;
    m->cap = oc ? 2 * oc : 1024;
    m->key = (int64_t*)malloc(sizeof(int64_t) * (size_t)m->cap);
    m->slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)m->cap);
    for (int64_t i = 0; i < m->cap; ++i) m->key[i] = -1;
    for (int64_t i = 0; i < oc; ++i)
      if (ok[i] >= 0) {
        uint64_t h = ((uint64_t)ok[i] * 0x9E3779B97F4A7C15ull) & (uint64_t)(m->cap - 1);
        while (m->key[h] >= 0) h = (h + 1) & (uint64_t)(m->cap - 1);
        m->key[h] = ok[i];
        m->slot[h] = os[i];
      }
    free(ok);
    free(os);
  }
  const int64_t key = ((int64_t)r << 32) | (uint32_t)c;
  uint64_t h = ((uint64_t)key * 0x9E3779B97F4A7C15ull) & (uint64_t)(m->cap - 1);
  while (m->key[h] >= 0) {
    if (m->key[h] == key) return m->slot[h];
    h = (h + 1) & (uint64_t)(m->cap - 1);
  }
  if (m->n == m->vcap) {
    m->vcap = m->vcap ? 2 * m->vcap : 1024;
    m->row = (int32_t*)realloc(m->row, sizeof(int32_t) * (size_t)m->vcap);
    m->col = (int32_t*)realloc(m->col, sizeof(int32_t) * (size_t)m->vcap);
    m->val = (double*)realloc(m->val, sizeof(double) * 9 * (size_t)m->vcap);
  }
  m->key[h] = key;
  m->slot[h] = m->n;
  m->row[m->n] = r;
  m->col[m->n] = c;
  memset(m->val + 9 * m->n, 0, 9 * sizeof(double));
  return m->n++;
}

static blockmap* g_sort_map;
static int cmp_block(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  const blockmap* m = g_sort_map;
  if (m->row[i] != m->row[j]) return m->row[i] < m->row[j] ? -1 : 1;
  if (m->col[i] != m->col[j]) return m->col[i] < m->col[j] ? -1 : 1;
  return 0;
}

/* contact_energy.hpp:146-179 */
int orc_add_contact_gradient_hessian(const orc_state* S, const gmcp_barrier_params* P, const double* x,
                                     double* grad, double* energy, int64_t* bad, int64_t* n_blocks,
                                     int32_t* brow, int32_t* bcol, double* bval, int64_t* n_triplets) {
  double e = 0;
  int64_t ntrip = 0;
  *bad = -1;
  blockmap m;
  memset(&m, 0, sizeof m);
  int rc = GMCP_OK;
  for (int64_t i = 0; i < S->n && !rc; ++i) {
    const sample_t* s = &S->s[i];
    kin_t k;
    double B, dB, ddB;
    if ((rc = kinematics(s, x, 1, &k))) break;
    if (!(k.g > 0)) {
      rc = infeasible(i, k.g, bad);
      break;
    }
    if ((rc = barrier_eval(k.g, s->eps, &B, &dB, &ddB))) break;
    const double coef = sample_kappa(s->type, P) * s->weight * s->gamma;
    e += coef * B;
    const double h = coef * dmax(ddB, 0.0);
    for (int v = 0; v < k.nv; ++v) {
      const double f = coef * dB;
      for (int a = 0; a < 3; ++a) grad[3 * k.ids[v] + a] = grad[3 * k.ids[v] + a] + f * k.dg[v].v[a];
      if (h == 0) continue;
      for (int w = 0; w < k.nv; ++w) {
        int64_t slot = -1;
        for (int a = 0; a < 3; ++a) {
          const double va = k.dg[v].v[a];
          if (va == 0) continue;
          for (int c = 0; c < 3; ++c) {
            const double entry = h * (va * k.dg[w].v[c]);
            if (entry != 0) {
              if (slot < 0) slot = bm_get(&m, k.ids[v], k.ids[w]);
              double* b = m.val + 9 * slot + 3 * a + c;
              *b = *b + entry;
              ++ntrip;
            }
          }
        }
      }
    }
  }
  if (!rc) {
    *energy = e;
    *n_blocks = m.n;
    if (n_triplets) *n_triplets = ntrip;
    if (brow) {
      int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m.n > 0 ? m.n : 1));
      for (int64_t i = 0; i < m.n; ++i) order[i] = i;
      g_sort_map = &m;
      qsort(order, (size_t)m.n, sizeof(int64_t), cmp_block);
      for (int64_t i = 0; i < m.n; ++i) {
        brow[i] = m.row[order[i]];
        bcol[i] = m.col[order[i]];
        memcpy(bval + 9 * i, m.val + 9 * order[i], 9 * sizeof(double));
      }
      free(order);
    }
  }
  free(m.key);
  free(m.slot);
  free(m.row);
  free(m.col);
  free(m.val);
  return rc;
}

/* contact_energy.hpp:184-193 */
int orc_step_filter(const orc_state* S, const double* x, const double* dx, double* alpha) {
  double a = 1.0;
  for (int64_t i = 0; i < S->n; ++i) {
    kin_t k;
    const int rc = kinematics(&S->s[i], x, 1, &k);
    if (rc) return rc;
    double dgdx = 0;
    for (int v = 0; v < k.nv; ++v) dgdx += dot3(k.dg[v], ld3(dx, k.ids[v]));
    if (dgdx < 0) a = dmin(a, 0.9 * k.g / (-dgdx));
  }
  *alpha = a;
  return GMCP_OK;
}

/* contact_energy.hpp:198-213 */
int orc_displacement_cap(const orc_state* S, const gmcp_barrier_params* P, const double* x, const double* dx,
                         int64_t n_dof, double* alpha) {
  int active = 0;
  for (int64_t i = 0; i < S->n; ++i) {
    double g;
    const int rc = sample_gap_(&S->s[i], x, &g);
    if (rc) return rc;
    if (g < S->s[i].eps) {
      active = 1;
      break;
    }
  }
  if (!active) {
    *alpha = 1.0;
    return GMCP_OK;
  }
  double max_move = 0;
  for (int64_t v = 0; v < n_dof / 3; ++v) max_move = dmax(max_move, nrm3(ld3(dx, v)));
  *alpha = (max_move <= 0.5 * P->eps_max) ? 1.0 : 0.5 * P->eps_max / max_move;
  return GMCP_OK;
}

/* contact_energy.hpp:225-242 */
int orc_pressure_field(const orc_state* S, const gmcp_barrier_params* P, const double* x, int64_t* n,
                       gmcp_pressure_record* out) {
  int64_t m = 0;
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    if (s->type != GMCP_FACE) continue;
    if (out) {
      kin_t k;
      double B, dB, ddB;
      int rc = kinematics(s, x, 0, &k);
      if (rc) return rc;
      if ((rc = barrier_eval(k.g, s->eps, &B, &dB, &ddB))) return rc;
      out[m].sample = i;
      memcpy(out[m].position, k.xs.v, sizeof k.xs.v);
      out[m].radius = hypot(k.xs.v[0], k.xs.v[1]);
      out[m].gap = k.g;
      out[m].pressure = P->kappa_face * s->gamma * (-dB);
    }
    ++m;
  }
  *n = m;
  return GMCP_OK;
}

/* contact_energy.hpp:253-276 */
int orc_force_summary(const orc_state* S, const gmcp_barrier_params* P, const double* x, double* out) {
  v3 face = mk3(0, 0, 0), edge = face, point = face;
  for (int64_t i = 0; i < S->n; ++i) {
    const sample_t* s = &S->s[i];
    kin_t k;
    double B, dB, ddB;
    int rc = kinematics(s, x, 1, &k);
    if (rc) return rc;
    if (!(k.g > 0)) continue;
    const double coef = sample_kappa(s->type, P) * s->weight * s->gamma;
    v3 f = mk3(0, 0, 0);
    for (int v = 0; v < 3; ++v) {
      if ((rc = barrier_eval(k.g, s->eps, &B, &dB, &ddB))) return rc;
      f = sub3(f, scl3(coef * dB, k.dg[v]));
    }
    if (s->type == GMCP_FACE) face = add3(face, f);
    else if (s->type == GMCP_EDGE) edge = add3(edge, f);
    else point = add3(point, f);
  }
  const v3 total = add3(add3(face, edge), point);
  const v3 all[4] = {face, edge, point, total};
  for (int j = 0; j < 4; ++j) memcpy(out + 3 * j, all[j].v, sizeof all[j].v);
  return GMCP_OK;
}

int orc_time_assembly(const orc_state* S, const gmcp_barrier_params* P, const double* x, int32_t reps,
                      double* best_seconds, int64_t* n_triplets) {
  double best = 1e300;
  double* grad = (double*)calloc((size_t)(S->n_dof > 0 ? S->n_dof : 1), sizeof(double));
  for (int32_t r = 0; r < reps; ++r) {
    int64_t bad, nb;
    double e;
    memset(grad, 0, sizeof(double) * (size_t)S->n_dof);
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const int rc = orc_add_contact_gradient_hessian(S, P, x, grad, &e, &bad, &nb, NULL, NULL, NULL, n_triplets);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (rc) {
      free(grad);
      return rc;
    }
    const double dt = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    if (dt < best) best = dt;
  }
  free(grad);
  *best_seconds = best;
  return GMCP_OK;
}


/* ------------------------------------------------------------------------ */
/* embedding.hpp                                                             */

/* geometry.hpp:26-34 */
static int solve_barycentric_gram(v3 d, v3 e1, v3 e2, double* v, double* w) {
  const double a11 = dot3(e1, e1), a12 = dot3(e1, e2), a22 = dot3(e2, e2);
  const double b1 = dot3(d, e1), b2 = dot3(d, e2);
  const double det = a11 * a22 - a12 * a12;
  const double gram_eps = 1e-14 * a11 * a22;
  if (!(det > gram_eps)) return set_err(GMCP_ERR_DEGENERATE, "solve_barycentric_gram: near-degenerate edge basis");
  *v = (a22 * b1 - a12 * b2) / det;
  *w = (a11 * b2 - a12 * b1) / det;
  return GMCP_OK;
}

/* geometry.hpp:45-103: closest point on the closed triangle (Voronoi regions) */
static v3 closest_point_on_triangle(v3 p, v3 a, v3 b, v3 c) {
  const v3 ab = sub3(b, a), ac = sub3(c, a), ap = sub3(p, a);
  const double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0 && d2 <= 0) return a;
  const v3 bp = sub3(p, b);
  const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0 && d4 <= d3) return b;
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    const double v = d1 / (d1 - d3);
    return add3(a, scl3(v, ab));
  }
  const v3 cp = sub3(p, c);
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0 && d5 <= d6) return c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    const double w = d2 / (d2 - d6);
    return add3(a, scl3(w, ac));
  }
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return add3(b, scl3(w, sub3(c, b)));
  }
  const double denom = 1.0 / ((va + vb) + vc);
  const double v = vb * denom, w = vc * denom;
  return add3(add3(a, scl3(v, ab)), scl3(w, ac));
}

/* embedding.hpp:26-84 (brute-force scan == the tree's result: min squared
 * distance, lowest triangle index on exact ties) */
int orc_embed_in_surface(const double* points, int64_t n_points, const double* host_v, int64_t n_hv,
                         const int32_t* host_t, int64_t n_ht, int32_t use_tree, int32_t* tri, double* bary,
                         double* offset, int64_t* bad) {
  (void)n_hv;
  (void)use_tree;
  *bad = -1;
  if (n_ht <= 0) return set_err(GMCP_ERR_CONFIG, "embedding host has no triangles");
  for (int64_t t = 0; t < n_ht; ++t) {
    const v3 a = ld3(host_v, host_t[3 * t]), b = ld3(host_v, host_t[3 * t + 1]), c = ld3(host_v, host_t[3 * t + 2]);
    if (!(nrm3(crs3(sub3(b, a), sub3(c, a))) > 0)) {
      *bad = t;
      return set_err(GMCP_ERR_DEGENERATE, "embedding host triangle is degenerate");
    }
  }
  for (int64_t i = 0; i < n_points; ++i) {
    const v3 p = ld3(points, i);
    int64_t best = -1;
    double best_d2 = DBL_MAX;
    for (int64_t t = 0; t < n_ht; ++t) {
      const v3 a = ld3(host_v, host_t[3 * t]), b = ld3(host_v, host_t[3 * t + 1]), c = ld3(host_v, host_t[3 * t + 2]);
      v3 n;
      if (triangle_normal(a, b, c, &n) != GMCP_OK) return GMCP_ERR_DEGENERATE;  /* closest_point_on_triangle */
      const v3 q = sub3(closest_point_on_triangle(p, a, b, c), p);
      const double d2 = dot3(q, q);
      if (d2 < best_d2) {
        best_d2 = d2;
        best = t;
      }
    }
    const v3 a = ld3(host_v, host_t[3 * best]), b = ld3(host_v, host_t[3 * best + 1]), c = ld3(host_v, host_t[3 * best + 2]);
    v3 n;
    if (triangle_normal(a, b, c, &n) != GMCP_OK) return GMCP_ERR_DEGENERATE;
    const v3 d = sub3(p, a);
    double v, w;
    if (solve_barycentric_gram(d, sub3(b, a), sub3(c, a), &v, &w) != GMCP_OK) return GMCP_ERR_DEGENERATE;
    tri[i] = (int32_t)best;
    bary[3 * i] = (1.0 - v) - w;
    bary[3 * i + 1] = v;
    bary[3 * i + 2] = w;
    offset[i] = dot3(n, d);
  }
  return GMCP_OK;
}

/* embedding.hpp:87-106 */
int orc_apply_embedding(const int32_t* tri, const double* bary, const double* offset, int64_t n,
                        const int32_t* host_t, int64_t n_ht, const double* host_x, int64_t n_hv, double* out,
                        int64_t* bad) {
  (void)n_ht;
  (void)n_hv;
  *bad = -1;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t* t = host_t + 3 * (int64_t)tri[i];
    const v3 v0 = ld3(host_x, t[0]), v1 = ld3(host_x, t[1]), v2 = ld3(host_x, t[2]);
    v3 nn;
    if (triangle_normal(v0, v1, v2, &nn) != GMCP_OK) {
      *bad = tri[i];
      return set_err(GMCP_ERR_DEGENERATE, "host triangle is degenerate in the deformed configuration");
    }
    const v3 r = add3(add3(add3(scl3(bary[3 * i], v0), scl3(bary[3 * i + 1], v1)), scl3(bary[3 * i + 2], v2)),
                      scl3(offset[i], nn));
    out[3 * i] = r.v[0];
    out[3 * i + 1] = r.v[1];
    out[3 * i + 2] = r.v[2];
  }
  return GMCP_OK;
}
