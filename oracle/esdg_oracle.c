/* esdg_oracle.c -- see esdg_oracle.h. TEST INFRASTRUCTURE ONLY.
 *
 * Precision-independent pieces (mesh, Morton order, LGL operators, flux
 * schedule, partition, exchange plan, initial-condition cases) live here; the
 * precision-generic solver is in esdg_oracle_impl.inc, included twice below.
 *
 * Build: gcc -std=c99 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps the arithmetic identical to the reference built
 * for baseline x86-64 (no FMA), which is what the bitwise pin relies on.
 */
#define _GNU_SOURCE
#include "esdg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#ifndef M_LN2
#define M_LN2 0.69314718055994530942
#endif

/* ======================================================================== */
/* Morton key (include/esdg/morton.hpp:9-26)                                 */
/* ======================================================================== */

static uint64_t spread_every_third(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | (x << 32)) & 0x1f00000000ffffull;
  x = (x | (x << 16)) & 0x1f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

uint64_t orc_morton_key(uint32_t i, uint32_t j, uint32_t k) {
  return spread_every_third(i) | (spread_every_third(j) << 1) |
         (spread_every_third(k) << 2);
}

/* ======================================================================== */
/* Mesh (src/mesh.cpp:11-132)                                                */
/* ======================================================================== */

struct orc_mesh {
  orc_mesh_config cfg;
  int32_t dims[3];
  double delta[3];
  double jacobian;
  int64_t ne;
  int32_t* lattice; /* ne*3 */
  int64_t* elem_at; /* lattice index -> element id */
  int32_t nfaces;
  int32_t faces_cap;
  orc_face* faces;
  int32_t* face_of; /* ne*6 */
};

typedef struct {
  uint64_t key;
  int64_t raw;
} morton_entry;

static int morton_entry_cmp(const void* pa, const void* pb) {
  const morton_entry* a = (const morton_entry*)pa;
  const morton_entry* b = (const morton_entry*)pb;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  if (a->raw != b->raw) return a->raw < b->raw ? -1 : 1;
  return 0;
}

static size_t lattice_index(const orc_mesh* m, int i, int j, int k) {
  return (size_t)i + (size_t)m->dims[0] * ((size_t)j + (size_t)m->dims[1] * (size_t)k);
}

static int32_t push_face(orc_mesh* m, orc_face f) {
  if (m->nfaces == m->faces_cap) {
    m->faces_cap = m->faces_cap ? 2 * m->faces_cap : 64;
    m->faces = (orc_face*)realloc(m->faces, sizeof(orc_face) * (size_t)m->faces_cap);
  }
  m->faces[m->nfaces] = f;
  return m->nfaces++;
}

/* src/mesh.cpp:78-132: per element in Morton order, per direction: the hi
 * face (interior / periodic wrap / reflecting), then the lo reflecting face
 * of first-layer elements. The lower-index element of an interior face is its
 * minus side. */
static void build_faces(orc_mesh* m) {
  m->face_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)m->ne * 6);
  for (int64_t i = 0; i < m->ne * 6; ++i) m->face_of[i] = -1;
  for (int64_t e = 0; e < m->ne; ++e) {
    const int32_t* lat = m->lattice + 3 * e;
    for (int d = 0; d < 3; ++d) {
      const int next = lat[d] + 1;
      const int wraps = next == m->dims[d];
      if (wraps && m->cfg.bc[d] == 1) {
        orc_face f = {(int32_t)e, -1, (uint8_t)d, 1, 1, 0};
        m->face_of[e * 6 + d * 2 + 1] = push_face(m, f);
      } else {
        int c[3] = {lat[0], lat[1], lat[2]};
        c[d] = wraps ? 0 : next;
        const int64_t nbr = m->elem_at[lattice_index(m, c[0], c[1], c[2])];
        orc_face f = {-1, -1, (uint8_t)d, 1, 0, 0};
        if (nbr >= e) {
          f.minus_elem = (int32_t)e;
          f.plus_elem = (int32_t)nbr;
          f.minus_side = 1;
        } else {
          f.minus_elem = (int32_t)nbr;
          f.plus_elem = (int32_t)e;
          f.minus_side = 0;
        }
        const int32_t id = push_face(m, f);
        m->face_of[e * 6 + d * 2 + 1] = id;
        m->face_of[nbr * 6 + d * 2 + 0] = id;
      }
      if (lat[d] == 0 && m->cfg.bc[d] == 1) {
        orc_face f = {(int32_t)e, -1, (uint8_t)d, 0, 1, 0};
        m->face_of[e * 6 + d * 2 + 0] = push_face(m, f);
      }
    }
  }
}

orc_mesh* orc_mesh_create(const orc_mesh_config* cfg) {
  for (int d = 0; d < 3; ++d) {
    if (cfg->base[d] < 1) return NULL;
    if (!(cfg->hi[d] > cfg->lo[d])) return NULL;
  }
  if (cfg->refinement < 0 || cfg->refinement > 20) return NULL;
  orc_mesh* m = (orc_mesh*)calloc(1, sizeof(orc_mesh));
  m->cfg = *cfg;
  const int64_t scale = (int64_t)1 << cfg->refinement;
  int64_t ne = 1;
  for (int d = 0; d < 3; ++d) {
    const int64_t n = cfg->base[d] * scale;
    if (n > ((int64_t)1 << 21)) {
      free(m);
      return NULL;
    }
    m->dims[d] = (int32_t)n;
    ne *= n;
    m->delta[d] = (cfg->hi[d] - cfg->lo[d]) / (double)n;
  }
  if (ne > ((int64_t)1 << 50)) {
    free(m);
    return NULL;
  }
  m->ne = ne;
  m->jacobian = 0.125 * m->delta[0] * m->delta[1] * m->delta[2];

  /* global Morton order: interleave, then sort (src/mesh.cpp:43-66) */
  morton_entry* ent = (morton_entry*)malloc(sizeof(morton_entry) * (size_t)ne);
  int64_t at = 0;
  for (int k = 0; k < m->dims[2]; ++k)
    for (int j = 0; j < m->dims[1]; ++j)
      for (int i = 0; i < m->dims[0]; ++i) {
        ent[at].key = orc_morton_key((uint32_t)i, (uint32_t)j, (uint32_t)k);
        ent[at].raw = at;
        ++at;
      }
  qsort(ent, (size_t)ne, sizeof(morton_entry), morton_entry_cmp);
  m->lattice = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)ne);
  m->elem_at = (int64_t*)malloc(sizeof(int64_t) * (size_t)ne);
  for (int64_t e = 0; e < ne; ++e) {
    const int64_t raw = ent[e].raw;
    m->lattice[3 * e + 0] = (int32_t)(raw % m->dims[0]);
    m->lattice[3 * e + 1] = (int32_t)((raw / m->dims[0]) % m->dims[1]);
    m->lattice[3 * e + 2] = (int32_t)(raw / ((int64_t)m->dims[0] * m->dims[1]));
    m->elem_at[raw] = e;
  }
  free(ent);
  build_faces(m);
  return m;
}

void orc_mesh_destroy(orc_mesh* m) {
  if (!m) return;
  free(m->lattice);
  free(m->elem_at);
  free(m->faces);
  free(m->face_of);
  free(m);
}

int64_t orc_mesh_num_elements(const orc_mesh* m) { return m->ne; }
int32_t orc_mesh_num_faces(const orc_mesh* m) { return m->nfaces; }
void orc_mesh_dims(const orc_mesh* m, int32_t dims[3]) {
  for (int d = 0; d < 3; ++d) dims[d] = m->dims[d];
}
void orc_mesh_delta(const orc_mesh* m, double delta[3]) {
  for (int d = 0; d < 3; ++d) delta[d] = m->delta[d];
}
double orc_mesh_jacobian(const orc_mesh* m) { return m->jacobian; }
const int32_t* orc_mesh_lattice(const orc_mesh* m) { return m->lattice; }
const orc_face* orc_mesh_faces(const orc_mesh* m) { return m->faces; }
const int32_t* orc_mesh_face_of(const orc_mesh* m) { return m->face_of; }

/* include/esdg/mesh.hpp:73-77 */
double orc_mesh_node_coordinate(const orc_mesh* m, int64_t elem, int dir,
                                double ref_node) {
  const int32_t* lat = m->lattice + 3 * elem;
  return m->cfg.lo[dir] +
         ((double)lat[dir] + 0.5 * (ref_node + 1.0)) * m->delta[dir];
}

/* include/esdg/mesh.hpp:107-114: face node (s,t) -> element node */
static int face_node(int nq, int dir, int side, int fnode) {
  const int s = fnode % nq, t = fnode / nq;
  int c[3];
  c[dir] = side ? nq - 1 : 0;
  c[(dir + 1) % 3] = s;
  c[(dir + 2) % 3] = t;
  return c[0] + nq * (c[1] + nq * c[2]);
}

/* ======================================================================== */
/* LGL reference element (src/reference_element.cpp:11-138)                  */
/* ======================================================================== */

typedef struct {
  double p, dp;
} legendre_pair;

/* three-term recurrence; P_N' from N (x P_N - P_{N-1}) / (x^2 - 1) */
static legendre_pair legendre_eval(int n, double x) {
  legendre_pair r;
  if (n == 0) {
    r.p = 1.0;
    r.dp = 0.0;
    return r;
  }
  double below = 1.0, cur = x;
  for (int k = 2; k <= n; ++k) {
    const double nxt = ((2.0 * k - 1.0) * x * cur - (k - 1.0) * below) / k;
    below = cur;
    cur = nxt;
  }
  if (fabs(x) == 1.0) {
    if (x == 1.0)
      r.dp = n * (n + 1) / 2.0;
    else
      r.dp = ((n % 2 == 0) ? -1.0 : 1.0) * n * (n + 1) / 2.0;
  } else {
    r.dp = n * (x * cur - below) / (x * x - 1.0);
  }
  r.p = cur;
  return r;
}

static double lobatto_poly(int n, double x) {
  return (1.0 - x * x) * legendre_eval(n, x).dp;
}

/* safeguarded Newton on q(x) = (1-x^2) P_N'(x) inside [lo, hi]
 * (src/reference_element.cpp:36-71) */
static int lgl_root(int n, double lo, double hi, double* root) {
  double qlo = lobatto_poly(n, lo), qhi = lobatto_poly(n, hi);
  for (int k = 0; k < 8 && ((qlo > 0) == (qhi > 0)); ++k) {
    const double w = 0.25 * (hi - lo);
    lo = fmax(lo - w, -1.0 + 1e-14);
    hi = fmin(hi + w, 1.0 - 1e-14);
    qlo = lobatto_poly(n, lo);
    qhi = lobatto_poly(n, hi);
  }
  if ((qlo > 0) == (qhi > 0)) return -1;
  double x = 0.5 * (lo + hi);
  for (int it = 0; it < 200; ++it) {
    const double qx = lobatto_poly(n, x);
    if (qx == 0.0) break;
    if ((qx > 0) == (qlo > 0)) {
      lo = x;
      qlo = qx;
    } else {
      hi = x;
    }
    const double dq = -(double)n * (n + 1) * legendre_eval(n, x).p;
    double xn = (dq != 0.0) ? x - qx / dq : x;
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    if (xn == x) break;
    x = xn;
    if (hi - lo <= 2.0 * fabs(x) * 2.220446049250313e-16) break;
  }
  *root = x;
  return 0;
}

/* barycentric D, diagonal = -rowsum (src/reference_element.cpp:119-138) */
static void diff_matrix(int nq, const double* x, double* d) {
  double* lam = (double*)malloc(sizeof(double) * (size_t)nq);
  for (int i = 0; i < nq; ++i) {
    lam[i] = 1.0;
    for (int j = 0; j < nq; ++j)
      if (j != i) lam[i] /= (x[i] - x[j]);
  }
  for (int i = 0; i < nq; ++i) {
    double rowsum = 0.0;
    for (int j = 0; j < nq; ++j) {
      if (j == i) continue;
      const double dij = (lam[j] / lam[i]) / (x[i] - x[j]);
      d[i * nq + j] = dij;
      rowsum += dij;
    }
    d[i * nq + i] = -rowsum;
  }
  free(lam);
}

int orc_reference_element(int order, double* nodes, double* weights,
                          double* diff) {
  if (order < 1 || order > 32) return -1;
  const int nq = order + 1;
  for (int i = 0; i < nq; ++i) nodes[i] = weights[i] = 0.0;
  nodes[0] = -1.0;
  nodes[nq - 1] = 1.0;
  double* guess = (double*)malloc(sizeof(double) * (size_t)nq);
  for (int i = 0; i < nq; ++i) guess[i] = -cos(M_PI * i / order);
  const int first = nq / 2 + (nq % 2);
  for (int i = first; i < nq - 1; ++i) {
    double lo = 0.5 * (guess[i - 1] + guess[i]);
    double hi = 0.5 * (guess[i] + guess[i + 1]);
    if (i == first && nq % 2 == 0) lo = 0.0;
    double x;
    if (lgl_root(order, lo, hi, &x) != 0) {
      free(guess);
      return -1;
    }
    nodes[i] = x;
    nodes[nq - 1 - i] = -x;
  }
  free(guess);
  if (nq % 2 == 1) nodes[nq / 2] = 0.0;

  const double wf = 2.0 / ((double)order * (order + 1));
  for (int i = 0; i < nq; ++i) {
    if (2 * i < nq) continue;
    const double p = legendre_eval(order, nodes[i]).p;
    weights[i] = wf / (p * p);
    weights[nq - 1 - i] = weights[i];
  }
  if (nq % 2 == 1) {
    const double p = legendre_eval(order, 0.0).p;
    weights[nq / 2] = wf / (p * p);
  }
  diff_matrix(nq, nodes, diff);
  return 0;
}

/* ======================================================================== */
/* Flux schedule (src/schedule.cpp:8-43)                                     */
/* ======================================================================== */

int orc_schedule(int nq, int variant, int16_t* partner_index,
                 int16_t* half_weight, int32_t* offsets) {
  if (nq < 2) return -1;
  const int half = nq / 2;
  int total = 0;
  offsets[0] = 0;
  for (int i = 0; i < nq; ++i) {
    int count = half;
    if (variant == 0 && nq % 2 == 0) count = i < half ? half : half - 1;
    int16_t idx[64], hw[64];
    for (int o = 1; o <= count; ++o) {
      idx[o - 1] = (int16_t)((i + o) % nq);
      hw[o - 1] = (variant == 1 && nq % 2 == 0 && o == half) ? 1 : 2;
    }
    /* ascending partner index (insertion sort; count <= 16) */
    for (int a = 1; a < count; ++a) {
      const int16_t ki = idx[a], kh = hw[a];
      int b = a - 1;
      while (b >= 0 && idx[b] > ki) {
        idx[b + 1] = idx[b];
        hw[b + 1] = hw[b];
        --b;
      }
      idx[b + 1] = ki;
      hw[b + 1] = kh;
    }
    for (int a = 0; a < count; ++a) {
      partner_index[total] = idx[a];
      half_weight[total] = hw[a];
      ++total;
    }
    offsets[i + 1] = total;
  }
  return total;
}

/* ======================================================================== */
/* Partition and exchange plan (src/partition.cpp:13-66)                     */
/* ======================================================================== */

int orc_partition(int64_t n_elements, int ranks, int64_t* range_begin) {
  if (ranks < 1 || ranks > n_elements) return -1;
  const int64_t base = n_elements / ranks, rem = n_elements % ranks;
  int64_t at = 0;
  for (int r = 0; r < ranks; ++r) {
    range_begin[r] = at;
    at += base + (r < rem ? 1 : 0);
  }
  range_begin[ranks] = at;
  return 0;
}

static int rank_of_elem(const int64_t* range_begin, int ranks, int64_t e) {
  int r = 0;
  while (r + 1 < ranks && e >= range_begin[r + 1]) ++r;
  return r;
}

int orc_exchange_plan(const orc_mesh* m, int ranks, int32_t* ghost_count,
                      int32_t* interior_count, orc_ghost_face* ghosts,
                      int32_t* interior) {
  int64_t* rb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ranks + 1));
  if (orc_partition(m->ne, ranks, rb) != 0) {
    free(rb);
    return -1;
  }
  /* pass 1: counts */
  int32_t* gc = (int32_t*)calloc((size_t)ranks, sizeof(int32_t));
  int32_t* ic = (int32_t*)calloc((size_t)ranks, sizeof(int32_t));
  for (int32_t f = 0; f < m->nfaces; ++f) {
    const orc_face* fc = &m->faces[f];
    const int rm = rank_of_elem(rb, ranks, fc->minus_elem);
    if (fc->reflecting || fc->plus_elem < 0 ||
        rank_of_elem(rb, ranks, fc->plus_elem) == rm) {
      ++ic[rm];
    } else {
      ++gc[rm];
      ++gc[rank_of_elem(rb, ranks, fc->plus_elem)];
    }
  }
  int n_ghost = 0;
  if (ghosts && interior) {
    int32_t* goff = (int32_t*)calloc((size_t)ranks + 1, sizeof(int32_t));
    int32_t* ioff = (int32_t*)calloc((size_t)ranks + 1, sizeof(int32_t));
    for (int r = 0; r < ranks; ++r) {
      goff[r + 1] = goff[r] + gc[r];
      ioff[r + 1] = ioff[r] + ic[r];
    }
    int32_t* gfill = (int32_t*)calloc((size_t)ranks, sizeof(int32_t));
    int32_t* ifill = (int32_t*)calloc((size_t)ranks, sizeof(int32_t));
    for (int32_t f = 0; f < m->nfaces; ++f) {
      const orc_face* fc = &m->faces[f];
      const int rm = rank_of_elem(rb, ranks, fc->minus_elem);
      if (fc->reflecting || fc->plus_elem < 0 ||
          rank_of_elem(rb, ranks, fc->plus_elem) == rm) {
        interior[ioff[rm] + ifill[rm]++] = f;
        continue;
      }
      const int rp = rank_of_elem(rb, ranks, fc->plus_elem);
      const int32_t box_minus = 2 * n_ghost, box_plus = 2 * n_ghost + 1;
      orc_ghost_face gm = {f, rp, 0, gfill[rm], box_minus, box_plus};
      ghosts[goff[rm] + gfill[rm]++] = gm;
      orc_ghost_face gp = {f, rm, 1, gfill[rp], box_plus, box_minus};
      ghosts[goff[rp] + gfill[rp]++] = gp;
      ++n_ghost;
    }
    free(goff);
    free(ioff);
    free(gfill);
    free(ifill);
  } else {
    for (int r = 0; r < ranks; ++r) n_ghost += gc[r];
    n_ghost /= 2;
  }
  for (int r = 0; r < ranks; ++r) {
    if (ghost_count) ghost_count[r] = gc[r];
    if (interior_count) interior_count[r] = ic[r];
  }
  free(gc);
  free(ic);
  free(rb);
  return 2 * n_ghost;
}

/* ======================================================================== */
/* Cases (include/esdg/cases.hpp:15-156)                                     */
/* ======================================================================== */

static double gas_cv(const orc_gas* g) { return g->R / (g->gamma - 1.0); }
static double gas_cp(const orc_gas* g) { return g->gamma * gas_cv(g); }

/* isentropic hydrostatic column with optional theta perturbation at constant
 * pressure (cases.hpp:18-38 for dtheta = 0, :58-69 otherwise). The two
 * reference functions differ only in T = theta0*pi vs (theta0+dtheta)*pi. */
static int column_state(const orc_gas* g, double theta0, double dtheta,
                        int perturbed, double z, double phi, double q[5]) {
  const double pi = 1.0 - g->gravity * z / (gas_cp(g) * theta0);
  if (pi <= 0.0) return -1;
  double T;
  if (perturbed) {
    const double theta = theta0 + dtheta;
    T = theta * pi;
  } else {
    T = theta0 * pi;
  }
  const double p = g->p0 * pow(pi, gas_cp(g) / g->R);
  const double rho = p / (g->R * T);
  q[0] = rho;
  q[1] = q[2] = q[3] = 0.0;
  q[4] = rho * (gas_cv(g) * T + phi);
  return 0;
}

/* cases.hpp:40-55 */
static double bubble_dtheta(double x, double y, double z, int sharp) {
  const double dx = x - 0.0, dy = y - 0.0, dz = z - 260.0;
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  if (r > 250.0) return 0.0;
  if (sharp) return 0.5;
  return 0.5 * 0.5 * (1.0 + cos(M_PI * r / 250.0));
}

/* cases.hpp:72-84 */
static uint64_t splitmix64_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double unit_real_next(uint64_t* s) {
  return (double)(splitmix64_next(s) >> 11) * (1.0 / 9007199254740992.0);
}

/* cases.hpp:86-118 */
typedef struct {
  int k[3][3];
  double amp[3];
  double phase[3];
} fourier_field;

static fourier_field fourier_field_make(uint64_t* s) {
  fourier_field f;
  for (int m = 0; m < 3; ++m) {
    for (int d = 0; d < 3; ++d) f.k[m][d] = 1 + (int)(splitmix64_next(s) % 2);
    f.amp[m] = (2.0 * unit_real_next(s) - 1.0) / 3;
    f.phase[m] = 2.0 * M_PI * unit_real_next(s);
  }
  return f;
}

static double fourier_field_value(const fourier_field* f, const double xh[3]) {
  double v = 0.0;
  for (int m = 0; m < 3; ++m)
    v += f->amp[m] *
         sin(2.0 * M_PI * (f->k[m][0] * xh[0] + f->k[m][1] * xh[1] +
                           f->k[m][2] * xh[2]) +
             f->phase[m]);
  return v;
}

/* cases.hpp:120-156 */
typedef struct {
  double lo[3], hi[3];
  orc_gas gas;
  fourier_field rho_f, p_f, u_f[3];
} entropy_test_gen;

static entropy_test_gen entropy_test_make(const orc_mesh_config* mc,
                                          const orc_gas* g, uint64_t seed) {
  entropy_test_gen t;
  for (int d = 0; d < 3; ++d) {
    t.lo[d] = mc->lo[d];
    t.hi[d] = mc->hi[d];
  }
  t.gas = *g;
  uint64_t s = seed;
  t.rho_f = fourier_field_make(&s);
  t.p_f = fourier_field_make(&s);
  for (int d = 0; d < 3; ++d) t.u_f[d] = fourier_field_make(&s);
  return t;
}

static void entropy_test_state(const entropy_test_gen* t, double x, double y,
                               double z, double phi, double q[5]) {
  const double xh[3] = {(x - t->lo[0]) / (t->hi[0] - t->lo[0]),
                        (y - t->lo[1]) / (t->hi[1] - t->lo[1]),
                        (z - t->lo[2]) / (t->hi[2] - t->lo[2])};
  const double rho = 1.16 * (1.0 + 0.05 * fourier_field_value(&t->rho_f, xh));
  const double p = t->gas.p0 * (1.0 + 0.05 * fourier_field_value(&t->p_f, xh));
  const double u[3] = {15.0 * fourier_field_value(&t->u_f[0], xh),
                       15.0 * fourier_field_value(&t->u_f[1], xh),
                       15.0 * fourier_field_value(&t->u_f[2], xh)};
  q[0] = rho;
  q[1] = rho * u[0];
  q[2] = rho * u[1];
  q[3] = rho * u[2];
  q[4] = p / (t->gas.gamma - 1.0) +
         0.5 * rho * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]) + rho * phi;
}

/* evaluates the named case at one point; returns 0 or -1 */
typedef struct {
  int case_id;
  orc_gas gas;
  entropy_test_gen et;
  double cst[5];
} case_eval;

static int case_point(const case_eval* c, double x, double y, double z,
                      double phi, double q[5]) {
  switch (c->case_id) {
    case ORC_CASE_BUBBLE_SHARP:
      return column_state(&c->gas, 300.0, bubble_dtheta(x, y, z, 1), 1, z, phi, q);
    case ORC_CASE_BUBBLE_SMOOTH:
      return column_state(&c->gas, 300.0, bubble_dtheta(x, y, z, 0), 1, z, phi, q);
    case ORC_CASE_HYDROSTATIC:
      return column_state(&c->gas, 300.0, 0.0, 0, z, phi, q);
    case ORC_CASE_ENTROPY_TEST:
      entropy_test_state(&c->et, x, y, z, phi, q);
      return 0;
    case ORC_CASE_CONSTANT: {
      /* tests/test_helpers.hpp:41-52 */
      const double rho = c->cst[0], u1 = c->cst[1], u2 = c->cst[2],
                   u3 = c->cst[3], p = c->cst[4];
      q[0] = rho;
      q[1] = rho * u1;
      q[2] = rho * u2;
      q[3] = rho * u3;
      q[4] = p / (c->gas.gamma - 1.0) +
             0.5 * rho * (u1 * u1 + u2 * u2 + u3 * u3) + rho * phi;
      return 0;
    }
  }
  return -1;
}

/* ======================================================================== */
/* LSRK(5,4) (include/esdg/time_integration.hpp:17-37)                       */
/* ======================================================================== */

static const double kLsrkA[5] = {0.0, -567301805773.0 / 1357537059087.0,
                                 -2404267990393.0 / 2016746695238.0,
                                 -3550918686646.0 / 2091501179385.0,
                                 -1275806237668.0 / 842570457699.0};
static const double kLsrkB[5] = {1432997174477.0 / 9575080441755.0,
                                 5161836677717.0 / 13612068292357.0,
                                 1720146321549.0 / 2090206949498.0,
                                 3134564353537.0 / 4481467310338.0,
                                 2277821191437.0 / 14882151754819.0};
static const double kLsrkC[5] = {0.0, 1432997174477.0 / 9575080441755.0,
                                 2526269341429.0 / 6820363962896.0,
                                 2006345519317.0 / 3224310063776.0,
                                 2802321613138.0 / 2924317926251.0};

void orc_lsrk_coefficients(double a[5], double b[5], double c[5]) {
  for (int s = 0; s < 5; ++s) {
    a[s] = kLsrkA[s];
    b[s] = kLsrkB[s];
    c[s] = kLsrkC[s];
  }
}

uint64_t orc_fnv1a64(const void* data, uint64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* Neumaier-compensated sum (include/esdg/diagnostics.hpp:17-26) */
typedef struct {
  double s, comp;
} neumaier;
static void neumaier_add(neumaier* k, double x) {
  const double t = k->s + x;
  k->comp += (fabs(k->s) >= fabs(x)) ? (k->s - t) + x : (x - t) + k->s;
  k->s = t;
}

/* ======================================================================== */
/* precision-generic solver, instantiated twice                              */
/* ======================================================================== */

#define REAL double
#define SUF(name) name##_f64
#define R_LOG log
#define R_SQRT sqrt
#define R_ABS fabs
#define R_SERIES_THRESHOLD_SQ 1e-8
#define R_SERIES_TERMS 3
#include "esdg_oracle_impl.inc"
#undef REAL
#undef SUF
#undef R_LOG
#undef R_SQRT
#undef R_ABS
#undef R_SERIES_THRESHOLD_SQ
#undef R_SERIES_TERMS

#define REAL float
#define SUF(name) name##_f32
#define R_LOG logf
#define R_SQRT sqrtf
#define R_ABS fabsf
#define R_SERIES_THRESHOLD_SQ 1e-4f
#define R_SERIES_TERMS 1
#include "esdg_oracle_impl.inc"
