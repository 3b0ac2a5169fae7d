/*
 * ffo_oracle.c -- CPU ORACLE for the UCCSD state-vector hot path.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference). The product never links it.
 *
 * Written as a literal restatement of the reference SPEC (file:line cited per
 * function), favouring per-qubit loops over bit tricks so that it shares no
 * code or shortcuts with the CUDA product path.
 *
 * PARITY UNPINNED against the reference: the reference holds no code, golden
 * vectors or fixtures for this path, and it cannot be built here
 * (Eigen3, doctest absent), so there is no oracle/_ref. What pins this oracle
 * instead (tests/test_oracle.py, tests/test_golden.py, tools/make_golden.py):
 * every SPEC example and KAT, dense numpy/scipy matrices at <= 10 qubits, the
 * agreement of its two evaluators (Pauli-string rotations; JW-free fermionic
 * Givens rotations on determinants), scipy sparse matrix exponentials at configs
 * 1-3 (tests/sparse_ref.py), the mt19937_64 known answer, and the reference's one
 * number on the path (proj/tests/test_fmo.cpp:182-185).
 */
#include "ffo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================================================================== */
/* mt19937_64 -- the C++ standard's generator, restated (raw output).       */
/* Value mapping (pinned):                    */
/*   U[0,1)  = (x >> 11) * 2^-53                                            */
/*   N(0,1)  = sqrt(-2 ln(1-U1)) * cos(2 pi U2)   (one normal per 2 draws)  */
/* ======================================================================== */
typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int k = 1; k < 312; ++k)
    s->mt[k] = 6364136223846793005ULL * (s->mt[k - 1] ^ (s->mt[k - 1] >> 62)) + (uint64_t)k;
  s->i = 312;
}

static uint64_t mt64_next(mt64* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (s->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (s->mt[k] & UM) | (s->mt[(k + 1) % 312] & LM);
      uint64_t v = s->mt[(k + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= A;
      s->mt[k] = v;
    }
    s->i = 0;
  }
  uint64_t x = s->mt[s->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double mt64_uniform(mt64* s) { return (double)(mt64_next(s) >> 11) * (1.0 / 9007199254740992.0); }

static double mt64_normal(mt64* s) {
  double u1 = mt64_uniform(s);
  double u2 = mt64_uniform(s);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

uint64_t ffo_mt64_nth(uint64_t seed, int nth) {
  mt64 s;
  mt64_seed(&s, seed);
  uint64_t v = 0;
  for (int k = 0; k < nth; ++k) v = mt64_next(&s);
  return v;
}

void ffo_uniform_array(uint64_t seed, int count, double lo, double hi, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (int k = 0; k < count; ++k) out[k] = lo + (hi - lo) * mt64_uniform(&s);
}

/* BASELINE.json configs: symmetric h ~ N(0, sigma_h), 8-fold symmetric
 * chemists' (pq|rs) ~ N(0, sigma_g); canonical quadruples drawn in the loop
 * order p, q<=p, r<=p, s<=(r==p ? q : r). */
void ffo_synthetic_integrals(int m, uint64_t seed, double sigma_h, double sigma_g,
                             double* h, double* g) {
  mt64 s;
  mt64_seed(&s, seed);
  for (int p = 0; p < m; ++p)
    for (int q = 0; q <= p; ++q) {
      double v = sigma_h * mt64_normal(&s);
      h[p * m + q] = v;
      h[q * m + p] = v;
    }
#define G4(a, b, c, d) g[(((size_t)(a) * m + (b)) * m + (c)) * m + (d)]
  for (int p = 0; p < m; ++p)
    for (int q = 0; q <= p; ++q)
      for (int r = 0; r <= p; ++r) {
        int smax = (r == p) ? q : r;
        for (int t = 0; t <= smax; ++t) {
          double v = sigma_g * mt64_normal(&s);
          G4(p, q, r, t) = v; G4(q, p, r, t) = v; G4(p, q, t, r) = v; G4(q, p, t, r) = v;
          G4(r, t, p, q) = v; G4(t, r, p, q) = v; G4(r, t, q, p) = v; G4(t, r, q, p) = v;
        }
      }
#undef G4
}

/* ======================================================================== */
/* Pauli algebra. Letters per qubit: I, X, Y, Z.          */
/* Multiplication done letter by letter with the textbook table.            */
/* ======================================================================== */
enum { LI = 0, LX = 1, LY = 2, LZ = 3 };

static int letter_of(uint64_t x, uint64_t z, int q) {
  int xb = (int)((x >> q) & 1), zb = (int)((z >> q) & 1);
  if (xb && zb) return LY;
  if (xb) return LX;
  if (zb) return LZ;
  return LI;
}

/* a*b = i^phase * c for single-qubit letters */
static int letter_mul(int a, int b, int* c) {
  if (a == LI) { *c = b; return 0; }
  if (b == LI) { *c = a; return 0; }
  if (a == b) { *c = LI; return 0; }
  /* the remaining letter */
  *c = 6 - a - b;
  /* cyclic X->Y->Z->X gives +i */
  if ((a == LX && b == LY) || (a == LY && b == LZ) || (a == LZ && b == LX)) return 1;
  return 3;
}

int ffo_pauli_mul(int n, uint64_t x1, uint64_t z1, uint64_t x2, uint64_t z2, uint64_t* x3,
                  uint64_t* z3) {
  int phase = 0;
  uint64_t xo = 0, zo = 0;
  for (int q = 0; q < n; ++q) {
    int c;
    phase += letter_mul(letter_of(x1, z1, q), letter_of(x2, z2, q), &c);
    if (c == LX || c == LY) xo |= 1ULL << q;
    if (c == LZ || c == LY) zo |= 1ULL << q;
  }
  *x3 = xo;
  *z3 = zo;
  return phase & 3;
}

typedef struct {
  uint64_t x, z;
  double cr, ci;
} term_t;

struct ffo_psum {
  int n;
  int size, cap;
  term_t* t;
};

ffo_psum* ffo_psum_new(int n_qubits) {
  ffo_psum* s = (ffo_psum*)calloc(1, sizeof(ffo_psum));
  s->n = n_qubits;
  return s;
}
void ffo_psum_free(ffo_psum* s) {
  if (!s) return;
  free(s->t);
  free(s);
}
int ffo_psum_size(const ffo_psum* s) { return s->size; }
int ffo_psum_nqubits(const ffo_psum* s) { return s->n; }
void ffo_psum_get(const ffo_psum* s, uint64_t* x, uint64_t* z, double* cr, double* ci) {
  for (int k = 0; k < s->size; ++k) {
    x[k] = s->t[k].x; z[k] = s->t[k].z; cr[k] = s->t[k].cr; ci[k] = s->t[k].ci;
  }
}

static void psum_push(ffo_psum* s, uint64_t x, uint64_t z, double cr, double ci) {
  if (s->size == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 64;
    s->t = (term_t*)realloc(s->t, (size_t)s->cap * sizeof(term_t));
  }
  term_t* t = &s->t[s->size++];
  t->x = x; t->z = z; t->cr = cr; t->ci = ci;
}

ffo_psum* ffo_psum_from_arrays(int n, int count, const uint64_t* x, const uint64_t* z,
                               const double* cr, const double* ci) {
  ffo_psum* s = ffo_psum_new(n);
  for (int k = 0; k < count; ++k) psum_push(s, x[k], z[k], cr[k], ci[k]);
  ffo_psum_simplify(s);
  return s;
}

/* canonical order: lexicographic on (x, z) as unsigned integers */
static int term_cmp(const void* a, const void* b) {
  const term_t* u = (const term_t*)a;
  const term_t* v = (const term_t*)b;
  if (u->x != v->x) return u->x < v->x ? -1 : 1;
  if (u->z != v->z) return u->z < v->z ? -1 : 1;
  return 0;
}

/* merge equal strings; drop |c| <= 1e-14 (pinned simplify threshold) */
void ffo_psum_simplify(ffo_psum* s) {
  if (s->size == 0) return;
  qsort(s->t, (size_t)s->size, sizeof(term_t), term_cmp);
  int out = 0;
  for (int k = 0; k < s->size;) {
    term_t acc = s->t[k];
    int j = k + 1;
    while (j < s->size && s->t[j].x == acc.x && s->t[j].z == acc.z) {
      acc.cr += s->t[j].cr;
      acc.ci += s->t[j].ci;
      ++j;
    }
    if (hypot(acc.cr, acc.ci) > 1e-14) s->t[out++] = acc;
    k = j;
  }
  s->size = out;
}

/* JW: a^dag_p = 1/2 (X_p - i Y_p) Z_{p-1}..Z_0,
 *                       a_p     = 1/2 (X_p + i Y_p) Z_{p-1}..Z_0.
 * The product of n_ops ladder operators expands to 2^n_ops Pauli products. */
void ffo_jw_add_product(ffo_psum* s, int n_ops, const int* idx, const int* dag, double cr,
                        double ci) {
  const int n = s->n;
  const int combos = 1 << n_ops;
  for (int c = 0; c < combos; ++c) {
    uint64_t x = 0, z = 0;
    double pr = cr, pi = ci;
    for (int k = 0; k < n_ops; ++k) {
      const int p = idx[k];
      /* choose X (bit 0) or Y (bit 1) part of operator k */
      const int useY = (c >> k) & 1;
      uint64_t ox = 1ULL << p;
      uint64_t oz = (p > 0 ? ((1ULL << p) - 1ULL) : 0ULL) | (useY ? (1ULL << p) : 0ULL);
      /* this operator's factor: 1/2 for X; -i/2 (dag) or +i/2 for Y */
      double fr, fi;
      if (!useY) { fr = 0.5; fi = 0.0; }
      else { fr = 0.0; fi = dag[k] ? -0.5 : 0.5; }
      /* string letters: X_p or Y_p times Z below. As a phase-free string the
       * letters are exactly (ox, oz) because they sit on distinct qubits. */
      uint64_t nx, nz;
      int ph = ffo_pauli_mul(n, x, z, ox, oz, &nx, &nz);
      x = nx; z = nz;
      double tr = pr * fr - pi * fi, ti = pr * fi + pi * fr;
      /* multiply by i^ph */
      for (int r = 0; r < ph; ++r) { double u = tr; tr = -ti; ti = u; }
      pr = tr; pi = ti;
    }
    psum_push(s, x, z, pr, pi);
  }
}

/* SPEC.md:266-297 spin-orbital Hamiltonian, interleaved ordering
 * (spin orbital 2P = alpha of spatial P, 2P+1 = beta):
 *   H = sum_pq h_pq a+_p a_q + 1/2 sum_pqrs g_pqrs a+_p a+_q a_s a_r + E_const,
 *   g_pqrs (physicists') = (PR|QS) delta(sp,sr) delta(sq,ss). */
ffo_psum* ffo_hamiltonian_jw(int m, const double* h, const double* g, double e_const) {
  const int n = 2 * m;
  ffo_psum* s = ffo_psum_new(n);
  if (e_const != 0.0) psum_push(s, 0, 0, e_const, 0.0);
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) {
      if ((p & 1) != (q & 1)) continue;
      double v = h[(p >> 1) * m + (q >> 1)];
      if (v == 0.0) continue;
      int idx[2] = {p, q}, dg[2] = {1, 0};
      ffo_jw_add_product(s, 2, idx, dg, v, 0.0);
    }
  for (int p = 0; p < n; ++p)
    for (int q = 0; q < n; ++q) {
      if (p == q) continue;
      for (int r = 0; r < n; ++r) {
        if ((p & 1) != (r & 1)) continue;
        for (int t = 0; t < n; ++t) {
          if (r == t) continue;
          if ((q & 1) != (t & 1)) continue;
          const int P = p >> 1, Q = q >> 1, R = r >> 1, T = t >> 1;
          double v = g[(((size_t)P * m + R) * m + Q) * m + T];
          if (v == 0.0) continue;
          /* 1/2 g a+_p a+_q a_t a_r  (s of the formula is t here) */
          int idx[4] = {p, q, t, r}, dg[4] = {1, 1, 0, 0};
          ffo_jw_add_product(s, 4, idx, dg, 0.5 * v, 0.0);
        }
      }
    }
  ffo_psum_simplify(s);
  return s;
}

/* ======================================================================== */
/* Generators and magnitude ordering.   */
/* Canonical id order: all singles (i asc, a asc), then doubles by          */
/* (i, j, a, b) lexicographic with i<j occupied, a<b virtual. Spin of       */
/* spin-orbital p is p & 1. tau_single = a+_a a_i,                          */
/* tau_double = a+_a a+_b a_j a_i.                                          */
/* ======================================================================== */
int ffo_build_generators(int n_so, int n_e, int* kind, int* idx) {
  int cnt = 0;
  for (int i = 0; i < n_e; ++i)
    for (int a = n_e; a < n_so; ++a) {
      if ((i & 1) != (a & 1)) continue;
      if (kind) { kind[cnt] = 1; idx[4 * cnt] = i; idx[4 * cnt + 1] = -1; idx[4 * cnt + 2] = a; idx[4 * cnt + 3] = -1; }
      ++cnt;
    }
  for (int i = 0; i < n_e; ++i)
    for (int j = i + 1; j < n_e; ++j)
      for (int a = n_e; a < n_so; ++a)
        for (int b = a + 1; b < n_so; ++b) {
          if ((i & 1) + (j & 1) != (a & 1) + (b & 1)) continue;
          if (kind) { kind[cnt] = 2; idx[4 * cnt] = i; idx[4 * cnt + 1] = j; idx[4 * cnt + 2] = a; idx[4 * cnt + 3] = b; }
          ++cnt;
        }
  return cnt;
}

/* JW image of (tau - tau^dag) with unit amplitude */
ffo_psum* ffo_generator_image(int n_so, int kind, const int* id4) {
  ffo_psum* s = ffo_psum_new(n_so);
  if (kind == 1) {
    int i = id4[0], a = id4[2];
    int idx[2] = {a, i}, dg[2] = {1, 0};
    ffo_jw_add_product(s, 2, idx, dg, 1.0, 0.0);
    int idx2[2] = {i, a}, dg2[2] = {1, 0}; /* tau^dag = a+_i a_a */
    ffo_jw_add_product(s, 2, idx2, dg2, -1.0, 0.0);
  } else {
    int i = id4[0], j = id4[1], a = id4[2], b = id4[3];
    int idx[4] = {a, b, j, i}, dg[4] = {1, 1, 0, 0};
    ffo_jw_add_product(s, 4, idx, dg, 1.0, 0.0);
    /* tau^dag = a+_i a+_j a_b a_a */
    int idx2[4] = {i, j, b, a}, dg2[4] = {1, 1, 0, 0};
    ffo_jw_add_product(s, 4, idx2, dg2, -1.0, 0.0);
  }
  ffo_psum_simplify(s);
  return s;
}

static const double* g_sort_amps;
static int order_cmp(const void* a, const void* b) {
  int u = *(const int*)a, v = *(const int*)b;
  double fu = fabs(g_sort_amps[u]), fv = fabs(g_sort_amps[v]);
  if (fu != fv) return fu > fv ? -1 : 1; /* descending |t| */
  return u < v ? -1 : (u > v ? 1 : 0);   /* ties: canonical id */
}

void ffo_magnitude_order(int n_gen, const double* amps, int* order) {
  for (int k = 0; k < n_gen; ++k) order[k] = k;
  g_sort_amps = amps;
  qsort(order, (size_t)n_gen, sizeof(int), order_cmp);
}

/* ======================================================================== */
/* Simulator. Natural binary order, qubit 0 = LSB.        */
/* ======================================================================== */
static int g_threads = 0;
void ffo_set_threads(int n) {
  g_threads = n;
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#endif
}
int ffo_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ffo_hf_state(int n, uint64_t occ_bits, double* psi) {
  const int64_t dim = (int64_t)1 << n;
  memset(psi, 0, (size_t)dim * 2 * sizeof(double));
  psi[2 * occ_bits] = 1.0;
}

static int parity_of(uint64_t v) { return __builtin_popcountll(v) & 1; }

/* (P psi)[k] = i^{#Y} (-1)^{popc((k^x)&z)} psi[k^x];
 * e^{i theta P} psi = cos(theta) psi + i sin(theta) P psi */
void ffo_apply_pauli_rotation(int n, double* psi, uint64_t x, uint64_t z, double theta) {
  const int64_t dim = (int64_t)1 << n;
  const double c = cos(theta), sn = sin(theta);
  const int ny = __builtin_popcountll(x & z) & 3;
  /* i * i^{ny} as a unit complex (wr, wi) */
  double wr = 0.0, wi = 1.0;
  for (int r = 0; r < ny; ++r) { double u = wr; wr = -wi; wi = u; }
  if (x == 0) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < dim; ++k) {
      double sg = parity_of((uint64_t)k & z) ? -1.0 : 1.0;
      double fr = c + sn * sg * wr, fi = sn * sg * wi;
      double ar = psi[2 * k], ai = psi[2 * k + 1];
      psi[2 * k] = fr * ar - fi * ai;
      psi[2 * k + 1] = fr * ai + fi * ar;
    }
    return;
  }
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < dim; ++k) {
    const uint64_t kp = (uint64_t)k ^ x;
    if (kp < (uint64_t)k) continue;
    double ar = psi[2 * k], ai = psi[2 * k + 1];
    double br = psi[2 * kp], bi = psi[2 * kp + 1];
    /* new[k]  = c a + i s i^ny (-1)^{popc(kp & z)} b */
    double s1 = parity_of(kp & z) ? -sn : sn;
    double s2 = parity_of((uint64_t)k & z) ? -sn : sn;
    double nar = c * ar + s1 * (wr * br - wi * bi);
    double nai = c * ai + s1 * (wr * bi + wi * br);
    double nbr = c * br + s2 * (wr * ar - wi * ai);
    double nbi = c * bi + s2 * (wr * ai + wi * ar);
    psi[2 * k] = nar; psi[2 * k + 1] = nai;
    psi[2 * kp] = nbr; psi[2 * kp + 1] = nbi;
  }
}

/* pairwise summation of an array */
static void pairwise_sum(const double* re, const double* im, int64_t n, double* sr, double* si) {
  if (n <= 8) {
    double a = 0, b = 0;
    for (int64_t k = 0; k < n; ++k) { a += re[k]; b += im[k]; }
    *sr = a; *si = b;
    return;
  }
  int64_t h = n / 2;
  double a1, b1, a2, b2;
  pairwise_sum(re, im, h, &a1, &b1);
  pairwise_sum(re + h, im + h, n - h, &a2, &b2);
  *sr = a1 + a2; *si = b1 + b2;
}

/* <psi|P|psi> with fixed 1024-amplitude blocks summed pairwise */
static void pauli_expect(int n, const double* psi, uint64_t x, uint64_t z, double* er,
                         double* ei, double* blk_re, double* blk_im) {
  const int64_t dim = (int64_t)1 << n;
  const int64_t B = dim < 1024 ? dim : 1024;
  const int64_t nb = dim / B;
  const int ny = __builtin_popcountll(x & z) & 3;
  double wr = 1.0, wi = 0.0;
  for (int r = 0; r < ny; ++r) { double u = wr; wr = -wi; wi = u; }
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    double sr = 0, si = 0;
    for (int64_t k = b * B; k < (b + 1) * B; ++k) {
      uint64_t kp = (uint64_t)k ^ x;
      double sg = parity_of(kp & z) ? -1.0 : 1.0;
      /* conj(psi_k) * i^ny * sg * psi_kp */
      double pr = psi[2 * kp] * wr - psi[2 * kp + 1] * wi;
      double pi = psi[2 * kp] * wi + psi[2 * kp + 1] * wr;
      double ar = psi[2 * k], ai = -psi[2 * k + 1];
      sr += sg * (ar * pr - ai * pi);
      si += sg * (ar * pi + ai * pr);
    }
    blk_re[b] = sr; blk_im[b] = si;
  }
  pairwise_sum(blk_re, blk_im, nb, er, ei);
}

void ffo_expectation(int n, const double* psi, const ffo_psum* H, double* re, double* im) {
  const int64_t dim = (int64_t)1 << n;
  const int64_t nb = dim < 1024 ? 1 : dim / 1024;
  double* br = (double*)malloc((size_t)nb * sizeof(double));
  double* bi = (double*)malloc((size_t)nb * sizeof(double));
  double* tr = (double*)malloc((size_t)(H->size + 1) * sizeof(double));
  double* ti = (double*)malloc((size_t)(H->size + 1) * sizeof(double));
  for (int t = 0; t < H->size; ++t) {
    double er, ei;
    pauli_expect(n, psi, H->t[t].x, H->t[t].z, &er, &ei, br, bi);
    /* c_t * <P_t> */
    tr[t] = H->t[t].cr * er - H->t[t].ci * ei;
    ti[t] = H->t[t].cr * ei + H->t[t].ci * er;
  }
  pairwise_sum(tr, ti, H->size, re, im);
  free(br); free(bi); free(tr); free(ti);
}

/* generators in plan order; each generator's Pauli terms in
 * canonical order; the image of (tau - tau^dag) has coefficients i*c_j, so
 * exp(t (tau - tau^dag)) = prod_j e^{i (t c_j) P_j}. */
double ffo_energy_trotter(int n_so, int n_e, int n_gen, const int* kind, const int* idx,
                          const int* plan, const double* amps, const ffo_psum* H,
                          double* psi_out, double* im_out) {
  const int64_t dim = (int64_t)1 << n_so;
  double* psi = psi_out ? psi_out : (double*)malloc((size_t)dim * 2 * sizeof(double));
  uint64_t occ = (n_e >= 64) ? ~0ULL : ((1ULL << n_e) - 1ULL);
  ffo_hf_state(n_so, occ, psi);
  for (int s = 0; s < n_gen; ++s) {
    const int gid = plan[s];
    const double t = amps[gid];
    ffo_psum* img = ffo_generator_image(n_so, kind[gid], idx + 4 * gid);
    for (int k = 0; k < img->size; ++k) {
      /* coefficient is purely imaginary: i * c */
      ffo_apply_pauli_rotation(n_so, psi, img->t[k].x, img->t[k].z, t * img->t[k].ci);
    }
    ffo_psum_free(img);
  }
  double re, im;
  ffo_expectation(n_so, psi, H, &re, &im);
  if (im_out) *im_out = im;
  if (!psi_out) free(psi);
  return re;
}

/* ---- JW-free fermionic cross-check -------------------------------------- */
/* a_p |k>: returns 0 if annihilated, else sign and new determinant */
static int ann(uint64_t* k, int p) {
  if (!((*k >> p) & 1ULL)) return 0;
  int sg = parity_of(*k & ((1ULL << p) - 1ULL)) ? -1 : 1;
  *k ^= 1ULL << p;
  return sg;
}
static int cre(uint64_t* k, int p) {
  if ((*k >> p) & 1ULL) return 0;
  int sg = parity_of(*k & ((1ULL << p) - 1ULL)) ? -1 : 1;
  *k ^= 1ULL << p;
  return sg;
}

double ffo_energy_fermionic(int m, int n_e, const double* h, const double* g, double e_const,
                            int n_gen, const int* kind, const int* idx, const int* plan,
                            const double* amps, double* psi_out) {
  const int n = 2 * m;
  const int64_t dim = (int64_t)1 << n;
  double* psi = (double*)calloc((size_t)dim, sizeof(double)); /* real arithmetic */
  uint64_t hf = (1ULL << n_e) - 1ULL;
  psi[hf] = 1.0;
  for (int s = 0; s < n_gen; ++s) {
    const int gid = plan[s];
    const double t = amps[gid], c = cos(t), sn = sin(t);
    const int* id = idx + 4 * gid;
    for (int64_t kk = 0; kk < dim; ++kk) {
      uint64_t k = (uint64_t)kk;
      int sg;
      if (kind[gid] == 1) {
        sg = ann(&k, id[0]);
        if (sg) sg *= cre(&k, id[2]);
      } else {
        sg = ann(&k, id[0]);
        if (sg) sg *= ann(&k, id[1]);
        if (sg) sg *= cre(&k, id[3]);
        if (sg) sg *= cre(&k, id[2]);
      }
      if (!sg) continue;
      /* pair (kk -> k) with tau|kk> = sg |k> */
      double a = psi[kk], b = psi[k];
      psi[kk] = c * a - sg * sn * b;
      psi[k] = sg * sn * a + c * b;
    }
  }
  double e = e_const;
  for (int64_t kk = 0; kk < dim; ++kk) {
    double a = psi[kk];
    if (a == 0.0) continue;
    double acc = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        if ((p & 1) != (q & 1)) continue;
        uint64_t k = (uint64_t)kk;
        int sg = ann(&k, q);
        if (sg) sg *= cre(&k, p);
        if (sg) acc += h[(p >> 1) * m + (q >> 1)] * sg * psi[k];
      }
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        if (p == q) continue;
        for (int r = 0; r < n; ++r) {
          if ((p & 1) != (r & 1)) continue;
          for (int t = 0; t < n; ++t) {
            if (r == t || (q & 1) != (t & 1)) continue;
            uint64_t k = (uint64_t)kk;
            int sg = ann(&k, r);
            if (sg) sg *= ann(&k, t);
            if (sg) sg *= cre(&k, q);
            if (sg) sg *= cre(&k, p);
            if (!sg) continue;
            double v = g[((((size_t)(p >> 1)) * m + (r >> 1)) * m + (q >> 1)) * m + (t >> 1)];
            /* op|kk> = sg|k>: contributes 1/2 v sg psi[k] psi[kk] (real) */
            acc += 0.5 * v * sg * psi[k];
          }
        }
      }
    e += a * acc;
  }
  if (psi_out)
    for (int64_t k = 0; k < dim; ++k) { psi_out[2 * k] = psi[k]; psi_out[2 * k + 1] = 0.0; }
  free(psi);
  return e;
}

double ffo_fmo_assemble(int n_fragments, int n_mono, const double* mono, int n_dim,
                        const double* dim) {
  if (n_mono != n_fragments || n_dim != n_fragments * (n_fragments - 1) / 2) return NAN;
  double e = 0.0, em = 0.0;
  for (int k = 0; k < n_dim; ++k) e += dim[k];
  for (int k = 0; k < n_mono; ++k) em += mono[k];
  return e - (n_fragments - 2) * em;
}
