// ffq_compile.hpp -- host-side compilation of Pauli data into the device
// tables the kernels stream over. Pure C++ (no CUDA), unit-testable on CPU.
//
// Two objects are compiled:
//  * a Trotter plan: each generator A_g (the JW
//    image of tau - tau^dag, anti-Hermitian) becomes either ONE fused pass
//    (all strings share flip mask X, commute, and have a single "outside" Z
//    class -- true for every UCCSD generator) or a run of single-string
//    rotations e^{i phi P} in canonical term order (the general fallback).
//  * a qubit Hamiltonian: terms grouped by flip mask X; in
//    each group, terms are split into classes by their Z part outside X and
//    tabulated over the 2^|X| bit patterns of the amplitude index on X, so
//    the kernel evaluates one popcount per class per amplitude pair and only
//    visits patterns with a non-zero table entry.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <functional>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace ffq {

using cplx = std::complex<double>;
constexpr int kSectorHeadPad = 8;   // empty ops behind gen_head (>= the kernel's prefetch depth)
constexpr int kSectorHeadSmall = 128, kSectorHeadLarge = 1024;  // threads of the real one-CTA program
constexpr int kMaxTableBits = 6;  // |X| up to 6 -> pattern tables of <= 64 entries

struct BadInput : std::invalid_argument {
  int code;
  BadInput(const std::string& w, int c) : std::invalid_argument(w), code(c) {}
};

inline int popc64(uint64_t v) { return __builtin_popcountll(v); }

// i^k as a complex number
inline cplx ipow(int k) {
  switch (k & 3) {
    case 0: return {1, 0};
    case 1: return {0, 1};
    case 2: return {-1, 0};
    default: return {0, -1};
  }
}

// bits of pattern index pi (bit i of pi -> qubit q[i]) as an amplitude mask
inline uint64_t pattern_bits(uint32_t pi, const int* q, int w) {
  uint64_t b = 0;
  for (int i = 0; i < w; ++i)
    if ((pi >> i) & 1u) b |= 1ULL << q[i];
  return b;
}

// ---- plan ------------------------------------------------------------------
struct FusedDesc {  // POD, copied to the device
  uint64_t x, zout;
  int32_t w, npair, pair_off, whi;  // whi: flip bits at positions >= 5 (word-index bits)
  int32_t q[kMaxTableBits];
  uint64_t qpack;     // q[i] in bits [6i, 6i+6): register-friendly copy for kernels
  uint64_t qpack_hi;  // positions - 5 of the flip bits >= 5 (support-word insertion)
  double alpha;
};

// 32-amplitude support words: offsets o in a word whose bits on X & 31 equal
// those of pattern bits pb
inline uint32_t low_pattern_mask(uint64_t X, uint64_t pb) {
  const uint32_t L = (uint32_t)(X & 31u), P = (uint32_t)(pb & 31u) & L;
  uint32_t m = 0;
  for (uint32_t o = 0; o < 32; ++o)
    if ((o & L) == P) m |= 1u << o;
  return m;
}
inline void hi_positions(uint64_t X, int32_t& whi, uint64_t& qpack_hi) {
  whi = 0;
  qpack_hi = 0;
  for (int qb = 5; qb < 64; ++qb)
    if ((X >> qb) & 1ULL) qpack_hi |= (uint64_t)(qb - 5) << (6 * whi++);
}

inline uint64_t pack_q(const int32_t* q, int w) {
  uint64_t v = 0;
  for (int i = 0; i < w; ++i) v |= (uint64_t)q[i] << (6 * i);
  return v;
}

struct CompiledPlan {
  int n_qubits = 0, n_gen = 0;
  // op stream in execution order
  std::vector<int32_t> op_kind;  // 0 fused, 1 string
  std::vector<int32_t> op_gen;   // generator index (theta column)
  std::vector<int32_t> op_idx;   // index into fused[] or str_*[]
  std::vector<double> op_cfac;   // phi = theta * cfac
  std::vector<double> op_sscale; // s = sin(phi) * sscale
  std::vector<FusedDesc> fused;
  std::vector<uint64_t> pair_bits;  // pattern bits of the "low" member
  std::vector<uint32_t> pair_low;   // low_pattern_mask of each pair's low member
  std::vector<double> pair_f;       // [pair][4]: F[pi] re,im, F[~pi] re,im
  std::vector<uint64_t> str_x, str_z;
  std::vector<int32_t> str_ny;
  int n_fused() const { return (int)fused.size(); }
  int n_string_ops() const { return (int)str_x.size(); }
};

inline CompiledPlan compile_plan(int n, int n_gen, const int64_t* off, const uint64_t* x,
                                 const uint64_t* z, const double* cr, const double* ci) {
  if (n < 1 || n > 40) throw BadInput("plan: n_qubits out of range [1, 40]", -1);
  if (n_gen < 0) throw BadInput("plan: negative generator count", -1);
  const uint64_t full = (n == 64) ? ~0ULL : ((1ULL << n) - 1ULL);
  CompiledPlan P;
  P.n_qubits = n;
  P.n_gen = n_gen;
  for (int g = 0; g < n_gen; ++g) {
    const int64_t b = off[g], e = off[g + 1];
    if (e < b) throw BadInput("plan: term_off not monotone", -1);
    // merge duplicates, canonical order (x, z) ascending
    std::map<std::pair<uint64_t, uint64_t>, cplx> terms;
    double scale = 0.0;
    for (int64_t t = b; t < e; ++t) {
      if ((x[t] | z[t]) & ~full) throw BadInput("plan: Pauli string exceeds n_qubits", -1);
      terms[{x[t], z[t]}] += cplx(cr[t], ci[t]);
      scale = std::max(scale, std::abs(cplx(cr[t], ci[t])));
    }
    std::vector<std::pair<std::pair<uint64_t, uint64_t>, cplx>> tl;
    for (auto& kv : terms)
      if (std::abs(kv.second) > 1e-14 * std::max(1.0, scale)) tl.push_back(kv);
    for (auto& kv : tl)
      if (std::abs(kv.second.real()) > 1e-12)
        throw BadInput("plan: generator " + std::to_string(g) +
                           " is not anti-Hermitian (real coefficient)", -1);
    if (tl.empty()) continue;  // identity rotation
    // fused eligibility
    bool fuse = true;
    const uint64_t X = tl[0].first.first;
    const int w = popc64(X);
    if (X == 0 || w > kMaxTableBits) fuse = false;
    const uint64_t zout = tl[0].first.second & ~X;
    for (auto& kv : tl) {
      if (kv.first.first != X || (kv.first.second & ~X) != zout) { fuse = false; break; }
    }
    if (fuse) {
      for (size_t i = 0; i < tl.size() && fuse; ++i)
        for (size_t j = i + 1; j < tl.size(); ++j)
          if (popc64(X & (tl[i].first.second ^ tl[j].first.second)) & 1) { fuse = false; break; }
    }
    FusedDesc d{};
    std::vector<cplx> F;
    if (fuse) {
      d.x = X; d.zout = zout; d.w = w;
      int wi = 0;
      for (int qb = 0; qb < 64; ++qb)
        if ((X >> qb) & 1ULL) d.q[wi++] = qb;
      d.qpack = pack_q(d.q, w);
      hi_positions(X, d.whi, d.qpack_hi);
      const uint32_t np = 1u << w;
      F.assign(np, cplx(0, 0));
      // F[pi] = <k^X|A|k> / s_out(k) = sum_j (i c_j) i^{ny_j} (-1)^{popc(pibits & z_j)}
      for (uint32_t pi = 0; pi < np; ++pi) {
        const uint64_t pb = pattern_bits(pi, d.q, w);
        cplx acc(0, 0);
        for (auto& kv : tl) {
          const uint64_t zj = kv.first.second;
          const int ny = popc64(X & zj);
          const double sg = (popc64(pb & zj) & 1) ? -1.0 : 1.0;
          acc += kv.second * ipow(ny) * sg;
        }
        F[pi] = acc;
      }
      double amax = 0;
      for (auto& f : F) amax = std::max(amax, std::abs(f));
      const double tol = 1e-12 * std::max(amax, 1e-300);
      double alpha = 0;
      for (auto& f : F)
        if (std::abs(f) > tol) {
          if (alpha == 0) alpha = std::abs(f);
          else if (std::abs(std::abs(f) - alpha) > 1e-12 * alpha) { fuse = false; break; }
        }
      if (alpha == 0) continue;  // A == 0 on every pattern: identity
      d.alpha = alpha;
      if (fuse) {
        d.pair_off = (int32_t)P.pair_bits.size();
        for (uint32_t pi = 0; pi < np; ++pi) {
          const uint32_t pb = pi ^ (np - 1u);
          if (pi > pb) continue;
          if (std::abs(F[pi]) <= tol && std::abs(F[pb]) <= tol) continue;
          P.pair_bits.push_back(pattern_bits(pi, d.q, w));
          P.pair_low.push_back(low_pattern_mask(X, pattern_bits(pi, d.q, w)));
          P.pair_f.push_back(F[pi].real()); P.pair_f.push_back(F[pi].imag());
          P.pair_f.push_back(F[pb].real()); P.pair_f.push_back(F[pb].imag());
        }
        d.npair = (int32_t)P.pair_bits.size() - d.pair_off;
      }
    }
    if (fuse) {
      P.op_kind.push_back(0);
      P.op_gen.push_back(g);
      P.op_idx.push_back((int32_t)P.fused.size());
      P.op_cfac.push_back(d.alpha);
      P.op_sscale.push_back(1.0 / d.alpha);
      P.fused.push_back(d);
    } else {
      for (auto& kv : tl) {  // canonical order, e^{i theta c_j P_j}
        P.op_kind.push_back(1);
        P.op_gen.push_back(g);
        P.op_idx.push_back((int32_t)P.str_x.size());
        P.op_cfac.push_back(kv.second.imag());
        P.op_sscale.push_back(1.0);
        P.str_x.push_back(kv.first.first);
        P.str_z.push_back(kv.first.second);
        P.str_ny.push_back(popc64(kv.first.first & kv.first.second) & 3);
      }
    }
  }
  return P;
}

// ---- Hamiltonian -------------------------------------------------------------
struct GroupDesc {  // POD
  uint64_t x;
  int32_t w;        // inserted bits (0 in generic mode)
  int32_t nact;     // active patterns
  int32_t act_off;  // into act_bits
  int32_t cls_off;  // into cls_z
  int32_t ncls;
  int32_t val_off;  // into cls_f (complex), layout [cls][nact]
  int32_t q[kMaxTableBits];
  uint64_t qpack;
  uint64_t qpack_hi;  // flip-bit positions >= 5, minus 5 (support-word insertion)
  int32_t whi, pad;
};

struct CompiledHam {
  int n_qubits = 0;
  int64_t n_terms = 0;
  std::vector<GroupDesc> groups;
  std::vector<uint64_t> act_bits;
  std::vector<uint32_t> act_low;  // low_pattern_mask per active pattern
  std::vector<uint64_t> cls_z;
  std::vector<double> cls_f;  // interleaved complex
  // global-path work items (group, active pattern, first u); fixed decomposition
  int64_t item_chunk = 0;
  std::vector<int32_t> item_g, item_p;
  std::vector<int64_t> item_u0;
  bool has_generic = false;  // some group has |X| > kMaxTableBits (random Pauli strings)
  // support-tracked path: items (group, pattern, first support word)
  std::vector<int32_t> sitem_g, sitem_p;
  std::vector<int64_t> sitem_w0;
  int64_t sitem_words = 0;
  int64_t n_classes() const { return (int64_t)cls_z.size(); }
};

constexpr int64_t kItemChunk = 4096;
constexpr int64_t kSupportWordsPerItem = 2048;

inline CompiledHam compile_ham(int n, int64_t nt, const uint64_t* x, const uint64_t* z,
                               const double* cr, const double* ci) {
  if (n < 1 || n > 40) throw BadInput("hamiltonian: n_qubits out of range [1, 40]", -1);
  const uint64_t full = (1ULL << n) - 1ULL;
  std::map<uint64_t, std::map<uint64_t, double>> byx;  // x -> z -> real coefficient
  for (int64_t t = 0; t < nt; ++t) {
    if ((x[t] | z[t]) & ~full) throw BadInput("hamiltonian: Pauli string exceeds n_qubits", -1);
    if (std::abs(ci[t]) > 1e-12)
      throw BadInput("hamiltonian: non-Hermitian term (imaginary coefficient)", -2);
    byx[x[t]][z[t]] += cr[t];
  }
  // Each x-group G = sum_t c_t P_t (c_t real) is Hermitian, so with
  //   b(m) = sum_t c_t i^{ny_t} (-1)^{popc(m & z_t)},   b(m ^ X) = conj(b(m)),
  // <G> = sum_m conj(psi[m^X]) psi[m] b(m) visits every unordered pair
  // {m, m^X} once as 2 Re(conj(psi[m^X]) psi[m] b(m)) (X != 0) and the
  // diagonal group as |psi[m]|^2 b(m). m runs over the inserted bits Q:
  //   table mode (|X| <= 6): Q = X, b(m) = sum_o sgn(m & zout_o) F_o[pattern]
  //   generic mode:          Q = {highest bit of X}, one class per term (members and
  //                          partners then run over contiguous index ranges: whole
  //                          32-byte sectors for any X).
  CompiledHam H;
  H.n_qubits = n;
  H.n_terms = 0;
  for (auto& gx : byx) {
    const uint64_t X = gx.first;
    std::vector<std::pair<uint64_t, double>> terms;
    double sabs = 0;
    for (auto& kv : gx.second)
      if (kv.second != 0.0) { terms.push_back(kv); sabs += std::abs(kv.second); }
    if (terms.empty()) continue;
    H.n_terms += (int64_t)terms.size();
    GroupDesc d{};
    d.x = X;
    const int w = popc64(X);
    const double wgt = (X == 0) ? 1.0 : 2.0;
    d.cls_off = (int32_t)H.cls_z.size();
    d.val_off = (int32_t)(H.cls_f.size() / 2);
    d.act_off = (int32_t)H.act_bits.size();
    if (w <= kMaxTableBits) {
      d.w = w;
      int wi = 0;
      for (int qb = 0; qb < 64; ++qb)
        if ((X >> qb) & 1ULL) d.q[wi++] = qb;
      d.qpack = pack_q(d.q, w);
      const uint32_t np = 1u << w;
      std::map<uint64_t, std::vector<std::pair<uint64_t, double>>> cls;  // by z outside X
      for (auto& t : terms) cls[t.first & ~X].push_back(t);
      std::vector<std::vector<cplx>> tab;
      for (auto& c : cls) {
        std::vector<cplx> F(np, cplx(0, 0));
        for (uint32_t pi = 0; pi < np; ++pi) {
          const uint64_t pb = pattern_bits(pi, d.q, w);
          cplx acc(0, 0);
          for (auto& t : c.second) {
            const int ny = popc64(X & t.first);
            const double sg = (popc64(pb & t.first) & 1) ? -1.0 : 1.0;
            acc += t.second * sg * ipow(ny);
          }
          F[pi] = acc;
        }
        tab.push_back(F);
      }
      // rounding-level residues of exact cancellations are dropped
      const double tol = 64.0 * 2.220446049250313e-16 * sabs;
      std::vector<uint32_t> act;  // lower member of each active pattern pair
      for (uint32_t pi = 0; pi < np; ++pi) {
        const uint32_t pb = pi ^ (np - 1u);
        if (X != 0 && pi > pb) continue;
        bool any = false;
        for (auto& F : tab) any |= std::abs(F[pi]) > tol || std::abs(F[pb]) > tol;
        if (any) act.push_back(pi);
      }
      if (act.empty()) continue;
      d.nact = (int32_t)act.size();
      for (uint32_t pi : act) {
        H.act_bits.push_back(pattern_bits(pi, d.q, w));
        H.act_low.push_back(low_pattern_mask(X, pattern_bits(pi, d.q, w)));
      }
      int ci2 = 0;
      for (auto& c : cls) {
        bool used = false;
        for (uint32_t pi : act) used |= std::abs(tab[ci2][pi]) > tol;
        if (used) {
          H.cls_z.push_back(c.first);
          for (uint32_t pi : act) {
            const cplx f = std::abs(tab[ci2][pi]) > tol ? wgt * tab[ci2][pi] : cplx(0, 0);
            H.cls_f.push_back(f.real());
            H.cls_f.push_back(f.imag());
          }
        }
        ++ci2;
      }
    } else {
      H.has_generic = true;
      d.w = 1;
      d.q[0] = 63 - __builtin_clzll(X);
      d.qpack = pack_q(d.q, 1);
      d.nact = 1;
      H.act_bits.push_back(0);
      H.act_low.push_back(low_pattern_mask(X & (1ULL << d.q[0]), 0));
      const uint64_t keep = ~(1ULL << d.q[0]);
      for (auto& t : terms) {
        const cplx f = wgt * t.second * ipow(popc64(X & t.first));
        H.cls_z.push_back(t.first & keep);
        H.cls_f.push_back(f.real());
        H.cls_f.push_back(f.imag());
      }
    }
    d.ncls = (int32_t)H.cls_z.size() - d.cls_off;
    // support words: generic mode inserts only q[0], so only that bit is fixed
    hi_positions(d.w == popc64(X) ? X : (X & (1ULL << d.q[0])), d.whi, d.qpack_hi);
    H.groups.push_back(d);
  }
  // fixed work decomposition for the global (large-state) path: chunks of
  // 4096 pairs, at most 256 chunks per (group, pattern) for very large n
  H.item_chunk = std::max<int64_t>(kItemChunk, (1LL << (n - 1)) / 256);
  for (size_t g = 0; g < H.groups.size(); ++g) {
    const auto& d = H.groups[g];
    const int64_t U = 1LL << (n - d.w);
    for (int p = 0; p < d.nact; ++p)
      for (int64_t u0 = 0; u0 < U; u0 += H.item_chunk) {
        H.item_g.push_back((int32_t)g);
        H.item_p.push_back(p);
        H.item_u0.push_back(u0);
      }
  }
  // support-tracked decomposition: fixed word ranges per (group, pattern),
  // 2048 words per item, at most 256 items per (group, pattern) for large n
  if (n >= 6) {
    H.sitem_words = std::max<int64_t>(kSupportWordsPerItem, (1LL << (n - 5)) / 256);
    for (size_t g = 0; g < H.groups.size(); ++g) {
      const auto& d = H.groups[g];
      const int64_t W = 1LL << (n - 5 - d.whi);
      for (int p = 0; p < d.nact; ++p)
        for (int64_t w0 = 0; w0 < W; w0 += H.sitem_words) {
          H.sitem_g.push_back((int32_t)g);
          H.sitem_p.push_back(p);
          H.sitem_w0.push_back(w0);
        }
    }
  }
  return H;
}

}  // namespace ffq

namespace ffq {

// ---- sharded state: global-qubit swap schedule -----------------------------------
// The state of n qubits is split over R = 2^g ranks: physical index bits
// [0, l) are local (l = n - g), bits [l, n) are the rank. perm[q] = physical
// position of logical qubit q. An op whose flip mask touches a global
// position first swaps it with a free local position (pairwise half-shard
// exchange between ranks r and r ^ (1 << j)); the local position chosen is the
// one whose logical qubit is next used furthest in the future (Belady).
struct ShardStep {
  int kind;      // 0 = swap physical global position gpos (>= l) with local lpos; 1 = apply plan op
  int gpos, lpos, op;
};

struct ShardSchedule {
  int n = 0, g = 0;
  std::vector<int> init_perm, final_perm;
  std::vector<ShardStep> steps;
  int n_swaps() const {
    int s = 0;
    for (auto& st : steps) s += st.kind == 0;
    return s;
  }
};

inline uint64_t permute_mask(uint64_t m, const std::vector<int>& perm) {
  uint64_t r = 0;
  for (size_t q = 0; q < perm.size(); ++q)
    if ((m >> q) & 1ULL) r |= 1ULL << perm[q];
  return r;
}

// logical flip mask of plan op `op`
inline uint64_t op_flip_mask(const CompiledPlan& P, int op) {
  return P.op_kind[op] == 0 ? P.fused[P.op_idx[op]].x : P.str_x[P.op_idx[op]];
}

inline ShardSchedule schedule_shards(const CompiledPlan& P, int g) {
  const int n = P.n_qubits, l = n - g;
  if (g < 0 || l < 2) throw BadInput("shard: need 0 <= n_global <= n_qubits - 2", -1);
  ShardSchedule S;
  S.n = n;
  S.g = g;
  const int n_ops = (int)P.op_kind.size();
  // global = the g logical qubits least often flipped by the plan (ties: higher index)
  std::vector<int> uses(n, 0);
  for (int op = 0; op < n_ops; ++op)
    for (int q = 0; q < n; ++q) uses[q] += (op_flip_mask(P, op) >> q) & 1ULL;
  std::vector<int> order(n);
  for (int q = 0; q < n; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return uses[a] != uses[b] ? uses[a] < uses[b] : a > b;
  });
  // local positions by ascending use: the least-flipped local qubits take the
  // lowest positions, so a generator's flip mask sits high and its active
  // patterns are long contiguous runs (a flip mask holding positions 0 and 1
  // leaves one live amplitude per 64-byte DRAM atom: k_fused_gen at 26% of HBM
  // against 88%)
  std::vector<int> perm(n, -1);
  for (int i = 0; i < g; ++i) perm[order[i]] = l + i;
  for (int i = g; i < n; ++i) perm[order[i]] = i - g;
  S.init_perm = perm;
  std::vector<int> inv(n);
  for (int q = 0; q < n; ++q) inv[perm[q]] = q;
  auto next_use = [&](int logical, int from) {
    for (int op = from; op < n_ops; ++op)
      if ((op_flip_mask(P, op) >> logical) & 1ULL) return op;
    return n_ops + n;  // never again
  };
  for (int op = 0; op < n_ops; ++op) {
    const uint64_t X = op_flip_mask(P, op);
    uint64_t xphys = permute_mask(X, perm);
    for (int gpos = l; gpos < n; ++gpos) {
      if (!((xphys >> gpos) & 1ULL)) continue;
      int best = -1, best_d = -1;
      for (int lpos = 0; lpos < l; ++lpos) {
        if ((xphys >> lpos) & 1ULL) continue;
        const int d = next_use(inv[lpos], op + 1);
        if (d > best_d) { best_d = d; best = lpos; }
      }
      if (best < 0) throw BadInput("shard: flip mask wider than the local qubits", -1);
      S.steps.push_back({0, gpos, best, -1});
      const int qa = inv[gpos], qb = inv[best];
      std::swap(perm[qa], perm[qb]);
      inv[perm[qa]] = qa;
      inv[perm[qb]] = qb;
      xphys = permute_mask(X, perm);
    }
    S.steps.push_back({1, -1, -1, op});
  }
  S.final_perm = perm;
  return S;
}

// Plan op descriptors mapped to physical positions (pattern tables unchanged:
// they are attached to pattern pairs, whose bits are permuted with the masks).
inline FusedDesc physical_fused(const FusedDesc& d, const std::vector<int>& perm) {
  FusedDesc p = d;
  p.x = permute_mask(d.x, perm);
  p.zout = permute_mask(d.zout, perm);
  int wi = 0;
  for (int qb = 0; qb < 64; ++qb)
    if ((p.x >> qb) & 1ULL) p.q[wi++] = qb;
  p.qpack = pack_q(p.q, p.w);
  hi_positions(p.x, p.whi, p.qpack_hi);
  return p;
}

}  // namespace ffq

#include <unordered_map>

namespace ffq {

// ---- support-closure ("sector") program ------------------------------------------
// S = amplitudes reachable from |hf> through the plan's pair maps (k <-> k ^ X
// on the active patterns of each fused generator), computed once per
// (plan, Hamiltonian, hf). Every amplitude outside S is identically zero for
// ANY theta, so an evaluation only needs the |S| amplitudes of S:
//  * generator g updates its pairs (i, j) inside S (indices into S, ascending k),
//  * <H> = sum over pairs (m, m ^ X) with both members in S of
//    Re(conj(psi[m ^ X]) psi[m] f(m)),  f(m) = sum_o sgn(m & z_o) F_o[p]
//    precomputed per pair and deduplicated into a table.
constexpr size_t kSegChunk = 512;

// Shared-memory bank order for a list of pairs. A warp's loads of psi[i] (and
// of psi[j]) are served conflict-free when each group of G lanes served by one
// wavefront hits G distinct bank slots: G = 8 lanes x 16 B (complex amplitudes)
// or G = 16 lanes x 8 B (real amplitudes), slot = index mod G. ri[t], rj[t] are
// those residues for pair t; the returned order packs the list into groups of G
// whose ri and rj are both all-distinct wherever the residue histogram allows
// (rows with most pairs left first, each taking the largest free column); the
// rest fill in as they come.
inline std::vector<uint32_t> bank_order(const std::vector<uint8_t>& ri, const std::vector<uint8_t>& rj,
                                        int G = 8) {
  const size_t n = ri.size();
  std::vector<uint32_t> out;
  out.reserve(n);
  if (n <= 1) {
    for (size_t t = 0; t < n; ++t) out.push_back((uint32_t)t);
    return out;
  }
  // buckets (ri, rj) as one flat array, each taken front to back (ascending t)
  const int NB = G * G;
  std::vector<uint32_t> head((size_t)NB + 1, 0), items(n);
  for (size_t t = 0; t < n; ++t) ++head[(size_t)ri[t] * G + rj[t] + 1];
  for (int b = 0; b < NB; ++b) head[b + 1] += head[b];
  std::vector<uint32_t> tail(head.begin(), head.end() - 1);
  for (size_t t = 0; t < n; ++t) items[tail[(size_t)ri[t] * G + rj[t]]++] = (uint32_t)t;
  auto size_of = [&](int b) { return tail[b] - head[b]; };
  int64_t row_left[16] = {0};
  for (size_t t = 0; t < n; ++t) ++row_left[ri[t]];
  size_t left = n;
  auto take = [&](int b) {
    out.push_back(items[head[b]++]);
    --row_left[b / G];
    --left;
  };
  // per group: a maximum matching rows (ri) -> columns (rj) over non-empty
  // buckets: greedy (rows with most pairs left first, largest free bucket),
  // then Kuhn's augmenting paths for the rows left unmatched
  int match_col[16], match_row[16], rows[16], order[16][16], n_order[16];
  bool seen[16];
  struct Aug {
    int G;
    int (*order)[16];
    int* n_order;
    int* match_col;
    int* match_row;
    bool* seen;
    bool run(int r) {
      for (int k = 0; k < n_order[r]; ++k) {
        const int c = order[r][k];
        if (seen[c]) continue;
        seen[c] = true;
        if (match_col[c] < 0 || run(match_col[c])) {
          match_col[c] = r;
          match_row[r] = c;
          return true;
        }
      }
      return false;
    }
  } aug{G, order, n_order, match_col, match_row, seen};
  while (left > 0) {
    int nr = 0;
    for (int r = 0; r < G; ++r) {
      match_row[r] = -1;
      match_col[r] = -1;
      if (row_left[r] > 0) rows[nr++] = r;
    }
    std::sort(rows, rows + nr, [&](int x, int y) { return row_left[x] > row_left[y]; });
    for (int k = 0; k < nr; ++k) {  // columns of row r by bucket size, largest first
      const int r = rows[k];
      int m = 0;
      for (int c = 0; c < G; ++c)
        if (size_of(r * G + c)) order[r][m++] = c;
      std::sort(order[r], order[r] + m, [&](int x, int y) { return size_of(r * G + x) > size_of(r * G + y); });
      n_order[r] = m;
    }
    for (int k = 0; k < nr; ++k) {  // greedy pass
      const int r = rows[k];
      for (int q = 0; q < n_order[r]; ++q)
        if (match_col[order[r][q]] < 0) {
          match_col[order[r][q]] = r;
          match_row[r] = order[r][q];
          break;
        }
    }
    for (int k = 0; k < nr; ++k)
      if (match_row[rows[k]] < 0) {
        for (int c = 0; c < G; ++c) seen[c] = false;
        aug.run(rows[k]);
      }
    int taken = 0;
    for (int r = 0; r < G; ++r)
      if (match_row[r] >= 0) {
        take(r * G + match_row[r]);
        ++taken;
      }
    for (; taken < G && left > 0; ++taken) {  // no conflict-free member left: largest bucket
      int best = 0;
      for (int b2 = 1; b2 < NB; ++b2)
        if (size_of(b2) > size_of(best)) best = b2;
      take(best);
    }
  }
  return out;
}

struct SectorProgram {
  bool ok = false;
  std::string why;  // reason when !ok
  int n = 0;
  uint32_t size = 0, hf_idx = 0;
  // S is split over n_parts = 2^s CTAs by the parities of the s masks in
  // split_masks (see compile_sector); part r holds S[part_start[r],
  // part_start[r + 1]), ordered by (part, k). op_cross[op] = 1 when generator
  // op has pairs across CTAs (its step ends with a cluster barrier).
  int n_parts = 1;
  std::vector<uint64_t> split_masks;
  std::vector<uint8_t> op_cross;
  std::vector<uint32_t> part_start;  // [n_parts + 1]
  std::vector<uint32_t> basis;
  // Amplitudes are addressed by 15-bit slots r << slot_bits | (i - part_start[r])
  // (rank r of the owning CTA, offset in its part): the device turns a slot into
  // a shared::cluster address with a shift, a mask and a select.
  int slot_bits = 15;
  uint32_t hf_slot = 0;
  std::vector<int64_t> gen_off;     // [n_ops * n_parts + 1]: op g, owner rank r -> gen_off[g * n_parts + r]
  std::vector<uint32_t> gen_pairs;  // slot_i | slot_j << 15 | sgn(k & zout) < 0 << 30 (i: low-pattern member)
  std::vector<uint8_t> gen_flags;   // bit 0: sgn(k & zout) < 0; bits 1..5: pattern pair index
  // Real one-CTA program (elem_bytes 8, one part): a negative sign swaps the
  // pair's members instead (F_hi = -F_lo: the 2x2 block is a rotation, so the
  // swapped pair is the same arithmetic bit for bit) and a word is
  // slot_i | slot_j << 16 (one mask and one shift to decode; bits 15, 31 clear).
  // gen_head[(2 op + h) * head_threads + tid] is thread tid's h-th
  // pair word of op (0xFFFFFFFF: none), bit 15 of the second word set when the
  // thread has further words in gen_pairs (ops with more than 2 head_threads
  // pairs); kSectorHeadPad all-empty ops follow (prefetch never leaves the table).
  std::vector<uint32_t> gen_head;
  int head_threads = 0;
  // Expectation pairs, slot_i | slot_j << 15 | sign << 30 (i: enumerated m,
  // j: m ^ X), in rows of 32 (one per warp lane). A row holds pairs of one
  // (group, pattern) set owned by one CTA; sets are padded to whole rows with
  // pairs of the owner's zero slot (an amplitude that stays 0). Rows whose
  // pairs share |f| ("shared" rows, sign per pair) carry f once (row_fre/fim);
  // the rest ("per-pair" rows) carry f per pair in pf_re/pf_im.
  //
  // Each rank's rows come in sections: first the pairs with both members in
  // its own part, then, per chunk of a peer's part, the cross pairs whose peer
  // member lies in that chunk. Before a chunk section the CTA copies the chunk
  // (one coalesced DSMEM pass) into a buffer behind its own amplitudes (slots
  // buf_off .. buf_off + buf_len - 1, overlaying the generator tables, dead by
  // then) and the pairs address the copy, so cross pairs cost local smem reads.
  struct ExpSection {
    int32_t src_rank, src_off, len;  // chunk to copy (len 0: no copy)
    int32_t sh0, sh1, pp1;           // shared rows [sh0, sh1), per-pair rows [sh1, pp1)
    int32_t pf_base;                 // per-pair row ordinal of row sh1 (pf index (pf_base + row - sh1) * 32 + lane)
  };
  std::vector<ExpSection> sections;
  std::vector<int32_t> sec_off;              // [n_parts + 1]
  uint32_t hmax = 0, buf_off = 0, buf_len = 0;
  int64_t exp_pair_count = 0;                // expectation pairs without the row padding
  std::vector<uint32_t> row_pairs;           // [n_rows * 32]
  std::vector<double> row_fre, row_fim;      // [n_rows] (0 on per-pair rows; row_fim empty if all f real)
  std::vector<double> pf_re, pf_im;          // [per-pair rows * 32] (pf_im empty if all f real)
  std::vector<uint32_t> zero_slot;           // [n_parts]
  bool f_real = true;
  // Product layout (one-CTA real program, see compile_blocks): S is the set
  // product of its alpha strings (even qubits) and beta strings (odd qubits),
  // and amplitude k lives at slot idx_a(k) * stride_b + idx_b(k) (stride_b odd,
  // so consecutive alpha or beta strings hit distinct banks). n_slots counts
  // the padded slots; the zero slot is n_slots. Without it, n_slots = size.
  bool product = false;
  uint32_t n_slots = 0, stride_b = 0, n_alpha = 0, n_beta = 0;
  std::vector<uint32_t> slot_of;  // one-CTA programs: slot of basis[i]
  // Anchored string blocks: expectation pairs that share one member ("anchor")
  // per lane and one partner offset per row. A unit is one chunk of <= 32
  // lanes run by one warp: lane word = anchor slot | B slot << 15; row r's
  // partner of lane l is slot B_l + O_r. Shared rows (one |f| per row) carry a
  // word per lane, O_r | sign << 15 | ftab index << 16, with f in ftab (kernel
  // parameter space: read through the constant cache, not the LSU); per-lane
  // rows carry O_r and f per lane. Units are assigned to warps at compile time
  // (blk_warp_off), balanced with the generic rows.
  std::vector<int32_t> blk_warp_off;   // [n_warps + 1]
  std::vector<int32_t> blk_units;      // [units * 8]: lw_off, sh_off (rows), pl_off, pf_off, 1, nsh, npl, 0
  std::vector<uint32_t> blk_lanes;     // [units * 32]
  std::vector<uint32_t> blk_sh;        // [shared rows * 32] lane words
  std::vector<uint32_t> blk_plo;       // per-lane rows: O*8
  std::vector<double> blk_plf;         // per-lane rows: [row][32] f
  std::vector<double> ftab;            // distinct shared-row f values
  std::vector<double> blk_shf;         // [shared rows] f per row
  // Per-warp row streams (what the device runs): the units of warp w back to
  // back, rows [blk_warp[4w], blk_warp[4w+1]) of 32 lane words each, cut into
  // three segments at rows blk_warp[4w+2] <= blk_warp[4w+3] (unit boundaries;
  // every segment padded with zero rows to whole prefetch rounds):
  //   bit 30 clear: shared row  O | sign << 15 | ftab index << 16
  //   bit 30 set:   anchor row  anchor slot | B slot << 15 | 1 << 30 (closes the previous unit)
  std::vector<uint32_t> blk_stream;
  std::vector<double> blk_fs;
  std::vector<int32_t> blk_warp;
  int64_t blk_pairs = 0;               // expectation pairs held by the blocks
  // Alpha-beta cliques (compile_cliques): the expectation pairs whose flip
  // mask is one alpha and one beta single excitation, evaluated as
  // sum_k s_k u_k^T C v_k over beta cliques (see compile_cliques), in the
  // alpha-first sign gauge: before the clique phase the device negates the
  // slots set in eps_flip.
  std::vector<uint32_t> alpha_strings, beta_strings;  // product layout: string of each alpha / beta index
  std::vector<uint32_t> eps_flip;      // [n_slots / 32 + 1] bitset over slots
  std::vector<uint32_t> cq_rows;       // ia * stride | ia' * stride << 15 | neg << 31
  std::vector<int32_t> cq_desc;        // [warp tasks][32][4]: columns 0-3 (bytes), columns 4-5, row begin, row end
  std::vector<double> cq_coef;         // [warp tasks][15][32]: C_ij of the lane's clique, pairs (i < j) in order
  std::vector<int32_t> cq_warp;        // [warps][2]: warp-task range of each warp
  int64_t cq_pairs = 0;                // expectation pairs held by the cliques
  int64_t cq_conflicts = 0;            // extra shared wavefronts per row over all half-warp tasks (bank model)
};

constexpr int kBlockMaxNC = 1;        // lane chunks per unit (the device runs one)
constexpr int kFTabMax = 3968;        // shared-row f values (kernel parameter space, 31 KiB)
constexpr int kBlockMinLanes = 16;    // smaller chunks go to the generic rows
constexpr int kBlockRowQuantum = 1;   // shared rows per unit padded to a multiple of this
constexpr int kBlkTrips = 6;          // k_sector_eval_real: four-row trips of block words in flight per warp (4: 877k, 6: 869k, 8: 906k expectation cycles, config 3)
constexpr int kStreamQuantum = 4 * kBlkTrips;  // rows per warp stream segment padded to a multiple of this
constexpr int kBlkSegments = 3;       // segments of a warp's block stream (summed separately, added in order)

// Anchored string blocks for the expectation pairs of a product-layout sector
// (see SectorProgram). For pair (i, j = i ^ X) with X = Xa | Xb (alpha / beta
// parts of the flip mask):
//   Xb = 0 (alpha type, also the diagonal X = 0): anchor = member with the lower
//     alpha index, block = its alpha string, lane = beta index, row = partner
//     alpha string: B_l = anchor slot, O_r = (ja - ia) * stride_b;
//   Xa = 0 (beta type): the same with the roles of the strings swapped;
//   both (alpha-beta): anchor = member holding Xa's lowest qubit, block = (Xa,
//     anchor beta string), lane = anchor alpha index, row = partner beta string:
//     B_l = idx_a(partner) * stride_b, O_r = idx_b(partner).
// In every case the partner slot is B_l + O_r, so a row costs one uniform
// descriptor load and one shared load per lane chunk, and the anchor is read
// once per unit. Pairs of chunks with fewer than kBlockMinLanes lanes stay in
// the generic rows (in_block[t] = 0).
struct BlockPair { uint32_t key_hi, key_lo, lane, row, anchor, partner; int64_t t; };
inline void compile_blocks(SectorProgram& S, const std::vector<uint32_t>& list,
                           const std::vector<std::pair<uint32_t, uint32_t>>& ij,  // closure indices per pair
                           const std::vector<double>& f, const std::vector<uint32_t>& slot_of,
                           const std::vector<uint32_t>& ia_of, const std::vector<uint32_t>& ib_of,
                           uint64_t amask, std::vector<uint8_t>& in_block) {
  const uint32_t sb = S.stride_b;
  std::vector<BlockPair> bp;
  bp.reserve(ij.size());
  for (size_t t = 0; t < ij.size(); ++t) {
    uint32_t i = ij[t].first, j = ij[t].second;
    const uint64_t X = (uint64_t)(list[i] ^ list[j]);
    const uint64_t xa = X & amask, xb = X & ~amask;
    BlockPair p{};
    p.t = (int64_t)t;
    if (xb == 0) {
      if (ia_of[j] < ia_of[i]) std::swap(i, j);
      p.key_hi = 0; p.key_lo = ia_of[i]; p.lane = ib_of[i]; p.row = (ia_of[j] - ia_of[i]) * sb;
    } else if (xa == 0) {
      if (ib_of[j] < ib_of[i]) std::swap(i, j);
      p.key_hi = 1; p.key_lo = ib_of[i]; p.lane = ia_of[i]; p.row = ib_of[j] - ib_of[i];
    } else {
      // alpha-beta blocks are keyed by the alpha flip mask (n <= 26: <= 13 alpha qubits)
      // and the anchor's beta string; the anchor holds Xa's lowest qubit
      if (!(list[i] & (xa & (~xa + 1)))) std::swap(i, j);
      p.key_hi = 2u + (uint32_t)xa; p.key_lo = ib_of[i]; p.lane = ia_of[i]; p.row = ib_of[j];
    }
    p.anchor = i;
    p.partner = j;
    bp.push_back(p);
  }
  std::sort(bp.begin(), bp.end(), [](const BlockPair& a, const BlockPair& b) {
    if (a.key_hi != b.key_hi) return a.key_hi < b.key_hi;
    if (a.key_lo != b.key_lo) return a.key_lo < b.key_lo;
    if (a.lane != b.lane) return a.lane < b.lane;
    return a.row < b.row;
  });
  const uint32_t zero = S.n_slots;
  std::map<double, uint32_t> ftab_index{{0.0, 0u}};  // ftab[0] = 0: padding rows
  S.ftab.assign(1, 0.0);
  size_t b0 = 0;
  while (b0 < bp.size()) {
    size_t b1 = b0;
    while (b1 < bp.size() && bp[b1].key_hi == bp[b0].key_hi && bp[b1].key_lo == bp[b0].key_lo) ++b1;
    // lanes of the block in ascending order, chunked by 32
    std::vector<size_t> lane_start;  // first entry of each distinct lane
    for (size_t u = b0; u < b1; ++u)
      if (u == b0 || bp[u].lane != bp[u - 1].lane) lane_start.push_back(u);
    lane_start.push_back(b1);
    const size_t nl = lane_start.size() - 1;
    std::vector<std::vector<size_t>> chunks;  // lane positions of the good chunks
    if (bp[b0].key_hi >= 2 && nl > 32 && nl < 32 + (size_t)kBlockMinLanes) {
      // alpha-beta block a little over one warp: keep the 32 lanes whose
      // partner loads spread best over the 16 eight-byte bank pairs (partner
      // slot = idx_a(partner) * stride_b + O_r, stride_b odd), the rest stay generic
      std::vector<size_t> keep(nl);
      for (size_t l = 0; l < nl; ++l) keep[l] = l;
      auto color = [&](size_t l) { return (ia_of[bp[lane_start[l]].partner] * sb) & 15u; };
      while (keep.size() > 32) {
        int cnt[16] = {0};
        for (size_t l : keep) ++cnt[color(l)];
        const int cmax = (int)(std::max_element(cnt, cnt + 16) - cnt);
        for (size_t q = keep.size(); q-- > 0;)
          if ((int)color(keep[q]) == cmax) { keep.erase(keep.begin() + (long)q); break; }
      }
      // 8-byte loads are served per half warp: lanes 0-15 and 16-31 each want 16
      // distinct bank pairs, so the first member of every color goes to the first half
      std::stable_sort(keep.begin(), keep.end(), [&](size_t x, size_t y) { return color(x) < color(y); });
      std::vector<size_t> h0, h1;
      for (size_t q = 0; q < keep.size(); ++q)
        ((q == 0 || color(keep[q]) != color(keep[q - 1])) && h0.size() < 16 ? h0 : h1).push_back(keep[q]);
      while (h0.size() < 16 && !h1.empty()) { h0.push_back(h1.back()); h1.pop_back(); }
      h0.insert(h0.end(), h1.begin(), h1.end());
      chunks.push_back(h0);
    } else {
      for (size_t c0 = 0; c0 < nl; c0 += 32) {
        const size_t c1 = std::min(nl, c0 + 32);
        if (c1 - c0 < (size_t)kBlockMinLanes) continue;
        chunks.emplace_back();
        for (size_t l = c0; l < c1; ++l) chunks.back().push_back(l);
      }
    }
    for (size_t g0 = 0; g0 < chunks.size(); g0 += kBlockMaxNC) {
      const int nc = (int)std::min<size_t>(kBlockMaxNC, chunks.size() - g0);
      // rows of the unit: cell (chunk, lane in chunk, row) -> pair entry
      std::map<uint32_t, std::vector<int64_t>> rows;  // row -> [nc * 32] bp index or -1
      for (int c = 0; c < nc; ++c) {
        const auto& lanes = chunks[g0 + c];
        for (size_t q = 0; q < lanes.size(); ++q)
          for (size_t u = lane_start[lanes[q]]; u < lane_start[lanes[q] + 1]; ++u) {
            auto& v = rows[bp[u].row];
            if (v.empty()) v.assign((size_t)nc * 32, -1);
            v[(size_t)c * 32 + q] = (int64_t)u;
          }
      }
      int32_t hdr[8] = {0, 0, 0, 0, nc, 0, 0, 0};
      hdr[0] = (int32_t)(S.blk_lanes.size() / 32);
      for (int c = 0; c < nc; ++c) {
        const auto& lanes = chunks[g0 + c];
        for (size_t q = 0; q < 32; ++q) {
          uint32_t w = zero;  // idle lane: anchor = zero slot, B = 0
          if (q < lanes.size()) {
            const BlockPair& p = bp[lane_start[lanes[q]]];
            const uint32_t B = p.key_hi >= 2 ? ia_of[p.partner] * sb : slot_of[p.anchor];
            w = slot_of[p.anchor] | (B << 15);
          }
          S.blk_lanes.push_back(w);
        }
      }
      // shared rows: every active lane present with one |f|; the rest per lane
      std::vector<std::pair<uint32_t, const std::vector<int64_t>*>> sh, pl;
      for (const auto& [r, cells] : rows) {
        bool shared = true;
        double f0 = 0.0;
        bool have = false;
        for (int c = 0; c < nc && shared; ++c) {
          const size_t act = chunks[g0 + c].size();
          for (size_t l = 0; l < act; ++l) {
            const int64_t u = cells[(size_t)c * 32 + l];
            if (u < 0) { shared = false; break; }
            const double fv = f[bp[u].t];
            if (!have) { f0 = fv; have = true; }
            else if (!(fv == f0 || fv == -f0)) { shared = false; break; }
          }
        }
        (shared ? sh : pl).push_back({r, &cells});
      }
      // shared rows whose f fits the table; the rest go to the per-lane rows
      std::vector<std::pair<uint32_t, const std::vector<int64_t>*>> sh2;
      std::vector<uint32_t> fidx;
      for (const auto& e : sh) {
        double fv = 0.0;
        for (int l = 0; l < 32; ++l)
          if ((*e.second)[l] >= 0) { fv = f[bp[(*e.second)[l]].t]; break; }
        auto it = ftab_index.find(fv);
        if (it == ftab_index.end()) {
          if (S.ftab.size() >= (size_t)kFTabMax) { pl.push_back(e); continue; }
          it = ftab_index.emplace(fv, (uint32_t)S.ftab.size()).first;
          S.ftab.push_back(fv);
        }
        sh2.push_back(e);
        fidx.push_back(it->second);
      }
      hdr[1] = (int32_t)(S.blk_sh.size() / 32);
      hdr[5] = (int32_t)((sh2.size() + kBlockRowQuantum - 1) / kBlockRowQuantum * kBlockRowQuantum);
      for (size_t k = 0; k < (size_t)hdr[5]; ++k) {
        if (k >= sh2.size()) {  // padding row: O = 0, f = ftab[0] = 0
          S.blk_sh.insert(S.blk_sh.end(), 32, 0u);
          S.blk_shf.push_back(0.0);
          continue;
        }
        S.blk_shf.push_back(S.ftab[fidx[k]]);
        const auto& cells = *sh2[k].second;
        const double fv = S.ftab[fidx[k]];
        for (int l = 0; l < 32; ++l) {
          const int64_t u = cells[l];
          const uint32_t neg = (u >= 0 && f[bp[u].t] != fv) ? 1u : 0u;
          S.blk_sh.push_back(sh2[k].first | (neg << 15) | (fidx[k] << 16));
        }
      }
      // rows without one shared |f| (singles: f depends on the other
      // occupations) stay in the generic per-pair rows
      hdr[2] = (int32_t)S.blk_plo.size();
      hdr[3] = (int32_t)(S.blk_plf.size() / 32);
      hdr[6] = 0;
      for (const auto& e : sh2)
        for (int64_t u : *e.second)
          if (u >= 0) {
            in_block[bp[u].t] = 1;
            ++S.blk_pairs;
          }
      S.blk_units.insert(S.blk_units.end(), hdr, hdr + 8);
    }
    b0 = b1;
  }
}

// ---- alpha-beta cliques -------------------------------------------------------------
// A pair (m, m ^ X) whose flip mask is one alpha single excitation Xa and one
// beta single excitation Xb has weight f(m) = c(X) (-1)^popc(m & zout): one
// outside-Z class (two-body H). Reordered to the alpha-first gauge (amplitude
// psi'(k) = eps(k) psi(k), eps = sign of moving every alpha creator in front
// of the beta ones), the weight factorises as
//     f'(m) = eps(m) eps(m ^ X) f(m) = s_Xa(a) * C_Xa(b, b')
// (a, b: alpha / beta strings of the member m that holds Xa's lowest qubit;
// b' = b ^ Xb). This is checked pair by pair below, never assumed. Writing
// u_k = psi'[a_k][.], v_k = psi'[a_k ^ Xa][.] for the rows k of Xa,
//     E_ab = sum_Xa sum_k s_k sum_(b, b') C_Xa(b, b') u_k[b] v_k[b'].
// Every beta pair (b, b') lies in exactly one clique T = b | b' (the N_b + 1
// strings that are N_b-subsets of T, pairwise single excitations), so a lane
// owning (Xa, T) loads the 6 + 6 amplitudes of T in rows a_k and a_k ^ Xa and
// accumulates acc_ij += s_k (u_i v_j + u_j v_i) over the 15 member pairs (C is
// symmetric, checked), 30 FMAs per 12 shared loads; C_ij is applied once per
// task. The lanes of a half warp share Xa (so a row's base slot is uniform) and
// their member order is chosen so each of the 6 loads hits 16 distinct bank
// pairs where the columns allow.
constexpr int kCliqueMax = 6;
constexpr int kCliquePairs = kCliqueMax * (kCliqueMax - 1) / 2;

// parity of the reorder interleaved -> alpha-first for basis state k (alpha =
// even qubits): each occupied beta qubit passes the occupied alpha qubits above it
inline int alpha_first_parity(uint64_t k, int n) {
  uint64_t am = 0;
  for (int q = 0; q < n; q += 2) am |= 1ULL << q;
  int s = 0;
  for (int r = 1; r < n; r += 2)
    if ((k >> r) & 1ULL) s += popc64(k & am & ~((2ULL << r) - 1ULL));
  return s & 1;
}

// member order of each lane of a half warp (lanes: <= 16 column lists of
// kCliqueMax entries) so that load c of every lane hits distinct 8-byte bank
// pairs (column mod 16; equal columns broadcast). Returns the extra
// wavefronts per row over the 6 loads (0 = conflict-free).
inline int clique_color(std::vector<std::array<uint32_t, kCliqueMax>>& lanes) {
  const size_t L = lanes.size();
  auto cost_of = [&](int c) {
    int cnt[16] = {0};
    uint32_t seen[16][16];
    int ns[16] = {0};
    for (size_t l = 0; l < L; ++l) {
      const uint32_t col = lanes[l][c], r = col & 15u;
      bool dup = false;
      for (int q = 0; q < ns[r]; ++q) dup |= seen[r][q] == col;
      if (!dup) { seen[r][ns[r]++] = col; ++cnt[r]; }
    }
    return *std::max_element(cnt, cnt + 16) - 1;
  };
  // greedy: per load slot a maximum matching lanes -> residues (Kuhn)
  std::vector<std::array<uint32_t, kCliqueMax>> rem = lanes;
  std::vector<int> nrem(L, kCliqueMax);
  for (int c = 0; c < kCliqueMax; ++c) {
    int match_res[16], match_lane[16];
    for (int r = 0; r < 16; ++r) match_res[r] = -1;
    for (size_t l = 0; l < L; ++l) match_lane[l] = -1;
    std::function<bool(int, std::vector<bool>&)> aug = [&](int l, std::vector<bool>& vis) {
      for (int q = 0; q < nrem[l]; ++q) {
        const int r = (int)(rem[l][q] & 15u);
        if (vis[r]) continue;
        vis[r] = true;
        if (match_res[r] < 0 || aug(match_res[r], vis)) { match_res[r] = l; match_lane[l] = q; return true; }
      }
      return false;
    };
    // lanes with the fewest choices first
    std::vector<int> ord(L);
    for (size_t l = 0; l < L; ++l) ord[l] = (int)l;
    for (int l : ord) { std::vector<bool> vis(16, false); aug(l, vis); }
    for (int r = 0; r < 16; ++r)
      if (match_res[r] >= 0) {  // Kuhn may have re-pointed lanes: recover each lane's member by residue
        const int l = match_res[r];
        for (int q = 0; q < nrem[l]; ++q)
          if ((int)(rem[l][q] & 15u) == r) { match_lane[l] = q; break; }
      }
    for (size_t l = 0; l < L; ++l) {
      const int q = match_lane[l] >= 0 ? match_lane[l] : 0;
      lanes[l][c] = rem[l][q];
      rem[l][q] = rem[l][nrem[l] - 1];
      --nrem[l];
    }
  }
  int total = 0;
  for (int c = 0; c < kCliqueMax; ++c) total += cost_of(c);
  // local search: swap two load slots of one lane when the total does not grow
  uint64_t rng = 0x2545F4914F6CDD1Dull;
  for (int it = 0; it < 4000 && total > 0; ++it) {
    rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
    const size_t l = rng % L;
    const int c1 = (int)((rng >> 20) % kCliqueMax), c2 = (int)((rng >> 40) % kCliqueMax);
    if (c1 == c2) continue;
    const int before = cost_of(c1) + cost_of(c2);
    std::swap(lanes[l][c1], lanes[l][c2]);
    const int after = cost_of(c1) + cost_of(c2);
    if (after <= before) total += after - before;
    else std::swap(lanes[l][c1], lanes[l][c2]);
  }
  return total;
}

// f: pair weights already in the alpha-first gauge (compile_sector multiplies
// every expectation weight by eps(m) eps(m ^ X) when cliques are on)
inline void compile_cliques(SectorProgram& S, const std::vector<uint32_t>& list,
                            const std::vector<std::pair<uint32_t, uint32_t>>& ij, const std::vector<double>& f,
                            const std::vector<uint32_t>& slot_of, const std::vector<uint32_t>& ia_of,
                            const std::vector<uint32_t>& ib_of, uint64_t amask, std::vector<uint8_t>& in_clique) {
  const uint32_t NB = S.n_beta, stride = S.stride_b;
  if (NB >= 256) return;  // 8-bit columns
  const uint32_t zero_col = NB;  // slot a * stride + NB is padding (zero) in every row when stride > NB
  std::map<uint32_t, uint32_t> bpos;
  for (uint32_t q = 0; q < NB; ++q) bpos[S.beta_strings[q]] = q;
  struct Cand { uint32_t a, a2, b, b2; double w; size_t t; };
  std::map<uint64_t, std::vector<Cand>> by_xa;
  for (size_t t = 0; t < ij.size(); ++t) {
    uint32_t i = ij[t].first, j = ij[t].second;
    const uint64_t X = (uint64_t)(list[i] ^ list[j]), xa = X & amask, xb = X & ~amask;
    if (popc64(xa) != 2 || popc64(xb) != 2) continue;
    if (!(list[i] & (xa & (~xa + 1)))) std::swap(i, j);
    by_xa[xa].push_back({ia_of[i], ia_of[j], ib_of[i], ib_of[j], f[t], t});
  }
  struct Group { uint64_t xa; std::vector<uint32_t> rows; std::vector<int8_t> sgn; std::map<std::pair<uint32_t, uint32_t>, double> C; std::vector<uint64_t> cliques; };
  std::vector<Group> groups;
  for (auto& [xa, cs] : by_xa) {
    Group g;
    g.xa = xa;
    // dense index tables (alpha index -> row, (beta, beta') -> key): no maps on the 3 M pairs
    std::vector<int32_t> rix(S.n_alpha, -1), kix((size_t)NB * NB, -1);
    std::vector<std::pair<uint32_t, uint32_t>> keys;
    for (const Cand& c : cs) {
      if (rix[c.a] < 0) { rix[c.a] = (int32_t)g.rows.size(); g.rows.push_back(c.a); }
      int32_t& kk = kix[(size_t)c.b * NB + c.b2];
      if (kk < 0) { kk = (int32_t)keys.size(); keys.push_back({c.b, c.b2}); }
    }
    const size_t R = g.rows.size(), K = keys.size();
    if (R * K != cs.size()) continue;  // not every (row, key): some weights vanish
    std::vector<double> W(R * K, 0.0);
    std::vector<uint8_t> have(R * K, 0);
    for (const Cand& c : cs) {
      const size_t s = (size_t)rix[c.a] * K + (size_t)kix[(size_t)c.b * NB + c.b2];
      if (have[s]) goto reject;
      have[s] = 1;
      W[s] = c.w;
    }
    {
      // gauge: row 0 positive; C from row 0; every row's sign from key 0
      std::vector<double> C(W.begin(), W.begin() + (long)K);
      g.sgn.assign(R, 1);
      for (size_t r = 0; r < R; ++r) {
        g.sgn[r] = (W[r * K] > 0) == (C[0] > 0) ? 1 : -1;
        for (size_t k = 0; k < K; ++k) {
          const double want = g.sgn[r] * C[k];
          if (std::fabs(want - W[r * K + k]) > 1e-13 * std::fabs(W[r * K + k])) goto reject;
        }
      }
      for (size_t k = 0; k < K; ++k) {
        const int32_t kt = kix[(size_t)keys[k].second * NB + keys[k].first];
        if (kt < 0 || std::fabs(C[kt] - C[k]) > 1e-13 * std::fabs(C[k])) goto reject;
        g.C[keys[k]] = C[k];
      }
      std::set<uint64_t> ts;
      for (const auto& key : keys) ts.insert((uint64_t)S.beta_strings[key.first] | S.beta_strings[key.second]);
      for (uint64_t T : ts) {
        if (popc64(T) > kCliqueMax) goto reject;
        uint32_t nm = 0;
        for (int q = 0; q < S.n; ++q)
          if (((T >> q) & 1ULL) && bpos.count((uint32_t)(T ^ (1ULL << q)))) ++nm;
        if (nm < (uint32_t)kCliqueMax && stride <= NB) goto reject;  // no zero column to pad with
      }
      g.cliques.assign(ts.begin(), ts.end());
      for (const Cand& c : cs) in_clique[c.t] = 1;
      S.cq_pairs += (int64_t)cs.size();
      groups.push_back(std::move(g));
      continue;
    }
  reject:;
  }
  if (groups.empty()) return;
  // half-warp tasks: per group, its cliques in chunks of <= 16 lanes, member
  // orders colored per chunk (cached by clique list)
  struct Half { uint32_t row0, row1; std::vector<std::array<uint32_t, kCliqueMax>> cols; const Group* g; };
  std::vector<Half> halves;
  std::map<std::vector<uint64_t>, std::vector<std::vector<std::array<uint32_t, kCliqueMax>>>> cache;
  for (const Group& g : groups) {
    const uint32_t row0 = (uint32_t)S.cq_rows.size();
    for (size_t r = 0; r < g.rows.size(); ++r) {
      const uint32_t a = g.rows[r], a2 = (uint32_t)std::distance(
          S.alpha_strings.begin(), std::find(S.alpha_strings.begin(), S.alpha_strings.end(),
                                             S.alpha_strings[a] ^ (uint32_t)g.xa));
      S.cq_rows.push_back(a * stride | (a2 * stride) << 15 | (g.sgn[r] < 0 ? 1u << 31 : 0u));
    }
    auto it = cache.find(g.cliques);
    if (it == cache.end()) {
      const size_t nT = g.cliques.size(), nh = (nT + 15) / 16;
      std::vector<std::vector<std::array<uint32_t, kCliqueMax>>> hs(nh);
      for (size_t q = 0; q < nT; ++q) {
        const uint64_t T = g.cliques[q];
        std::array<uint32_t, kCliqueMax> m;
        m.fill(zero_col);
        int nm = 0;
        for (int b = 0; b < S.n; ++b)
          if ((T >> b) & 1ULL) {
            auto p = bpos.find((uint32_t)(T ^ (1ULL << b)));
            if (p != bpos.end()) m[nm++] = p->second;
          }
        hs[q * nh / nT].push_back(m);  // balanced chunks
      }
      for (auto& h : hs) S.cq_conflicts += clique_color(h);
      it = cache.emplace(g.cliques, std::move(hs)).first;
    }
    for (const auto& h : it->second) halves.push_back({row0, (uint32_t)S.cq_rows.size(), h, &g});
  }
  // warp tasks = two half-warp tasks; lanes beyond a half's cliques are idle
  const size_t nwt = (halves.size() + 1) / 2;
  S.cq_desc.assign(nwt * 32 * 4, 0);
  S.cq_coef.assign(nwt * kCliquePairs * 32, 0.0);
  for (size_t h = 0; h < halves.size(); ++h) {
    const Half& H = halves[h];
    const size_t wt = h / 2, l0 = (h % 2) * 16;
    for (size_t l = 0; l < H.cols.size(); ++l) {
      const auto& m = H.cols[l];
      int32_t* d = &S.cq_desc[(wt * 32 + l0 + l) * 4];
      d[0] = (int32_t)(m[0] | m[1] << 8 | m[2] << 16 | m[3] << 24);
      d[1] = (int32_t)(m[4] | m[5] << 8);
      d[2] = (int32_t)H.row0;
      d[3] = (int32_t)H.row1;
      int p = 0;
      for (int i = 0; i < kCliqueMax; ++i)
        for (int j = i + 1; j < kCliqueMax; ++j, ++p) {
          auto c = H.g->C.find({m[i], m[j]});
          S.cq_coef[(wt * kCliquePairs + p) * 32 + l0 + l] = c == H.g->C.end() ? 0.0 : c->second;
        }
    }
  }
}

// L1 wavefronts of a block unit (a lane word and a shared load per row;
// per-lane rows add a coalesced f load), used to balance warps
inline double block_unit_cost(const int32_t* hdr) {
  return 4.0 + hdr[5] * 3.2 + hdr[6] * 5.2;
}

// Order of the alpha strings for the product layout. An alpha-beta block with
// alpha flip mask Xa reads, per row, psi[idx_a(J) * stride + O] for the partner
// strings J of its lanes, so its shared-load wavefronts are the largest number
// of lanes on one 8-byte bank pair, color(J) = idx_a(J) * stride mod 16. The
// order is a local search over colors (capacities fixed by the string count)
// minimising the sum over masks of that maximum, after the block drops its
// lanes beyond 32 from the fullest colors (as compile_blocks does).
inline std::vector<uint32_t> alpha_order(const std::vector<uint32_t>& sa, const std::vector<uint64_t>& xas,
                                         uint32_t stride) {
  const size_t na = sa.size();
  if (na < 32 || xas.empty()) return sa;
  std::map<uint32_t, uint32_t> pos;
  for (uint32_t q = 0; q < (uint32_t)na; ++q) pos[sa[q]] = q;
  // partner sets (positions in sa) of each mask with 32 < size < 48
  std::vector<std::vector<uint32_t>> sets;
  for (uint64_t xa : xas) {
    const uint32_t low = (uint32_t)(xa & (~xa + 1));
    std::vector<uint32_t> P;
    for (uint32_t J : sa)
      if (!(J & low) && pos.count(J ^ (uint32_t)xa)) P.push_back(pos[J]);
    if (P.size() > 32 && P.size() < 48) sets.push_back(P);
    else if (P.size() >= 16 && P.size() <= 32) sets.push_back(P);
  }
  if (sets.empty()) return sa;
  const bool dbg = std::getenv("FFQ_DEBUG") != nullptr;
  std::vector<std::vector<uint32_t>> member(na);  // sets containing each string
  for (uint32_t k = 0; k < (uint32_t)sets.size(); ++k)
    for (uint32_t q : sets[k]) member[q].push_back(k);
  // initial colors: the natural order's (color of position q = q * stride mod 16)
  std::vector<uint8_t> col(na);
  for (size_t q = 0; q < na; ++q) col[q] = (uint8_t)((q * stride) & 15u);
  // cost: lanes beyond two per color after the block's drops (0 = every row's
  // partner loads conflict-free), squared per color so the search has a slope
  auto set_cost = [&](uint32_t k) {
    int cnt[16] = {0};
    for (uint32_t q : sets[k]) ++cnt[col[q]];
    for (size_t d = sets[k].size(); d > 32; --d) --*std::max_element(cnt, cnt + 16);
    int c2 = 0;
    for (int c = 0; c < 16; ++c)
      if (cnt[c] > 2) c2 += (cnt[c] - 2) * (cnt[c] - 2);
    return c2;
  };
  std::vector<int> cost(sets.size());
  long total = 0;
  for (uint32_t k = 0; k < (uint32_t)sets.size(); ++k) total += cost[k] = set_cost(k);
  uint64_t rng = 0x9E3779B97F4A7C15ull;
  auto next = [&]() {
    rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
    return rng;
  };
  if (dbg) std::fprintf(stderr, "[ffq] alpha_order: %zu sets, cost %ld before\n", sets.size(), total);
  for (int it = 0; it < 400000 && total > 0; ++it) {
    const size_t a = next() % na, b = next() % na;
    if (col[a] == col[b]) continue;
    std::swap(col[a], col[b]);
    std::vector<uint32_t> aff(member[a]);
    aff.insert(aff.end(), member[b].begin(), member[b].end());
    std::sort(aff.begin(), aff.end());
    aff.erase(std::unique(aff.begin(), aff.end()), aff.end());
    long delta = 0;
    std::vector<int> nc(aff.size());
    for (size_t t = 0; t < aff.size(); ++t) delta += (nc[t] = set_cost(aff[t])) - cost[aff[t]];
    if (delta <= 0) {
      for (size_t t = 0; t < aff.size(); ++t) cost[aff[t]] = nc[t];
      total += delta;
    } else {
      std::swap(col[a], col[b]);
    }
  }
  if (dbg) std::fprintf(stderr, "[ffq] alpha_order: cost %ld after (0 = conflict-free)\n", total);
  // positions with color c (q * stride mod 16 == c) take the strings of color c
  std::vector<std::vector<uint32_t>> by_col(16), slots(16);
  for (size_t q = 0; q < na; ++q) {
    by_col[col[q]].push_back(sa[q]);
    slots[(q * stride) & 15u].push_back((uint32_t)q);
  }
  std::vector<uint32_t> out(na);
  for (int c = 0; c < 16; ++c)
    for (size_t t = 0; t < by_col[c].size(); ++t) out[slots[c][t]] = by_col[c][t];
  return out;
}

// cap_amps: shared-memory capacity of a CTA in amplitudes (own part, zero
// slot and copy buffer); the buffer is used when at least kMinChunk fit.
constexpr uint32_t kMinChunk = 256;
inline SectorProgram compile_sector(const CompiledPlan& P, const CompiledHam& H, uint64_t hf,
                                    uint32_t max_size, uint32_t max_part = 0xFFFFFFFFu, int n_parts = 2,
                                    uint32_t cap_amps = 0xFFFFFFFFu, int row_quantum = 4,
                                    int elem_bytes = 16, int block_warps = 0, uint32_t block_min_size = 0,
                                    bool cliques = false) {
  // lanes per conflict-free shared-memory wavefront for this amplitude size
  const int bank_group = elem_bytes == 8 ? 16 : 8;
  const bool real_prog = elem_bytes == 8 && n_parts == 1;  // k_sector_eval_real's tables
  SectorProgram S;
  const int n = P.n_qubits;
  S.n = n;
  if (n > 26 || H.n_qubits != n) { S.why = "qubit count"; return S; }
  if (P.n_string_ops() > 0) { S.why = "plan has non-fused generators"; return S; }
  if (n_parts != 1 && n_parts != 2 && n_parts != 4 && n_parts != 8) { S.why = "parts must be 1, 2, 4 or 8"; return S; }
  const size_t dim = size_t(1) << n;
  const bool dbg_t = std::getenv("FFQ_DEBUG") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!dbg_t) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ffq] compile_sector %-22s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  std::vector<int32_t> idx(dim, -1);
  std::vector<uint32_t> list{(uint32_t)hf};
  idx[hf] = 0;
  // closure in plan order; record each generator's pairs in terms of k values
  const int n_ops = (int)P.op_kind.size();
  std::vector<std::vector<std::pair<uint32_t, uint8_t>>> gk(n_ops);
  // pos[k] = position of k in `list` (insertion order), -1 if absent; the
  // support before op g is list[0, cur)
  std::vector<int32_t> pos(dim, -1);
  pos[hf] = 0;
  for (int op = 0; op < n_ops; ++op) {
    const FusedDesc& d = P.fused[P.op_idx[op]];
    const size_t cur = list.size();
    for (size_t t = 0; t < cur; ++t) {
      const uint32_t k = list[t];
      const uint64_t pat = k & d.x;
      for (int p = 0; p < d.npair; ++p) {
        const uint64_t lo = P.pair_bits[d.pair_off + p], hi = lo ^ d.x;
        if (pat != lo && pat != hi) continue;
        const uint32_t kl = (pat == lo) ? k : (uint32_t)(k ^ d.x);  // low-pattern member
        const uint32_t kh = kl ^ (uint32_t)d.x;
        // record each pair once: from its low member when that was already supported
        if (pat == hi && pos[kl] >= 0 && (size_t)pos[kl] < cur) continue;
        const uint8_t flag = (uint8_t)(((__builtin_popcountll(kl & d.zout) & 1) ? 1 : 0) | (p << 1));
        gk[op].push_back({kl, flag});
        if (pos[kh] < 0) { pos[kh] = (int32_t)list.size(); list.push_back(kh); }
        if (pos[kl] < 0) { pos[kl] = (int32_t)list.size(); list.push_back(kl); }
      }
      if (list.size() > max_size) { S.why = "support closure too large"; return S; }
    }
  }
  stage("closure");
  // expectation pairs in k space with their class sums f(m)
  struct EP { uint32_t m; int g, p; double fr, fi; };
  std::vector<EP> ek;
  {
    // groups in contiguous chunks over host threads, concatenated in group order
    const size_t ng = H.groups.size();
    const int nth = (int)std::max<size_t>(1, std::min<size_t>({(size_t)std::thread::hardware_concurrency(), 16,
                                                               (ng + 63) / 64}));
    std::vector<std::vector<EP>> part((size_t)nth);
    auto work = [&](int t) {
      for (size_t gi = ng * t / nth; gi < ng * (t + 1) / nth; ++gi) {
        const auto& d = H.groups[gi];
        uint64_t Q = 0;
        for (int i = 0; i < d.w; ++i) Q |= 1ULL << d.q[i];
        for (int p = 0; p < d.nact; ++p) {
          const uint64_t pb = H.act_bits[d.act_off + p];
          for (uint32_t m : list) {
            if ((m & Q) != pb) continue;
            if (pos[m ^ (uint32_t)d.x] < 0) continue;
            double fr = 0.0, fi = 0.0;
            for (int o = 0; o < d.ncls; ++o) {
              const double sg = (__builtin_popcountll(m & H.cls_z[d.cls_off + o]) & 1) ? -1.0 : 1.0;
              fr += sg * H.cls_f[2 * (d.val_off + o * d.nact + p)];
              fi += sg * H.cls_f[2 * (d.val_off + o * d.nact + p) + 1];
            }
            if (fr == 0.0 && fi == 0.0) continue;
            part[t].push_back({m, (int)gi, p, fr, fi});
          }
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    size_t tot = 0;
    for (auto& v : part) tot += v.size();
    ek.reserve(tot);
    for (auto& v : part) ek.insert(ek.end(), v.begin(), v.end());
  }
  stage("expectation pairs");
  S.size = (uint32_t)list.size();
  if (S.size > 32767) { S.why = "support closure exceeds 15-bit indices"; return S; }
  // split S over 2^s CTAs by the parities of s qubit masks M_1..M_s (part bit
  // b = parity(k & M_b)); a pair (k, k ^ X) crosses CTAs iff some parity(X & M_b)
  // is odd. Masks are chosen greedily from single qubits and the occupied /
  // virtual / spin classes of hf (and their intersections) by a cost in
  // cycles fitted to per-step clocks on B200 (18 qubits, 2 CTAs): ~600 per
  // generator step that needs a cluster barrier instead of a CTA barrier,
  // ~2.1 per cross generator pair (a DSMEM load and store: DSMEM moves ~20
  // B/cycle), ~0.02 per cross expectation pair (those read a local copy of the
  // peer chunk); every part must fit a CTA.
  auto part_of = [&](uint32_t k, const std::vector<uint64_t>& ms) {
    uint32_t r = 0;
    for (size_t b = 0; b < ms.size(); ++b) r |= (uint32_t)(__builtin_popcountll(k & ms[b]) & 1) << b;
    return r;
  };
  auto crosses = [](uint64_t x, const std::vector<uint64_t>& ms) {
    for (uint64_t m : ms)
      if (__builtin_popcountll(x & m) & 1) return true;
    return false;
  };
  std::vector<uint64_t> cands;
  {
    const uint64_t all = n >= 64 ? ~0ULL : (1ULL << n) - 1, occ = hf & all, vir = all & ~hf;
    uint64_t alpha = 0;
    for (int q = 0; q < n; q += 2) alpha |= 1ULL << q;
    const uint64_t beta = all & ~alpha;
    for (int q = 0; q < n; ++q) cands.push_back(1ULL << q);
    for (uint64_t m : {occ, vir, alpha, beta, occ & alpha, occ & beta, vir & alpha, vir & beta})
      if (m != 0 && m != all && std::find(cands.begin(), cands.end(), m) == cands.end()) cands.push_back(m);
  }
  std::map<uint64_t, int64_t> exp_by_x;
  for (const auto& e : ek) ++exp_by_x[H.groups[e.g].x];
  std::vector<uint64_t> masks;
  double best_cost = 0.0;
  for (int s = 0; (1 << s) < n_parts; ++s) {
    int best = -1;
    for (size_t c = 0; c < cands.size(); ++c) {
      std::vector<uint64_t> m2 = masks;
      m2.push_back(cands[c]);
      std::vector<uint32_t> cnt(size_t(1) << (s + 1), 0);
      for (uint32_t k : list) ++cnt[part_of(k, m2)];
      bool fits = true;
      for (uint32_t v : cnt) fits &= v > 0;  // independent of the earlier masks on S
      if (s + 1 == __builtin_ctz(n_parts))  // final level: every part within a CTA
        for (uint32_t v : cnt) fits &= v <= max_part;
      if (!fits) continue;
      double cost = 0.0;
      for (int op = 0; op < n_ops; ++op) {
        const bool cr = crosses(P.fused[P.op_idx[op]].x, m2);
        const bool nx = op + 1 >= n_ops || crosses(P.fused[P.op_idx[op + 1]].x, m2);
        if (cr || nx) cost += 600.0;
        if (cr) cost += 2.1 * (double)gk[op].size();
      }
      for (const auto& [x, c2] : exp_by_x)
        if (crosses(x, m2)) cost += 0.02 * (double)c2;
      if (best < 0 || cost < best_cost) { best = (int)c; best_cost = cost; }
    }
    if (best < 0) { S.why = "no split of the support closure fits the CTAs"; return S; }
    masks.push_back(cands[best]);
  }
  stage("split");
  if (n_parts == 1 && S.size > max_part) { S.why = "support closure does not fit one CTA"; return S; }
  S.n_parts = n_parts;
  S.split_masks = masks;
  S.op_cross.assign((size_t)n_ops, 0);
  for (int op = 0; op < n_ops; ++op) S.op_cross[op] = crosses(P.fused[P.op_idx[op]].x, masks) ? 1 : 0;
  std::sort(list.begin(), list.end(), [&](uint32_t a, uint32_t c) {
    const uint32_t pa = part_of(a, masks), pc = part_of(c, masks);
    return pa != pc ? pa < pc : a < c;
  });
  S.basis = list;
  S.part_start.assign((size_t)n_parts + 1, 0);
  for (uint32_t k : list) ++S.part_start[part_of(k, masks) + 1];
  for (int r = 0; r < n_parts; ++r) S.part_start[r + 1] += S.part_start[r];
  for (uint32_t i = 0; i < S.size; ++i) idx[list[i]] = (int32_t)i;
  S.hf_idx = (uint32_t)idx[hf];
  // product layout for the one-CTA real program with anchored blocks: S must be
  // exactly (alpha strings) x (beta strings) and fit 15-bit slots when padded
  uint64_t amask = 0;
  for (int q = 0; q < n; q += 2) amask |= 1ULL << q;
  std::vector<uint32_t> slot_of, ia_of, ib_of;
  if (block_warps > 0 && n_parts == 1 && elem_bytes == 8 && S.size > block_min_size) {
    std::vector<uint32_t> sa, sbv;
    for (uint32_t k : list) {
      sa.push_back(k & (uint32_t)amask);
      sbv.push_back(k & ~(uint32_t)amask);
    }
    std::sort(sa.begin(), sa.end());
    sa.erase(std::unique(sa.begin(), sa.end()), sa.end());
    std::sort(sbv.begin(), sbv.end());
    sbv.erase(std::unique(sbv.begin(), sbv.end()), sbv.end());
    const uint32_t stride = (uint32_t)sbv.size() | 1u;
    if ((uint64_t)sa.size() * sbv.size() == S.size && (uint64_t)sa.size() * stride + 1 <= 32768) {
      // order the alpha strings so that the partner strings of every alpha flip
      // mask of the alpha-beta pairs spread over the bank pairs (see alpha_order)
      std::vector<uint64_t> xas;
      for (const auto& e : ek) {
        const uint64_t X = H.groups[e.g].x;
        if ((X & amask) && (X & ~amask)) xas.push_back(X & amask);
      }
      std::sort(xas.begin(), xas.end());
      xas.erase(std::unique(xas.begin(), xas.end()), xas.end());
      // (with the alpha-beta cliques those blocks are gone: natural order)
      if (!cliques) sa = alpha_order(sa, xas, stride);
      S.product = true;
      S.alpha_strings = sa;
      S.beta_strings = sbv;
      S.n_alpha = (uint32_t)sa.size();
      S.n_beta = (uint32_t)sbv.size();
      S.stride_b = stride;
      S.n_slots = S.n_alpha * stride;
      std::map<uint32_t, uint32_t> apos;
      for (uint32_t q = 0; q < (uint32_t)sa.size(); ++q) apos[sa[q]] = q;
      slot_of.resize(S.size);
      ia_of.resize(S.size);
      ib_of.resize(S.size);
      for (uint32_t i = 0; i < S.size; ++i) {
        ia_of[i] = apos.at(list[i] & (uint32_t)amask);
        ib_of[i] = (uint32_t)(std::lower_bound(sbv.begin(), sbv.end(), list[i] & ~(uint32_t)amask) - sbv.begin());
        slot_of[i] = ia_of[i] * stride + ib_of[i];
      }
    }
  }
  if (!S.product) S.n_slots = S.size;
  auto owner = [&](uint32_t i) {
    int r = 0;
    while (i >= S.part_start[r + 1]) ++r;
    return r;
  };
  S.slot_bits = 15 - __builtin_ctz((unsigned)n_parts);
  for (int r = 0; r < n_parts; ++r)
    if (S.part_start[r + 1] - S.part_start[r] >= (1u << S.slot_bits)) { S.why = "part exceeds the slot range"; return S; }
  auto slot = [&](uint32_t i) {
    if (S.product) return slot_of[i];
    const int r = owner(i);
    return ((uint32_t)r << S.slot_bits) | (i - S.part_start[r]);
  };
  S.hf_slot = slot(S.hf_idx);
  if (n_parts == 1) {
    S.slot_of.resize(S.size);
    for (uint32_t i = 0; i < S.size; ++i) S.slot_of[i] = slot(i);
  }
  // 16-byte bank group of S[i] within its CTA's amplitude array
  auto bank_slot = [&](uint32_t i) { return (uint8_t)(slot(i) & (uint32_t)(bank_group - 1)); };
  // a local pair stays with its CTA; a cross pair goes to the lighter of its two CTAs
  auto assign = [&](uint32_t i, uint32_t j, std::vector<int64_t>& load) {
    const int oi = owner(i), oj = owner(j);
    const int o = oi == oj ? oi : (load[oi] <= load[oj] ? oi : oj);
    load[o] += oi == oj ? 2 : 3;  // a cross pair costs one slow DSMEM access
    return o;
  };
  stage("layout");
  S.gen_off.assign(1, 0);
  for (int op = 0; op < n_ops; ++op) {
    const FusedDesc& d = P.fused[P.op_idx[op]];
    std::vector<uint8_t> own(gk[op].size());
    std::vector<int64_t> load((size_t)n_parts, 0);
    for (size_t t = 0; t < gk[op].size(); ++t) {
      const uint32_t i = (uint32_t)idx[gk[op][t].first], j = (uint32_t)idx[gk[op][t].first ^ (uint32_t)d.x];
      own[t] = (uint8_t)assign(i, j, load);
    }
    for (int r = 0; r < n_parts; ++r) {
      std::vector<uint32_t> pi, pj;
      std::vector<uint8_t> fl, ri, rj;
      for (size_t t = 0; t < gk[op].size(); ++t) {
        if (own[t] != r) continue;
        const auto& e = gk[op][t];
        pi.push_back((uint32_t)idx[e.first]);
        pj.push_back((uint32_t)idx[e.first ^ (uint32_t)d.x]);
        fl.push_back(e.second);
        if (real_prog && (fl.back() & 1u)) {  // the sign as a swap of the members
          std::swap(pi.back(), pj.back());
          fl.back() &= (uint8_t)~1u;
        }
        ri.push_back(bank_slot(pi.back()));
        rj.push_back(bank_slot(pj.back()));
      }
      for (uint32_t t : bank_order(ri, rj, bank_group)) {  // thread tid takes pair off + tid
        S.gen_pairs.push_back(real_prog ? slot(pi[t]) | (slot(pj[t]) << 16)
                                        : slot(pi[t]) | (slot(pj[t]) << 15) | ((uint32_t)(fl[t] & 1u) << 30));
        S.gen_flags.push_back(fl[t]);
      }
      S.gen_off.push_back((int64_t)S.gen_pairs.size());
    }
  }
  if (real_prog) {
    const int NT = S.size <= block_min_size ? kSectorHeadSmall : kSectorHeadLarge;
    S.head_threads = NT;
    S.gen_head.assign((size_t)(n_ops + kSectorHeadPad) * 2 * NT, 0xFFFFFFFFu);
    for (int op = 0; op < n_ops; ++op) {
      const int64_t b0 = S.gen_off[op], b1 = S.gen_off[op + 1];
      for (int64_t t = b0; t < std::min<int64_t>(b1, b0 + 2 * NT); ++t)
        S.gen_head[((size_t)2 * op + (size_t)((t - b0) / NT)) * NT + (size_t)((t - b0) % NT)] = S.gen_pairs[t];
      for (int64_t t = b0 + 2 * NT; t < std::min<int64_t>(b1, b0 + 3 * NT); ++t)
        S.gen_head[((size_t)2 * op + 1) * NT + (size_t)(t - b0 - 2 * NT)] |= 1u << 15;  // more words follow
    }
  }
  stage("generator pairs");
  for (const auto& e : ek)
    if (e.fi != 0.0) S.f_real = false;
  S.zero_slot.resize((size_t)n_parts);
  for (int r = 0; r < n_parts; ++r)
    S.zero_slot[r] = ((uint32_t)r << S.slot_bits) | (S.part_start[r + 1] - S.part_start[r]);
  if (S.product) S.zero_slot[0] = S.n_slots;
  for (int r = 0; r < n_parts; ++r) S.hmax = std::max(S.hmax, S.part_start[r + 1] - S.part_start[r]);
  if (S.product) S.hmax = S.n_slots;
  S.buf_off = S.hmax + 1;
  {
    const uint64_t lim = std::min<uint64_t>(cap_amps, 1ull << S.slot_bits);
    const uint64_t room = lim > S.buf_off ? lim - S.buf_off : 0;
    uint32_t peer_max = 0;
    for (int r = 0; r < n_parts; ++r) peer_max = std::max(peer_max, S.part_start[r + 1] - S.part_start[r]);
    S.buf_len = n_parts > 1 && room >= kMinChunk ? (uint32_t)std::min<uint64_t>(room / 32 * 32, peer_max) : 0u;
  }
  const bool buffered = S.buf_len > 0;
  S.exp_pair_count = (int64_t)ek.size();
  std::vector<uint8_t> in_block(ek.size(), 0);
  if (S.product && cliques) {
    // the whole expectation runs in the alpha-first gauge (see compile_cliques):
    // psi'(k) = eps(k) psi(k) (the device negates the eps_flip slots after the
    // generator phase), so every pair weight takes the factor eps(m) eps(m ^ X)
    std::vector<uint8_t> eps(list.size());
    for (size_t i = 0; i < list.size(); ++i) eps[i] = (uint8_t)alpha_first_parity(list[i], n);
    for (auto& e : ek)
      if (eps[idx[e.m]] ^ eps[idx[e.m ^ (uint32_t)H.groups[e.g].x]]) { e.fr = -e.fr; e.fi = -e.fi; }
    S.eps_flip.assign(S.n_slots / 32 + 1, 0u);
    for (size_t i = 0; i < list.size(); ++i)
      if (eps[i]) S.eps_flip[slot_of[i] / 32] |= 1u << (slot_of[i] % 32);
  }
  if (S.product) {
    std::vector<std::pair<uint32_t, uint32_t>> ij(ek.size());
    std::vector<double> fv(ek.size());
    for (size_t t = 0; t < ek.size(); ++t) {
      ij[t] = {(uint32_t)idx[ek[t].m], (uint32_t)idx[ek[t].m ^ (uint32_t)H.groups[ek[t].g].x]};
      fv[t] = ek[t].fr;
    }
    if (cliques) {
      // alpha-beta pairs that factorise go to the cliques, the rest to the blocks
      std::vector<uint8_t> in_clique(ek.size(), 0);
      stage("pair lists");
      compile_cliques(S, list, ij, fv, slot_of, ia_of, ib_of, amask, in_clique);
      stage("cliques");
      std::vector<std::pair<uint32_t, uint32_t>> ij2;
      std::vector<double> fv2;
      std::vector<size_t> back;
      for (size_t t = 0; t < ek.size(); ++t)
        if (!in_clique[t]) { ij2.push_back(ij[t]); fv2.push_back(fv[t]); back.push_back(t); }
      std::vector<uint8_t> in2(ij2.size(), 0);
      compile_blocks(S, list, ij2, fv2, slot_of, ia_of, ib_of, amask, in2);
      for (size_t u = 0; u < back.size(); ++u) in_block[back[u]] = in2[u];
      for (size_t t = 0; t < ek.size(); ++t) in_block[t] |= in_clique[t];
    } else {
      compile_blocks(S, list, ij, fv, slot_of, ia_of, ib_of, amask, in_block);
    }
  }
  stage("cliques+blocks");
  std::vector<uint8_t> eown(ek.size());
  {  // balance: with the chunk buffer a cross pair costs about what a local one does
    std::vector<int64_t> load((size_t)n_parts, 0);
    for (size_t t = 0; t < ek.size(); ++t) {
      const uint32_t i = (uint32_t)idx[ek[t].m], j = (uint32_t)idx[ek[t].m ^ (uint32_t)H.groups[ek[t].g].x];
      const int oi = owner(i), oj = owner(j);
      const int o = oi == oj ? oi : (load[oi] <= load[oj] ? oi : oj);
      load[o] += oi == oj || buffered ? 2 : 3;
      eown[t] = (uint8_t)o;
    }
  }
  S.sec_off.assign(1, 0);
  std::vector<uint32_t> pp_words;  // staged per-pair rows of the current section
  std::vector<double> pp_re, pp_im;
  int32_t pf_rows = 0;
  for (int r = 0; r < n_parts; ++r) {
    const uint32_t zpair = S.zero_slot[r] | (S.zero_slot[r] << 15);
    // section key: 0 = local (and, unbuffered, every cross pair), else 1 + chunk id
    auto key_of = [&](uint32_t i, uint32_t j) -> int64_t {
      const int oi = owner(i), oj = owner(j);
      if (oi == oj || !buffered) return 0;
      const uint32_t peer = oi == r ? j : i;
      const int rp = oi == r ? oj : oi;
      return 1 + (int64_t)rp * 65536 + (peer - S.part_start[rp]) / S.buf_len;
    };
    auto enc = [&](uint32_t x, int64_t key) -> uint32_t {
      if (owner(x) == r || key == 0) return slot(x);
      const int rp = owner(x);
      const uint32_t chunk0 = (uint32_t)(((key - 1) % 65536) * S.buf_len);
      return ((uint32_t)r << S.slot_bits) | (S.buf_off + (x - S.part_start[rp] - chunk0));
    };
    std::map<int64_t, std::vector<size_t>> secs;  // ek indices in (group, pattern) order
    for (size_t t = 0; t < ek.size(); ++t) {
      if (eown[t] != r || in_block[t]) continue;
      const uint32_t i = (uint32_t)idx[ek[t].m], j = (uint32_t)idx[ek[t].m ^ (uint32_t)H.groups[ek[t].g].x];
      secs[key_of(i, j)].push_back(t);
    }
    if (secs.empty()) secs[0];
    for (auto& [key, list] : secs) {
      SectorProgram::ExpSection es{};
      if (key > 0) {
        es.src_rank = (int32_t)((key - 1) / 65536);
        es.src_off = (int32_t)(((key - 1) % 65536) * S.buf_len);
        es.len = (int32_t)std::min<uint32_t>(S.buf_len, S.part_start[es.src_rank + 1] - S.part_start[es.src_rank] - es.src_off);
      }
      es.sh0 = (int32_t)(S.row_pairs.size() / 32);
      pp_words.clear();
      pp_re.clear();
      pp_im.clear();
      size_t a0 = 0;
      while (a0 < list.size()) {
        size_t b0 = a0 + 1;
        while (b0 < list.size() && ek[list[b0]].g == ek[list[a0]].g && ek[list[b0]].p == ek[list[a0]].p) ++b0;
        // one (group, pattern) set: encode, bank-order, pad to rows
        std::vector<uint32_t> si, sj;
        std::vector<uint8_t> ri, rj;
        for (size_t u = a0; u < b0; ++u) {
          const auto& e = ek[list[u]];
          const uint32_t i = (uint32_t)idx[e.m], j = (uint32_t)idx[e.m ^ (uint32_t)H.groups[e.g].x];
          si.push_back(enc(i, key));
          sj.push_back(enc(j, key));
          ri.push_back((uint8_t)(si.back() & (uint32_t)(bank_group - 1)));
          rj.push_back((uint8_t)(sj.back() & (uint32_t)(bank_group - 1)));
        }
        const std::vector<uint32_t> order = bank_order(ri, rj, bank_group);
        const double fr0 = ek[list[a0]].fr, fi0 = ek[list[a0]].fi;
        bool shared = true;
        for (size_t u = a0; u < b0; ++u) {
          const auto& e = ek[list[u]];
          if (!((e.fr == fr0 && e.fi == fi0) || (e.fr == -fr0 && e.fi == -fi0))) { shared = false; break; }
        }
        const size_t cnt = b0 - a0, padded = (cnt + 31) / 32 * 32;
        for (size_t u = 0; u < padded; ++u) {
          uint32_t word = zpair;
          double fr = 0.0, fi = 0.0;
          if (u < cnt) {
            const uint32_t v = order[u];
            const auto& e = ek[list[a0 + v]];
            const uint32_t neg = shared && (e.fr != fr0 || e.fi != fi0) ? 1u : 0u;
            word = si[v] | (sj[v] << 15) | (neg << 30);
            fr = e.fr;
            fi = e.fi;
          }
          if (shared) {
            S.row_pairs.push_back(word);
          } else {
            pp_words.push_back(word);
            pp_re.push_back(fr);
            pp_im.push_back(fi);
          }
        }
        if (shared)
          for (size_t u = 0; u < padded / 32; ++u) {
            S.row_fre.push_back(fr0);
            S.row_fim.push_back(fi0);
          }
        a0 = b0;
      }
      // pad both row ranges to whole multiples of row_quantum (4 rows x warps
      // per CTA on the device): every warp then owns whole groups of 4 rows
      auto pad_rows = [&](std::vector<uint32_t>& words, int64_t first_row, std::vector<double>* re,
                          std::vector<double>* im) {
        int64_t rows = (int64_t)words.size() / 32 - first_row;
        while (rows % row_quantum) {
          words.insert(words.end(), 32, zpair);
          if (re) re->insert(re->end(), 32, 0.0);
          if (im) im->insert(im->end(), 32, 0.0);
          ++rows;
        }
      };
      pad_rows(S.row_pairs, es.sh0, nullptr, nullptr);
      S.row_fre.resize(S.row_pairs.size() / 32, 0.0);
      S.row_fim.resize(S.row_pairs.size() / 32, 0.0);
      if (!pp_words.empty()) pad_rows(pp_words, 0, &pp_re, &pp_im);
      es.sh1 = (int32_t)(S.row_pairs.size() / 32);
      S.row_pairs.insert(S.row_pairs.end(), pp_words.begin(), pp_words.end());
      S.row_fre.resize(S.row_pairs.size() / 32, 0.0);
      S.row_fim.resize(S.row_pairs.size() / 32, 0.0);
      S.pf_re.insert(S.pf_re.end(), pp_re.begin(), pp_re.end());
      S.pf_im.insert(S.pf_im.end(), pp_im.begin(), pp_im.end());
      es.pp1 = (int32_t)(S.row_pairs.size() / 32);
      es.pf_base = pf_rows;
      pf_rows += es.pp1 - es.sh1;
      S.sections.push_back(es);
    }
    S.sec_off.push_back((int32_t)S.sections.size());
  }
  stage("generic rows");
  if (S.f_real) {
    S.row_fim.clear();
    S.pf_im.clear();
  }
  if (S.product) {
    // warps take equal shares of the generic rows (the kernel splits them
    // evenly); block units go to the least-loaded warp, largest first, and
    // each warp's units become one row stream
    const int nw = block_warps;
    const auto& es = S.sections[0];
    const double generic = (es.sh1 - es.sh0) * 7.5 + (es.pp1 - es.sh1) * 9.0;
    const size_t nu = S.blk_units.size() / 8;
    std::vector<size_t> ord(nu);
    for (size_t u = 0; u < nu; ++u) ord[u] = u;
    auto ucost = [&](size_t u) { const int32_t* h = &S.blk_units[8 * u]; return 4.0 * (1 + h[5]) + 6.0 * h[6]; };
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ucost(a) > ucost(b); });
    std::vector<double> load((size_t)nw, generic / nw);
    std::vector<std::vector<size_t>> mine((size_t)nw);
    // clique warp tasks first (the largest items), then the block units
    const size_t nwt = S.cq_desc.size() / 128;
    std::vector<std::vector<size_t>> cq_mine((size_t)nw);
    for (size_t t = 0; t < nwt; ++t) {
      int rows = 0;
      for (int l = 0; l < 32; ++l) rows = std::max(rows, S.cq_desc[(t * 32 + l) * 4 + 3] - S.cq_desc[(t * 32 + l) * 4 + 2]);
      const size_t w = (size_t)(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += 25.0 * rows + 30.0;
      cq_mine[w].push_back(t);
    }
    for (size_t u : ord) {
      const size_t w = (size_t)(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += ucost(u);
      mine[w].push_back(u);
    }
    if (nwt) {  // each warp's clique tasks contiguous
      std::vector<int32_t> desc;
      std::vector<double> coef;
      S.cq_warp.clear();
      for (int w = 0; w < nw; ++w) {
        S.cq_warp.push_back((int32_t)(desc.size() / 128));
        for (size_t t : cq_mine[w]) {
          desc.insert(desc.end(), &S.cq_desc[t * 128], &S.cq_desc[t * 128] + 128);
          coef.insert(coef.end(), &S.cq_coef[t * kCliquePairs * 32], &S.cq_coef[t * kCliquePairs * 32] + kCliquePairs * 32);
        }
        S.cq_warp.push_back((int32_t)(desc.size() / 128));
      }
      S.cq_desc.swap(desc);
      S.cq_coef.swap(coef);
    }
    // A warp's stream is cut at unit boundaries into kBlkSegments segments of about
    // equal length, each padded to whole prefetch rounds: the kernel sums every
    // segment from zero and adds the segment sums in order, so the role warps of a
    // split evaluation can take one segment each (same bits as one warp running all).
    // Among the unit boundaries within a twelfth of the stream of the even cuts,
    // the pair with the least padding is taken (ties: the most even cut).
    S.blk_warp.clear();
    for (int w = 0; w < nw; ++w) {
      std::sort(mine[w].begin(), mine[w].end());
      static_assert(kBlkSegments == 3, "two cuts are chosen below");
      std::vector<int64_t> edge{0};  // rows before unit k of this warp
      for (size_t u : mine[w]) edge.push_back(edge.back() + 1 + S.blk_units[8 * u + 5]);
      const int64_t total = edge.back();
      auto padded = [](int64_t rows) { return (rows + kStreamQuantum - 1) / kStreamQuantum * kStreamQuantum; };
      auto near = [&](int64_t target) {
        std::vector<size_t> c;
        for (size_t k = 0; k < edge.size(); ++k)
          if (std::llabs(edge[k] - target) * 12 <= total) c.push_back(k);
        if (c.empty()) c.push_back(std::lower_bound(edge.begin(), edge.end(), target) - edge.begin());
        return c;
      };
      size_t cut_unit[2] = {edge.size() - 1, edge.size() - 1};
      {
        int64_t best_pad = -1, best_skew = 0;
        for (size_t c1 : near(total / 3))
          for (size_t c2 : near(2 * total / 3)) {
            if (c2 < c1) continue;
            const int64_t l[3] = {edge[c1], edge[c2] - edge[c1], total - edge[c2]};
            const int64_t pad = padded(l[0]) + padded(l[1]) + padded(l[2]) - total;
            const int64_t skew = std::max({l[0], l[1], l[2]});
            if (best_pad < 0 || pad < best_pad || (pad == best_pad && skew < best_skew)) {
              best_pad = pad, best_skew = skew;
              cut_unit[0] = c1, cut_unit[1] = c2;
            }
          }
      }
      const int32_t r0 = (int32_t)(S.blk_stream.size() / 32);
      int32_t cut[kBlkSegments - 1], seg0 = r0;
      auto pad = [&]() {
        while ((S.blk_stream.size() / 32 - seg0) % kStreamQuantum) S.blk_stream.insert(S.blk_stream.end(), 32, 0u);
        seg0 = (int32_t)(S.blk_stream.size() / 32);
      };
      for (size_t k = 0; k <= mine[w].size(); ++k) {
        for (int c = 0; c < kBlkSegments - 1; ++c)
          if (k == cut_unit[c]) {
            pad();
            cut[c] = seg0;
          }
        if (k == mine[w].size()) break;
        const int32_t* h = &S.blk_units[8 * mine[w][k]];
        for (int l = 0; l < 32; ++l) S.blk_stream.push_back(S.blk_lanes[(size_t)h[0] * 32 + l] | (1u << 30));
        for (int r = 0; r < h[5]; ++r)
          S.blk_stream.insert(S.blk_stream.end(), &S.blk_sh[((size_t)h[1] + r) * 32],
                              &S.blk_sh[((size_t)h[1] + r) * 32] + 32);
      }
      pad();
      const int32_t r1 = seg0;
      static_assert(kBlkSegments == 3, "blk_warp holds {begin, end, cut 1, cut 2}");
      S.blk_warp.insert(S.blk_warp.end(), {r0, r1, cut[0], cut[1]});
    }
  }
  stage("warp streams");
  S.ok = true;
  return S;
}

}  // namespace ffq

namespace ffq {

// ---- Krylov space of a Hamiltonian (lanczos_ground / energy_exact) ---------------
// Basis = closure of |hf> under the Hamiltonian's pair maps (m <-> m ^ X on the
// active patterns of every x-group) and, optionally, a plan's generator maps;
// H and the generator matrix A = sum_g theta_g A_g restricted to it are kept as
// CSR (rows = basis states, deterministic row-wise sums on the device).
struct KrylovSpace {
  bool ok = false;
  std::string why;
  std::vector<uint32_t> basis;  // ascending
  uint32_t hf_idx = 0;
  // H: row i, entries (col, value) with value = <basis[i]|H|basis[col]>
  std::vector<int64_t> h_row;
  std::vector<uint32_t> h_col;
  std::vector<double> h_re, h_im;
  // A_g: entries (row, col, value, generator column in theta)
  std::vector<int64_t> a_row;
  std::vector<uint32_t> a_col;
  std::vector<double> a_re, a_im;
  std::vector<int32_t> a_gen;
};

// Closure under H's maps (lanczos_ground) or under the plan's maps only
// (energy_exact: <psi|H|psi> only needs H restricted to psi's support).
inline KrylovSpace compile_krylov(const CompiledHam& H, const CompiledPlan* P, uint64_t hf, uint32_t max_size,
                                  bool close_under_h) {
  KrylovSpace K;
  const int n = H.n_qubits;
  if (n > 26) { K.why = "qubit count"; return K; }
  if (P && P->n_string_ops() > 0) { K.why = "plan has non-fused generators"; return K; }
  const size_t dim = size_t(1) << n;
  std::vector<int32_t> pos(dim, -1);
  std::vector<uint32_t> list{(uint32_t)hf};
  pos[hf] = 0;
  // breadth-first closure under all maps
  for (size_t t = 0; t < list.size(); ++t) {
    const uint32_t k = list[t];
    auto add = [&](uint32_t m) {
      if (pos[m] < 0) { pos[m] = (int32_t)list.size(); list.push_back(m); }
    };
    for (const auto& d : H.groups) {
      if (d.x == 0 || !close_under_h) continue;
      uint64_t Q = 0;
      for (int i = 0; i < d.w; ++i) Q |= 1ULL << d.q[i];
      for (int p = 0; p < d.nact; ++p) {
        const uint64_t pb = H.act_bits[d.act_off + p];
        if ((k & Q) == pb || ((k ^ d.x) & Q) == pb) add(k ^ (uint32_t)d.x);
      }
    }
    if (P)
      for (const auto& d : P->fused)
        for (int p = 0; p < d.npair; ++p) {
          const uint64_t lo = P->pair_bits[d.pair_off + p];
          const uint64_t pat = k & d.x;
          if (pat == lo || pat == (lo ^ d.x)) add(k ^ (uint32_t)d.x);
        }
    if (list.size() > max_size) { K.why = "Krylov space too large"; return K; }
  }
  std::sort(list.begin(), list.end());
  for (size_t i = 0; i < list.size(); ++i) pos[list[i]] = (int32_t)i;
  K.basis = list;
  K.hf_idx = (uint32_t)pos[hf];
  // H entries: for pair (m, m^X) with pattern p (lower member m), <m^X|H|m> = f/2
  // (off-diagonal, f carries the pair weight 2) and its conjugate transpose
  std::vector<std::vector<std::tuple<uint32_t, double, double>>> rows(list.size());
  for (const auto& d : H.groups) {
    uint64_t Q = 0;
    for (int i = 0; i < d.w; ++i) Q |= 1ULL << d.q[i];
    for (int p = 0; p < d.nact; ++p) {
      const uint64_t pb = H.act_bits[d.act_off + p];
      for (uint32_t i = 0; i < list.size(); ++i) {
        const uint32_t m = list[i];
        if ((m & Q) != pb) continue;
        const int32_t j = pos[m ^ (uint32_t)d.x];
        if (j < 0) continue;
        double fr = 0.0, fi = 0.0;
        for (int o = 0; o < d.ncls; ++o) {
          const double sg = (__builtin_popcountll(m & H.cls_z[d.cls_off + o]) & 1) ? -1.0 : 1.0;
          fr += sg * H.cls_f[2 * (d.val_off + o * d.nact + p)];
          fi += sg * H.cls_f[2 * (d.val_off + o * d.nact + p) + 1];
        }
        if (d.x == 0) {
          rows[i].emplace_back(i, fr, fi);
        } else {
          // <m^X|H|m> = b(m) = f/2; <m|H|m^X> = conj(b(m))
          rows[j].emplace_back(i, 0.5 * fr, 0.5 * fi);
          rows[i].emplace_back((uint32_t)j, 0.5 * fr, -0.5 * fi);
        }
      }
    }
  }
  K.h_row.push_back(0);
  for (auto& r : rows) {
    std::sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
    for (auto& e : r) {
      K.h_col.push_back(std::get<0>(e));
      K.h_re.push_back(std::get<1>(e));
      K.h_im.push_back(std::get<2>(e));
    }
    K.h_row.push_back((int64_t)K.h_col.size());
  }
  // A_g entries: <k^X|A_g|k> = s_out(k) F[pattern(k)], k on either pattern of a pair
  if (P) {
    std::vector<std::vector<std::tuple<uint32_t, double, double, int32_t>>> arows(list.size());
    for (size_t op = 0; op < P->op_kind.size(); ++op) {
      const FusedDesc& d = P->fused[P->op_idx[op]];
      for (int p = 0; p < d.npair; ++p) {
        const uint64_t lo = P->pair_bits[d.pair_off + p];
        const double flr = P->pair_f[4 * (d.pair_off + p)], fli = P->pair_f[4 * (d.pair_off + p) + 1];
        const double fhr = P->pair_f[4 * (d.pair_off + p) + 2], fhi = P->pair_f[4 * (d.pair_off + p) + 3];
        for (uint32_t i = 0; i < list.size(); ++i) {
          const uint32_t k = list[i];
          const uint64_t pat = k & d.x;
          if (pat != lo && pat != (lo ^ d.x)) continue;
          const int32_t j = pos[k ^ (uint32_t)d.x];
          if (j < 0) continue;
          const double sg = (__builtin_popcountll(k & d.zout) & 1) ? -1.0 : 1.0;
          const bool low = pat == lo;
          // A_g |k> = a(k) |k^X>, a(k) = s_out(k) F[pattern(k)] (compile_plan's F table)
          const double ar = sg * (low ? flr : fhr), ai = sg * (low ? fli : fhi);
          arows[j].emplace_back(i, ar, ai, P->op_gen[op]);
        }
      }
    }
    K.a_row.push_back(0);
    for (auto& r : arows) {
      for (auto& e : r) {
        K.a_col.push_back(std::get<0>(e));
        K.a_re.push_back(std::get<1>(e));
        K.a_im.push_back(std::get<2>(e));
        K.a_gen.push_back(std::get<3>(e));
      }
      K.a_row.push_back((int64_t)K.a_col.size());
    }
  }
  K.ok = true;
  return K;
}

}  // namespace ffq
