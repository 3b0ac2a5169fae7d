// ffq_kernels.cuh -- sm_100a kernels of the UCCSD state-vector hot path.
//
// State layout in HBM: [batch][2^n] complex128 (double2), natural binary
// order, qubit 0 = LSB. Every kernel is an HBM/L2 stream over
// amplitude pairs (k, k ^ X); none uses tensor cores (north_star).
//
//   k_pauli_rotation  e^{i phi P} on one string: 32-byte vector loads of two
//                     neighbouring amplitudes (ld.global.v4.f64), one pass of
//                     32 * 2^n bytes -- the "rotation pass" of the roofline.
//   k_fused_gen       one UCCSD generator exp(theta (tau - tau^dag)) as an
//                     exact rotation over the active bit patterns of X only
//                     (1/8 of the state for a double, 1/2 for a single).
//   k_expect_items    <psi|H|psi> over (group, pattern, chunk) work items;
//                     each amplitude pair read once per x-group; block
//                     partials in fixed slots -> k_reduce_partials (fixed tree).
//   k_smem_eval       n <= 13: one CTA per energy evaluation, state resident
//                     in shared memory from HF build to the final reduction.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ffq_compile.hpp"

namespace ffq {

struct PlanDev {
  int n_ops;
  const int32_t* op_kind;
  const int32_t* op_gen;
  const int32_t* op_idx;
  const double* op_cfac;
  const double* op_sscale;
  const FusedDesc* fused;
  const uint64_t* pair_bits;
  const double2* pair_f;  // [pair][2]: F[pi], F[~pi]
  const uint64_t* str_x;
  const uint64_t* str_z;
  const int32_t* str_ny;
};

struct HamDev {
  int n_groups;
  const GroupDesc* groups;
  const uint64_t* act_bits;
  const uint64_t* cls_z;
  const double2* cls_f;
  int64_t n_items;
  const int32_t* item_g;
  const int32_t* item_p;
  const int64_t* item_u0;
  int64_t item_chunk;
  int64_t sitem_words;  // support words per support-path item
};

// ---- small helpers -----------------------------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// i^k
__device__ __forceinline__ double2 ipow_d(int k) {
  k &= 3;
  return make_double2(k == 0 ? 1.0 : (k == 2 ? -1.0 : 0.0), k == 1 ? 1.0 : (k == 3 ? -1.0 : 0.0));
}
// insert zero bits at the ascending positions packed 6 bits apiece in qpack
template <typename I>
__device__ __forceinline__ I insert_bits(I u, uint64_t qpack, int w) {
  for (int i = 0; i < w; ++i) {
    const int b = (int)((qpack >> (6 * i)) & 63u);
    u = ((u >> b) << (b + 1)) | (u & ((I(1) << b) - I(1)));
  }
  return u;
}
template <typename I>
__device__ __forceinline__ I insert_zero(I u, int b) {
  return ((u >> b) << (b + 1)) | (u & ((I(1) << b) - I(1)));
}
__device__ __forceinline__ double sgn_par(uint64_t v) { return (__popcll(v) & 1) ? -1.0 : 1.0; }

// 32-byte vector access (two complex128 amplitudes): LDG.E.ENL2.256 on sm_100a
__device__ __forceinline__ void ld256(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ void st256(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x),
               "d"(b.y)
               : "memory");
}

// ---- per-op rotation coefficients: cs[b][op] = (cos phi, sin phi * sscale) --
__global__ void k_op_cs(const double* __restrict__ theta, int theta_stride, int n_ops,
                        const int32_t* __restrict__ op_gen, const double* __restrict__ op_cfac,
                        const double* __restrict__ op_sscale, double2* __restrict__ cs, int batch) {
  const int64_t total = (int64_t)n_ops * batch;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / n_ops), op = (int)(t % n_ops);
    const double phi = theta[(int64_t)b * theta_stride + op_gen[op]] * op_cfac[op];
    double s, c;
    sincos(phi, &s, &c);
    cs[t] = make_double2(c, s * op_sscale[op]);
  }
}

// ---- basis state -------------------------------------------------------------
__global__ void k_set_basis(double2* __restrict__ psi, int64_t dim, int batch, uint64_t bits) {
  const int64_t total = dim * batch;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t % dim;
    psi[t] = make_double2(k == (int64_t)bits ? 1.0 : 0.0, 0.0);
  }
}

// ---- single Pauli-string rotation e^{i phi P} --------------------------------
// new[k]  = c a + s w sgn(k') b,  new[k'] = c b + s w sgn(k) a,  w = i * i^{ny}
// mode 0: x == 0 (diagonal phase), mode 1: bit 0 of x clear, mode 2: x == 1,
// mode 3: bit 0 of x set with other bits. Each thread owns one 32-byte vector
// pair so every global access is a full LDG/STG.256.
__global__ void __launch_bounds__(256) k_pauli_rotation(double2* __restrict__ psi, int n,
                                                        uint64_t x, uint64_t z, int ny,
                                                        const double2* __restrict__ cs,
                                                        int cs_stride, int op, int mode,
                                                        int hbit) {
  const int b = blockIdx.y;
  double2* s = psi + ((int64_t)b << n);
  const double2 csv = cs[(int64_t)b * cs_stride + op];
  const double c = csv.x, sn = csv.y;
  const double2 w = ipow_d(ny + 1);
  const int64_t nvec = (mode == 0 || mode == 2) ? (1LL << (n - 1)) : (1LL << (n - 2));
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nvec;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (mode == 0) {
      const uint64_t k = (uint64_t)t << 1;
      double2 a0, a1;
      ld256(s + k, a0, a1);
      // (c + i s sgn) a
      const double s0 = sn * sgn_par(k & z), s1 = sn * sgn_par((k + 1) & z);
      const double2 r0 = make_double2(c * a0.x - s0 * a0.y, c * a0.y + s0 * a0.x);
      const double2 r1 = make_double2(c * a1.x - s1 * a1.y, c * a1.y + s1 * a1.x);
      st256(s + k, r0, r1);
    } else if (mode == 1) {
      const uint64_t k = insert_zero<uint64_t>((uint64_t)t << 1, hbit);  // even, bit h clear
      const uint64_t kp = k ^ x;
      double2 a0, a1, b0, b1;
      ld256(s + k, a0, a1);
      ld256(s + kp, b0, b1);
      const double sk0 = sn * sgn_par(k & z), sk1 = sn * sgn_par((k + 1) & z);
      const double sp0 = sn * sgn_par(kp & z), sp1 = sn * sgn_par((kp + 1) & z);
      const double2 wb0 = cmul(w, b0), wb1 = cmul(w, b1), wa0 = cmul(w, a0), wa1 = cmul(w, a1);
      const double2 na0 = make_double2(c * a0.x + sp0 * wb0.x, c * a0.y + sp0 * wb0.y);
      const double2 na1 = make_double2(c * a1.x + sp1 * wb1.x, c * a1.y + sp1 * wb1.y);
      const double2 nb0 = make_double2(c * b0.x + sk0 * wa0.x, c * b0.y + sk0 * wa0.y);
      const double2 nb1 = make_double2(c * b1.x + sk1 * wa1.x, c * b1.y + sk1 * wa1.y);
      st256(s + k, na0, na1);
      st256(s + kp, nb0, nb1);
    } else if (mode == 2) {
      const uint64_t k = (uint64_t)t << 1;  // pair (k, k+1) inside one vector
      double2 a, bb;
      ld256(s + k, a, bb);
      const double sk = sn * sgn_par(k & z), sp = sn * sgn_par((k + 1) & z);
      const double2 wb = cmul(w, bb), wa = cmul(w, a);
      const double2 na = make_double2(c * a.x + sp * wb.x, c * a.y + sp * wb.y);
      const double2 nb = make_double2(c * bb.x + sk * wa.x, c * bb.y + sk * wa.y);
      st256(s + k, na, nb);
    } else {
      // k even with bit h' (lowest bit of x & ~1) clear; j = k ^ (x & ~1)
      // pairs: (k, j+1) and (k+1, j)
      const uint64_t k = insert_zero<uint64_t>((uint64_t)t << 1, hbit);
      const uint64_t j = k ^ (x & ~1ULL);
      double2 a0, a1, b0, b1;
      ld256(s + k, a0, a1);
      ld256(s + j, b0, b1);
      // pair (k, j+1): a = a0, b = b1
      const double sA_k = sn * sgn_par(k & z), sA_p = sn * sgn_par((j + 1) & z);
      // pair (k+1, j): a = a1, b = b0
      const double sB_k = sn * sgn_par((k + 1) & z), sB_p = sn * sgn_par(j & z);
      const double2 wb1 = cmul(w, b1), wa0 = cmul(w, a0), wb0 = cmul(w, b0), wa1 = cmul(w, a1);
      const double2 na0 = make_double2(c * a0.x + sA_p * wb1.x, c * a0.y + sA_p * wb1.y);
      const double2 nb1 = make_double2(c * b1.x + sA_k * wa0.x, c * b1.y + sA_k * wa0.y);
      const double2 na1 = make_double2(c * a1.x + sB_p * wb0.x, c * a1.y + sB_p * wb0.y);
      const double2 nb0 = make_double2(c * b0.x + sB_k * wa1.x, c * b0.y + sB_k * wa1.y);
      st256(s + k, na0, na1);
      st256(s + j, nb0, nb1);
    }
  }
}

// ---- fused generator: exp(theta A) on the active patterns of X ----------------
// pair (k, kb = k ^ X), k = insert(u) | bits(pi_lo):
//   new[k]  = c a + s' sgn_out(k) F[pi_hi] b,  new[kb] = c b + s' sgn_out(k) F[pi_lo] a
// sign_base: rank bits of a shard (k | sign_base is the full index), 0 unsharded
template <bool VEC>
__global__ void __launch_bounds__(256) k_fused_gen(double2* __restrict__ psi, int n, FusedDesc d,
                                                   const uint64_t* __restrict__ pair_bits,
                                                   const double2* __restrict__ pair_f,
                                                   const double2* __restrict__ cs, int cs_stride,
                                                   int op, uint64_t sign_base) {
  const int b = blockIdx.y;
  double2* s = psi + ((int64_t)b << n);
  const double2 csv = cs[(int64_t)b * cs_stride + op];
  const double c = csv.x, sn = csv.y;
  const int ub = n - d.w;
  const int64_t per_pair = VEC ? (1LL << (ub - 1)) : (1LL << ub);
  const int64_t total = per_pair * d.npair;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / per_pair);
    const int64_t u = t - (int64_t)p * per_pair;
    const uint64_t pb = pair_bits[d.pair_off + p];
    const double2 flo = pair_f[2 * (d.pair_off + p)], fhi = pair_f[2 * (d.pair_off + p) + 1];
    if (VEC) {
      const uint64_t k = insert_bits<uint64_t>((uint64_t)u << 1, d.qpack, d.w) | pb;
      const uint64_t kb = k ^ d.x;
      double2 a0, a1, b0, b1;
      ld256(s + k, a0, a1);
      ld256(s + kb, b0, b1);
      // an all-zero pair stays zero: skip the write-back (exact)
      if (a0.x == 0.0 && a0.y == 0.0 && a1.x == 0.0 && a1.y == 0.0 && b0.x == 0.0 && b0.y == 0.0 &&
          b1.x == 0.0 && b1.y == 0.0)
        continue;
      const double g0 = sn * sgn_par((k | sign_base) & d.zout), g1 = sn * sgn_par(((k + 1) | sign_base) & d.zout);
      const double2 hb0 = cmul(fhi, b0), hb1 = cmul(fhi, b1);
      const double2 la0 = cmul(flo, a0), la1 = cmul(flo, a1);
      st256(s + k, make_double2(c * a0.x + g0 * hb0.x, c * a0.y + g0 * hb0.y),
            make_double2(c * a1.x + g1 * hb1.x, c * a1.y + g1 * hb1.y));
      st256(s + kb, make_double2(c * b0.x + g0 * la0.x, c * b0.y + g0 * la0.y),
            make_double2(c * b1.x + g1 * la1.x, c * b1.y + g1 * la1.y));
    } else {
      const uint64_t k = insert_bits<uint64_t>((uint64_t)u, d.qpack, d.w) | pb;
      const uint64_t kb = k ^ d.x;
      const double2 a = s[k], bb = s[kb];
      if (a.x == 0.0 && a.y == 0.0 && bb.x == 0.0 && bb.y == 0.0) continue;
      const double g = sn * sgn_par((k | sign_base) & d.zout);
      const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
      s[k] = make_double2(c * a.x + g * hb.x, c * a.y + g * hb.y);
      s[kb] = make_double2(c * bb.x + g * la.x, c * bb.y + g * la.y);
    }
  }
}

// ---- block reduction with a fixed tree (deterministic) -----------------------
template <int NT>
__device__ __forceinline__ double2 block_sum(double2 v, double2* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < NT / 32 ? sh[lane] : make_double2(0, 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_down_sync(0xffffffffu, v.x, o);
      v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
  }
  return v;  // valid in thread 0
}

// ---- expectation over work items ---------------------------------------------
// partial[b][item] = sum_{u in item} Re(conj(psi[m ^ X]) psi[m] sum_o sgn(m & z_o) F[o][p]);
// the imaginary lane stays 0 (Hermitian groups are enforced at upload)
template <int NT>
__global__ void __launch_bounds__(NT) k_expect_items(const double2* __restrict__ psi, int n,
                                                     HamDev h, double2* __restrict__ partial) {
  __shared__ double2 red[NT / 32];
  const int64_t item = blockIdx.x;
  const int b = blockIdx.y;
  const double2* s = psi + ((int64_t)b << n);
  const int g = h.item_g[item], p = h.item_p[item];
  const int64_t u0 = h.item_u0[item];
  const GroupDesc d = h.groups[g];
  const int64_t U = 1LL << (n - d.w);
  const int64_t u1 = min(U, u0 + h.item_chunk);
  const uint64_t pb = h.act_bits[d.act_off + p];
  double2 acc = make_double2(0, 0);
  // members with the X bits clear, stepped by NT with a masked add (the carries
  // run through the X positions): no per-member bit insertion
  uint64_t Q = 0;  // inserted positions: all of X in table mode, X's highest bit in generic mode
  for (int i = 0; i < d.w; ++i) Q |= 1ULL << ((d.qpack >> (6 * i)) & 63u);
  const uint64_t step = insert_bits<uint64_t>((uint64_t)NT, d.qpack, d.w);
  uint64_t mz = insert_bits<uint64_t>((uint64_t)(u0 + threadIdx.x), d.qpack, d.w);
  // four members per trip, every load issued before the class sums (the dense
  // path streams the whole state: the loads, not the arithmetic, are the cost)
  constexpr int UN = 4;
  for (int64_t u = u0 + threadIdx.x; u < u1; u += (int64_t)UN * NT) {
    uint64_t mm[UN];
    double2 av[UN], bv[UN];
#pragma unroll
    for (int j = 0; j < UN; ++j) {
      mm[j] = mz | pb;
      const bool live = u + (int64_t)j * NT < u1;
      av[j] = live ? s[mm[j]] : make_double2(0.0, 0.0);
      bv[j] = live ? s[mm[j] ^ d.x] : make_double2(0.0, 0.0);
      mz = ((mz | Q) + step) & ~Q;
    }
#pragma unroll
    for (int j = 0; j < UN; ++j) {
      const double2 a = av[j], bb = bv[j];
      if (a.x == 0.0 && a.y == 0.0) continue;  // zero product (also the members past the chunk)
      const uint64_t m = mm[j];
      double2 f = make_double2(0, 0);
      for (int o = 0; o < d.ncls; ++o) {
        const double sg = sgn_par(m & h.cls_z[d.cls_off + o]);
        const double2 fo = h.cls_f[d.val_off + o * d.nact + p];
        f.x = fma(sg, fo.x, f.x);
        f.y = fma(sg, fo.y, f.y);
      }
      // Re(conj(bb) * a * f); the weight 2 of off-diagonal pairs is folded into F
      const double2 pr = make_double2(bb.x * a.x + bb.y * a.y, bb.x * a.y - bb.y * a.x);
      acc.x = fma(pr.x, f.x, acc.x);
      acc.x = fma(-pr.y, f.y, acc.x);
    }
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)b * gridDim.x + item] = acc;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_reduce_partials(const double2* __restrict__ partial,
                                                        int64_t n_items,
                                                        double* __restrict__ e_out,
                                                        double* __restrict__ im_out) {
  __shared__ double2 red[NT / 32];
  const int b = blockIdx.x;
  const double2* pp = partial + (int64_t)b * n_items;
  double2 acc = make_double2(0, 0);
  for (int64_t i = threadIdx.x; i < n_items; i += NT) {
    acc.x += pp[i].x;
    acc.y += pp[i].y;
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) {
    e_out[b] = acc.x;
    if (im_out) im_out[b] = acc.y;
  }
}

// ---- sharded expectation -------------------------------------------------------
// One rank's contribution for the groups of one out-of-shard flip pattern hG:
// items (group, pattern, chunk); the enumerated member m lives on this rank
// (its pattern's rank bits must equal this rank's bits on hG), its partner
// m ^ X lives at local index m_local ^ X_local on rank r ^ hG (`partner`).
template <int NT>
__global__ void __launch_bounds__(NT) k_expect_shard(const double2* __restrict__ own,
                                                     const double2* __restrict__ partner, int l,
                                                     uint32_t rank, HamDev h, int64_t item0,
                                                     double2* __restrict__ partial) {
  __shared__ double2 red[NT / 32];
  const int64_t item = item0 + blockIdx.x;
  const int g = h.item_g[item], p = h.item_p[item];
  const int64_t u0 = h.item_u0[item];
  const GroupDesc d = h.groups[g];
  const uint64_t lmask = (1ULL << l) - 1ULL;
  const uint64_t XL = d.x & lmask;
  // inserted (pattern-fixed) positions: all of X in table mode, X's highest bit in generic mode
  uint64_t Q = 0;
  for (int i = 0; i < d.w; ++i) Q |= 1ULL << ((d.qpack >> (6 * i)) & 63u);
  const uint32_t QG = (uint32_t)(Q >> l);
  const uint64_t pb = h.act_bits[d.act_off + p];
  double acc = 0.0;
  if ((rank & QG) == ((uint32_t)(pb >> l) & QG)) {
    const int wl = __popcll(Q & lmask);
    const int64_t U = 1LL << (l - wl);
    const int64_t u1 = min(U, u0 + h.item_chunk);
    const uint64_t base = (uint64_t)rank << l;
    for (int64_t u = u0 + threadIdx.x; u < u1; u += NT) {
      const uint64_t ml = insert_bits<uint64_t>((uint64_t)u, d.qpack, wl) | (pb & lmask);
      const double2 a = own[ml];
      if (a.x == 0.0 && a.y == 0.0) continue;
      const double2 bb = partner[ml ^ XL];
      const uint64_t m = base | ml;
      double fx = 0.0, fy = 0.0;
      for (int o = 0; o < d.ncls; ++o) {
        const double sg = sgn_par(m & h.cls_z[d.cls_off + o]);
        const double2 fo = h.cls_f[d.val_off + o * d.nact + p];
        fx = fma(sg, fo.x, fx);
        fy = fma(sg, fo.y, fy);
      }
      const double prx = bb.x * a.x + bb.y * a.y, pry = bb.x * a.y - bb.y * a.x;
      acc = fma(prx, fx, acc);
      acc = fma(-pry, fy, acc);
    }
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) partial[item] = tot;
}

// Several one-term x-groups of one out-of-shard flip pattern hG in one pass over
// the shard's support bitmap: every non-zero local member m is enumerated (both
// orientations of a pair: sum_m Re(conj(psi[m ^ X]) psi[m] c i^ny (-1)^popc(m & z))
// equals the pair-once sum with weight 2 for a Hermitian term), so all groups
// share the m stream, and a partner amplitude is gathered only where the
// partner's bitmap has its bit set (for a random X a few percent of the
// partners of a UCCSD state are non-zero). Bitmaps: bit k % 32 of word k / 32,
// conservative supersets are fine (a zero amplitude contributes zero). CTA =
// (chunk of bitmap words, batch); partial[item0 + batch * chunks + chunk].
struct ShardTerm {
  uint64_t xl, z;  // flip mask inside the shard; full z (physical positions, rank bits included)
  double2 f;       // c i^ny
};
template <int NT>
__global__ void __launch_bounds__(NT) k_expect_shard_multi(const double2* __restrict__ own,
                                                           const double2* __restrict__ partner,
                                                           const uint32_t* __restrict__ own_sup,
                                                           const uint32_t* __restrict__ partner_sup, int l,
                                                           uint32_t rank, const ShardTerm* __restrict__ terms,
                                                           const int2* __restrict__ batches, int batch0,
                                                           int64_t chunk_words, int64_t item0,
                                                           double2* __restrict__ partial) {
  __shared__ double2 red[NT / 32];
  __shared__ ShardTerm st[16];
  const int2 bt = batches[batch0 + blockIdx.y];  // first term, term count (<= 16)
  if (threadIdx.x < bt.y) st[threadIdx.x] = terms[bt.x + threadIdx.x];
  __syncthreads();
  const uint64_t base = (uint64_t)rank << l;
  const int64_t w1 = min((int64_t)1 << (l - 5), ((int64_t)blockIdx.x + 1) * chunk_words);
  double acc = 0.0;
  for (int64_t w = (int64_t)blockIdx.x * chunk_words + threadIdx.x; w < w1; w += NT) {
    uint32_t bits = own_sup[w];
    while (bits) {
      const uint64_t m = ((uint64_t)w << 5) | (uint32_t)(__ffs((int)bits) - 1);
      bits &= bits - 1u;
      const double2 a = own[m];
      const uint64_t M = base | m;
      for (int t = 0; t < bt.y; ++t) {
        const uint64_t pm = m ^ st[t].xl;
        if (!((__ldg(partner_sup + (pm >> 5)) >> (pm & 31u)) & 1u)) continue;
        const double2 bb = partner[pm];
        const double sg = sgn_par(M & st[t].z);
        const double prx = bb.x * a.x + bb.y * a.y, pry = bb.x * a.y - bb.y * a.x;
        acc = fma(sg * prx, st[t].f.x, acc);
        acc = fma(-sg * pry, st[t].f.y, acc);
      }
    }
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) partial[item0 + (int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
}

// ---- global-qubit swap ------------------------------------------------------------
// Pack / unpack the half shard whose local bit `lpos` differs from this rank's
// bit `gbit` (it moves to the partner r ^ (1 << gbit)); in-place after exchange.
__global__ void k_swap_pack(const double2* __restrict__ s, double2* __restrict__ buf, int l, int lpos,
                            int val) {
  const int64_t half = 1LL << (l - 1);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < half;
       u += (int64_t)gridDim.x * blockDim.x)
    buf[u] = s[insert_zero<uint64_t>((uint64_t)u, lpos) | ((uint64_t)val << lpos)];
}
__global__ void k_swap_unpack(double2* __restrict__ s, const double2* __restrict__ buf, int l, int lpos,
                              int val) {
  const int64_t half = 1LL << (l - 1);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < half;
       u += (int64_t)gridDim.x * blockDim.x)
    s[insert_zero<uint64_t>((uint64_t)u, lpos) | ((uint64_t)val << lpos)] = buf[u];
}
// Support-compacted swap: only the amplitudes whose support bit is set move.
// bits of word w that belong to the half with local bit lpos == val
__device__ __forceinline__ uint32_t swap_half_bits(uint32_t word, int64_t w, int lpos, int val) {
  if (lpos >= 5) return (((uint64_t)w >> (lpos - 5)) & 1ULL) == (uint64_t)val ? word : 0u;
  uint32_t m = 0;  // offsets o in the word with bit lpos of o equal to val
#pragma unroll
  for (uint32_t o = 0; o < 32; ++o) m |= (((o >> lpos) & 1u) == (uint32_t)val ? 1u : 0u) << o;
  return word & m;
}
__global__ void k_swap_count(const uint32_t* __restrict__ sup, int l, int lpos, int val,
                             unsigned long long* __restrict__ count) {
  const int64_t words = 1LL << (l - 5);
  unsigned long long n = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
    n += (unsigned)__popc(swap_half_bits(sup[w], w, lpos, val));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(count, n);
}
// move the supported amplitudes of the half out: (index within the half, value)
// pairs in any order (the unpack scatters by index), slots and bits cleared
__global__ void k_swap_pack_sparse(double2* __restrict__ s, uint32_t* __restrict__ sup, int l, int lpos, int val,
                                   double2* __restrict__ vals, uint32_t* __restrict__ idx,
                                   unsigned long long* __restrict__ cursor) {
  const int64_t words = 1LL << (l - 5);
  const int lane = threadIdx.x & 31;
  // whole warps iterate together (words is a multiple of 32 for l >= 10; the
  // guard keeps short shards correct): one cursor atomic per warp
  for (int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; w0 < words;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = w0 + lane;
    const uint32_t word = w < words ? sup[w] : 0u;
    uint32_t bits = w < words ? swap_half_bits(word, w, lpos, val) : 0u;
    const uint32_t n = (uint32_t)__popc(bits);
    uint32_t incl = n;  // inclusive scan of the lane counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (!total) continue;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(cursor, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (!bits) continue;
    unsigned long long at = base + (incl - n);
    sup[w] = word & ~bits;
    while (bits) {
      const uint64_t k = ((uint64_t)w << 5) | (uint32_t)(__ffs((int)bits) - 1);
      bits &= bits - 1u;
      vals[at] = s[k];
      s[k] = make_double2(0.0, 0.0);
      idx[at] = (uint32_t)(((k >> (lpos + 1)) << lpos) | (k & ((1ULL << lpos) - 1ULL)));  // bit lpos removed
      ++at;
    }
  }
}
__global__ void k_swap_unpack_sparse(double2* __restrict__ s, uint32_t* __restrict__ sup, int lpos, int val,
                                     const double2* __restrict__ vals, const uint32_t* __restrict__ idx,
                                     unsigned long long count) {
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < count;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const uint64_t k = insert_zero<uint64_t>((uint64_t)idx[t], lpos) | ((uint64_t)val << lpos);
    s[k] = vals[t];
    atomicOr(&sup[k >> 5], 1u << (k & 31u));
  }
}
// both ranks of a pair on one device: exchange in place
__global__ void k_swap_pair(double2* __restrict__ s0, double2* __restrict__ s1, int l, int lpos) {
  const int64_t half = 1LL << (l - 1);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < half;
       u += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = insert_zero<uint64_t>((uint64_t)u, lpos);
    const uint64_t k0 = k | (1ULL << lpos), k1 = k;  // rank bit 0 sends lpos=1, rank bit 1 sends lpos=0
    const double2 t = s0[k0];
    s0[k0] = s1[k1];
    s1[k1] = t;
  }
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk copy of this thread's bulk group; the generic-proxy
// writes to the tile must be fenced (fence_async_smem) before it is issued
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---- fused run of low-qubit rotations on TMA-staged tiles ------------------------
// A run of consecutive rotations e^{i phi_r P_r} whose flip masks all lie in
// the low t qubits maps every 2^t-amplitude tile (contiguous: the high bits of
// the index are fixed) onto itself. One CTA stages its tile with bulk copies
// (cp.async.bulk + mbarrier), applies the whole run in shared memory, and
// writes the tile back with 32-byte stores: the state crosses HBM once per run
// (32 B per amplitude) instead of once per rotation.
// Inside the tile the run is cut (on the host) into groups of consecutive
// rotations whose flip masks span at most 3 dimensions over GF(2). A group has
// a reduced-echelon basis {b_0, b_1, b_2} with pivot bits p_i (b_i has bit p_i,
// no other b_j does); the cosets k ^ span{b} with the pivot bits of k clear
// partition the tile into 2^(t-3) sets of 8, and every pair (k', k' ^ x) of
// every rotation of the group lies inside one coset. Each thread loads one
// coset into registers, applies the group's rotations in order there, and
// stores it: one shared-memory round trip per group instead of per rotation,
// one CTA barrier per group. A pivot is the highest set bit of its reduced
// flip mask (padding vectors take the highest free bits), so it can be a low
// bit (x = 1 gives pivot 0): then consecutive coset indices u spread to
// non-adjacent k and a quarter warp's 16-byte accesses can conflict. This
// costs bandwidth only; the result does not depend on the pivot choice.
// z is unrestricted: the tile's high-bit parity is folded into sin once per
// rotation. Per pair the arithmetic is k_pauli_rotation's.
struct RotDesc {
  uint64_t x, z;  // in tile coordinates (pext by the run's qubit set Q): x, z < 2^t
  uint64_t zo;    // z & ~Q (full index bits): the tile's part of the parity
  int ny;         // popc(x & z) & 3 of the original string
  int cx;         // x in its group's basis: bit i set <=> b_i in x (x = 0: diagonal)
};
struct RotGroup {
  int r0, r1;        // rotations [r0, r1) of the run
  uint32_t b[3];     // reduced-echelon basis (padded with unit vectors to 3)
  int piv[3];        // pivot bits, ascending
};

// rotation of the coset registers v[0..7] on the pairs (e, e ^ CX), e < e ^ CX.
// w = i^(ny+1) is +-1 (IM = false, ws = w) or +-i (IM = true, ws = Im w), so
// w b is a sign and (for +-i) a swap: no complex multiply. sg[e] = +-sin phi.
// sg[e] already carries the sign of w (ws * sin phi * parity sign, exact).
template <int CX, bool IM>
__device__ __forceinline__ void coset_pairs(double2 (&v)[8], double c, const double (&sg)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (e < (e ^ CX)) {
      const int f = e ^ CX;
      const double2 a = v[e], b = v[f];
      if (IM) {
        v[e] = make_double2(c * a.x - sg[f] * b.y, c * a.y + sg[f] * b.x);
        v[f] = make_double2(c * b.x - sg[e] * a.y, c * b.y + sg[e] * a.x);
      } else {
        v[e] = make_double2(c * a.x + sg[f] * b.x, c * a.y + sg[f] * b.y);
        v[f] = make_double2(c * b.x + sg[e] * a.x, c * b.y + sg[e] * a.y);
      }
    }
  }
}
template <bool IM>
__device__ __forceinline__ void coset_rot(int cx, double2 (&v)[8], double c, const double (&sg)[8]) {
  switch (cx) {
    case 1: coset_pairs<1, IM>(v, c, sg); break;
    case 2: coset_pairs<2, IM>(v, c, sg); break;
    case 3: coset_pairs<3, IM>(v, c, sg); break;
    case 4: coset_pairs<4, IM>(v, c, sg); break;
    case 5: coset_pairs<5, IM>(v, c, sg); break;
    case 6: coset_pairs<6, IM>(v, c, sg); break;
    default: coset_pairs<7, IM>(v, c, sg); break;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 3) k_rotation_run(double2* __restrict__ psi, int n, int t, uint64_t q,
                                                     const RotGroup* __restrict__ grp, int n_grp,
                                                     const RotDesc* __restrict__ rd,
                                                     const double2* __restrict__ cs, int cs_stride) {
  // rotation r of row b: (cos phi, sin phi) = cs[b * cs_stride + r].
  // The tile is the 2^t amplitudes whose bits outside the qubit set q are
  // those of blockIdx.x; tile coordinate m <-> index base | pdep(m, q).
  // q = the low t bits: one contiguous block, staged by bulk copies. Otherwise
  // q holds the low 5 bits, so 32 consecutive m are 512 contiguous bytes
  // (one 512-byte bulk copy per entry of a 2^(t-5)-entry offset table).
  extern __shared__ __align__(128) double2 tl[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint64_t hi_off[128];
  const uint32_t tsize = 1u << t;
  const uint64_t nmask = (n >= 64) ? ~0ULL : ((1ULL << n) - 1ULL);
  const bool low = q == (uint64_t)(tsize - 1u);
  __shared__ uint64_t base_sh;
  uint64_t base = (uint64_t)blockIdx.x << t;
  if (!low) {  // pdep(blockIdx.x, ~q): one thread, broadcast
    if (threadIdx.x == 0) {
      uint64_t rest = ~q & nmask, bx = blockIdx.x, bs = 0;
      while (rest) {
        const uint64_t lsb = rest & (~rest + 1ULL);
        if (bx & 1ULL) bs |= lsb;
        bx >>= 1;
        rest ^= lsb;
      }
      base_sh = bs;
    }
    __syncthreads();
    base = base_sh;
  }
  double2* s = psi + ((int64_t)blockIdx.y << n) + base;
  const double2* csb = cs + (int64_t)blockIdx.y * cs_stride;
  // the tile arrives by bulk copies (TMA) on one mbarrier: two 32 KiB pieces when
  // q is the low t bits, else one 512-byte piece per offset-table entry
  if (low) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      const uint32_t bytes = tsize * (uint32_t)sizeof(double2);
      mbar_expect_tx(&bar, bytes);
      const uint32_t piece = 32768;
      for (uint32_t off = 0; off < bytes; off += piece)
        bulk_g2s((char*)tl + off, (const char*)s + off, min(piece, bytes - off), &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
  } else {
    const uint64_t qh = q & ~31ULL;
    for (uint32_t j = threadIdx.x; j < (tsize >> 5); j += NT) {
      uint64_t o = 0, rest = qh, bj = j;
      while (rest) {
        const uint64_t lsb = rest & (~rest + 1ULL);
        if (bj & 1ULL) o |= lsb;
        bj >>= 1;
        rest ^= lsb;
      }
      hi_off[j] = o;
    }
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, tsize * (uint32_t)sizeof(double2));
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < (tsize >> 5); j += NT) bulk_g2s(tl + 32 * j, s + hi_off[j], 512, &bar);
    mbar_wait(&bar, 0);
  }
  for (int g = 0; g < n_grp; ++g) {
    const RotGroup G = grp[g];
    uint32_t off[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      off[c] = ((c & 1) ? G.b[0] : 0u) ^ ((c & 2) ? G.b[1] : 0u) ^ ((c & 4) ? G.b[2] : 0u);
    for (uint32_t u = threadIdx.x; u < (tsize >> 3); u += NT) {
      const uint32_t k = insert_zero<uint32_t>(insert_zero<uint32_t>(insert_zero<uint32_t>(u, G.piv[0]), G.piv[1]),
                                               G.piv[2]);
      double2 v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = tl[k ^ off[c]];
      for (int r = G.r0; r < G.r1; ++r) {
        const uint32_t zl = (uint32_t)__ldg(&rd[r].z);
        const int cx = __ldg(&rd[r].cx);
        const double2 csv = __ldg(&csb[r]);
        const double c = csv.x, sn = csv.y * sgn_par(base & __ldg(&rd[r].zo));
        // parity of (k ^ off[e]) & z = parity(k & z) ^ parity(off[e] & z), the
        // second a XOR of the basis parities: one sign flip of sin per member
        const uint32_t p0 = (uint32_t)__popc(G.b[0] & zl) << 31, p1 = (uint32_t)__popc(G.b[1] & zl) << 31,
                       p2 = (uint32_t)__popc(G.b[2] & zl) << 31;  // basis parities in bit 31
        const int wk = cx ? (__ldg(&rd[r].ny) + 1) & 3 : 0;  // w = i^wk (pairs only)
        const double snw = (wk == 2 || wk == 3) ? -sn : sn;   // sign of w folded into sin
        const double snk = (__popc(k & zl) & 1u) ? -snw : snw;
        uint32_t hi[8];
        hi[0] = (uint32_t)__double2hiint(snk);
        hi[1] = hi[0] ^ p0;
        hi[2] = hi[0] ^ p1;
        hi[3] = hi[1] ^ p1;
#pragma unroll
        for (int e = 0; e < 4; ++e) hi[4 + e] = hi[e] ^ p2;
        const int lo = __double2loint(snk);
        double sg[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) sg[e] = __hiloint2double((int)hi[e], lo);
        if (cx == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const double2 a = v[e];
            v[e] = make_double2(c * a.x - sg[e] * a.y, c * a.y + sg[e] * a.x);
          }
        } else {
          if (wk & 1)
            coset_rot<true>(cx, v, c, sg);
          else
            coset_rot<false>(cx, v, c, sg);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) tl[k ^ off[c]] = v[c];
    }
    __syncthreads();
  }
  // write-back by bulk copies from the tile (the last group's barrier precedes)
  fence_async_smem();
  __syncthreads();
  if (low) {
    if (threadIdx.x == 0) {
      const uint32_t bytes = tsize * (uint32_t)sizeof(double2), piece = 32768;
      for (uint32_t off = 0; off < bytes; off += piece)
        bulk_s2g((char*)s + off, (const char*)tl + off, min(piece, bytes - off));
      bulk_commit_wait_read();
    }
  } else if (threadIdx.x < (tsize >> 5)) {
    for (uint32_t j = threadIdx.x; j < (tsize >> 5); j += NT) bulk_s2g(s + hi_off[j], tl + 32 * j, 512);
    bulk_commit_wait_read();
  }
}

// ---- shared-memory-resident evaluator (n <= 13) ------------------------------
// One CTA per evaluation: HF build, every plan op, and the grouped expectation
// run on the smem copy of the state; the only HBM traffic is theta in and E out.
template <int NT>
__global__ void __launch_bounds__(NT) k_smem_eval(int n, PlanDev pl, HamDev h, uint64_t hf_bits,
                                                  const double* __restrict__ theta,
                                                  int theta_stride, double* __restrict__ e_out,
                                                  double* __restrict__ im_out) {
  extern __shared__ double2 sm[];
  __shared__ double2 red[NT / 32];
  const int b = blockIdx.x;
  const uint32_t dim = 1u << n;
  double2* st = sm;                 // [dim]
  double2* cs = sm + dim;           // [n_ops]
  for (uint32_t k = threadIdx.x; k < dim; k += NT)
    st[k] = make_double2(k == (uint32_t)hf_bits ? 1.0 : 0.0, 0.0);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)b * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double s, c;
    sincos(phi, &s, &c);
    cs[op] = make_double2(c, s * pl.op_sscale[op]);
  }
  __syncthreads();
  for (int op = 0; op < pl.n_ops; ++op) {
    const double2 csv = cs[op];
    const double c = csv.x, sn = csv.y;
    if (pl.op_kind[op] == 0) {
      const FusedDesc d = pl.fused[pl.op_idx[op]];
      const int w = d.w;
      const uint64_t X = d.x, zo = d.zout;
      const int ub = n - w;
      const uint32_t total = (uint32_t)d.npair << ub;
      for (uint32_t t = threadIdx.x; t < total; t += NT) {
        const int p = (int)(t >> ub);
        const uint32_t u = t & ((1u << ub) - 1u);
        const uint32_t k = insert_bits<uint32_t>(u, d.qpack, w) | (uint32_t)pl.pair_bits[d.pair_off + p];
        const uint32_t kb = k ^ (uint32_t)X;
        const double2 flo = pl.pair_f[2 * (d.pair_off + p)], fhi = pl.pair_f[2 * (d.pair_off + p) + 1];
        const double2 a = st[k], bb = st[kb];
        const double g = sn * sgn_par(k & zo);
        const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
        st[k] = make_double2(c * a.x + g * hb.x, c * a.y + g * hb.y);
        st[kb] = make_double2(c * bb.x + g * la.x, c * bb.y + g * la.y);
      }
    } else {
      const int si = pl.op_idx[op];
      const uint32_t x = (uint32_t)pl.str_x[si], z = (uint32_t)pl.str_z[si];
      const double2 w = ipow_d(pl.str_ny[si] + 1);
      if (x == 0) {
        for (uint32_t k = threadIdx.x; k < dim; k += NT) {
          const double2 a = st[k];
          const double sg = sn * sgn_par(k & z);
          st[k] = make_double2(c * a.x - sg * a.y, c * a.y + sg * a.x);
        }
      } else {
        const int hb = __ffs(x) - 1;
        for (uint32_t t = threadIdx.x; t < dim / 2; t += NT) {
          const uint32_t k = insert_zero<uint32_t>(t, hb), kp = k ^ x;
          const double2 a = st[k], bb = st[kp];
          const double sk = sn * sgn_par(k & z), sp = sn * sgn_par(kp & z);
          const double2 wb = cmul(w, bb), wa = cmul(w, a);
          st[k] = make_double2(c * a.x + sp * wb.x, c * a.y + sp * wb.y);
          st[kp] = make_double2(c * bb.x + sk * wa.x, c * bb.y + sk * wa.y);
        }
      }
    }
    __syncthreads();
  }
  // grouped expectation, fixed per-thread order
  double2 acc = make_double2(0, 0);
  for (int g = 0; g < h.n_groups; ++g) {
    const GroupDesc d = h.groups[g];
    const uint32_t X = (uint32_t)d.x;
    const int ub = n - d.w;
    const uint32_t total = (uint32_t)d.nact << ub;
    for (uint32_t t = threadIdx.x; t < total; t += NT) {
      const int p = (int)(t >> ub);
      const uint32_t u = t & ((1u << ub) - 1u);
      const uint32_t m = insert_bits<uint32_t>(u, d.qpack, d.w) | (uint32_t)h.act_bits[d.act_off + p];
      const double2 a = st[m], bb = st[m ^ X];
      double2 f = make_double2(0, 0);
      for (int o = 0; o < d.ncls; ++o) {
        const double sg = sgn_par(m & h.cls_z[d.cls_off + o]);
        const double2 fo = h.cls_f[d.val_off + o * d.nact + p];
        f.x = fma(sg, fo.x, f.x);
        f.y = fma(sg, fo.y, f.y);
      }
      const double2 pr = make_double2(bb.x * a.x + bb.y * a.y, bb.x * a.y - bb.y * a.x);
      acc.x = fma(pr.x, f.x, acc.x);
      acc.x = fma(-pr.y, f.y, acc.x);
    }
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) {
    e_out[b] = acc.x;
    if (im_out) im_out[b] = acc.y;
  }
}

}  // namespace ffq
