// ffq_sector.cuh -- support-closure evaluator: one energy evaluation per
// thread-block cluster with the state's |S| amplitudes in distributed shared
// memory (see SectorProgram in ffq_compile.hpp).
//
// S (the amplitudes reachable from |hf> through the plan's pair maps) is
// theta-independent, and every amplitude outside it is identically zero, so
// the evaluation keeps exactly S on chip: 15 876 complex128 values = 254 KB
// at 18 qubits, split over the CL = 2 CTAs of a cluster. Generator g is one
// pass over its precompiled pairs (i, j) of S -- the (k, k ^ X) pairing of
// the dense pass restricted to S -- and consecutive generators are separated
// by a cluster barrier instead of a kernel launch. The expectation is one pass
// over the precompiled (m, m ^ X) pairs with their class sums f(m). Pair
// tables are shared by every evaluation of the batch (L2-resident); the only
// per-evaluation HBM traffic is theta in and E out.
#pragma once

#include <cooperative_groups.h>

#include "ffq_kernels.cuh"

namespace ffq {

namespace cg = cooperative_groups;

constexpr int kSectorMaxParts = 8;

struct SectorDev {
  uint32_t size, hf_slot;
  uint32_t part_start[kSectorMaxParts + 1];  // CTA r holds S[part_start[r], part_start[r + 1])
  int n_ops, n_parts, f_real;
  int real;                     // 1: real-amplitude program (k_sector_eval_real)
  const uint8_t* op_cross;      // [n_ops] 1: the generator has pairs across CTAs (cluster barrier)
  const int64_t* gen_off;       // [CL * n_ops + 1], per op and owner rank
  const uint32_t* gen_pairs;    // slot_i | slot_j << 15 | sign << 30
  const uint32_t* gen_head;     // real one-CTA program: per-thread head words (SectorProgram::gen_head)
  const uint8_t* gen_flags;     // pattern pair index << 1 (read only for multi-pattern ops)
  // expectation rows in sections (SectorProgram::ExpSection): 32 pair words each
  int32_t sec_off[kSectorMaxParts + 1];
  uint32_t buf_off, buf_len;    // chunk copy buffer: amplitude indices [buf_off, buf_off + buf_len)
  const int32_t* secs;          // [n_sec * 7]: src_rank, src_off, len, sh0, sh1, pp1, pf_base
  const uint32_t* row_pairs;
  const double* row_fre;        // [rows] (0 on per-pair rows)
  const double* row_fim;        // nullptr when every f is real
  const double* pf_re;          // [per-pair rows * 32]
  const double* pf_im;          // nullptr when every f is real
  // product layout + anchored string blocks (real one-CTA program; SectorProgram::blk_*)
  uint32_t n_slots;             // amplitude slots (zero slot = n_slots)
  const int4* blk_warp;         // [warps]: row stream [x, y); nullptr: no blocks
  const uint32_t* blk_stream;   // [rows * 32] lane words
  const double* ftab;           // [n_ftab] shared-row f values (copied to shared memory)
  int n_ftab;
  // alpha-beta cliques (SectorProgram::cq_*); nullptr: none
  const uint32_t* eps_flip;     // slots negated into the alpha-first gauge before the expectation (nullptr: none)
  const uint32_t* cq_rows;      // ia * stride | ia' * stride << 15 | neg << 31
  const int4* cq_desc;          // [warp tasks][32]: columns 0-3, columns 4-5, row begin, row end
  const int2* cq_warp;          // [warps]: warp-task range
  const double* cq_coef;        // [warp tasks][15][32]
  // host side only: the (address, bytes) ranges of the tables above, for k_l2_warm
  const ulonglong2* warm;
  int n_warm;
  int max_warp_tasks;  // most clique tasks of one warp share
};

// Pull table ranges into L2 with every SM: a batch far below the SM count would
// otherwise stream its ~13 MB of tables through the few SMs that compute, at
// single-SM HBM bandwidth, whenever the tables are not L2-resident.
__global__ void k_l2_warm(const ulonglong2* __restrict__ ranges, int n) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < n; ++r) {
    const ulonglong2 rg = ranges[r];
    for (uint64_t off = t * 128; off < rg.y; off += stride * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rg.x + off));
  }
}

// Amplitude slots (SectorProgram::slot_bits): 15 - log2(CL) offset bits, the
// owning rank above them. Addresses are 32-bit shared::cluster addresses (the
// shared::cta window when CL == 1).
template <int CL>
struct SlotMap {
  static constexpr int kBits = CL == 1 ? 15 : (CL == 2 ? 14 : (CL == 4 ? 13 : 12));
  uint32_t base[CL];
  uint32_t local;  // this CTA's amplitudes in the shared::cta window
  // slot of this CTA's own part (or its chunk buffer): shared::cta address
  __device__ __forceinline__ uint32_t laddr(uint32_t s) const {
    return local + ((s & ((1u << kBits) - 1u)) << 4);
  }
  __device__ __forceinline__ uint32_t addr(uint32_t s) const {
    const uint32_t off = (s & ((1u << kBits) - 1u)) << 4;
    if (CL == 1) return base[0] + off;
    const uint32_t r = (s >> kBits) & (CL - 1);
    uint32_t b = base[0];
#pragma unroll
    for (int q = 1; q < CL; ++q) b = r == (uint32_t)q ? base[q] : b;
    return b + off;
  }
};

template <int CL>
__device__ __forceinline__ double2 sld(uint32_t a) {
  double2 v;
  if (CL == 1)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  else
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

template <int CL>
__device__ __forceinline__ void sst(uint32_t a, double2 v) {
  if (CL == 1)
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y));
  else
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y));
}

// sum over shared-|f| rows [r0, r1) of f_row * sign * conj(psi[j]) psi[i]
// (real part; with !FR also the imaginary one); lane takes word row * 32 + lane,
// four rows per trip with the next trip's pair words already in flight
// LOCAL: every slot is this CTA's (own part or chunk buffer): plain shared::cta loads
template <int CL, bool FR, bool LOCAL>
__device__ __forceinline__ double shared_rows(const SectorDev& sd, int r0, int r1, int lane, const SlotMap<CL>& sm) {
  // r1 - r0 is a multiple of 4 (rows padded at compile time)
  double acc = 0.0;
  if (r0 >= r1) return acc;
  uint32_t wn[4];
  double fn[4], fin[4];
  auto fetch = [&](int row) {
    const uint32_t* p = sd.row_pairs + (size_t)row * 32 + lane;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      wn[u] = __ldg(p + 32 * u);
      fn[u] = __ldg(sd.row_fre + row + u);
      if (!FR) fin[u] = __ldg(sd.row_fim + row + u);
    }
  };
  fetch(r0);
  for (int row = r0; row < r1; row += 4) {
    uint32_t w[4];
    double f[4], fi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      w[u] = wn[u];
      f[u] = fn[u];
      if (!FR) fi[u] = fin[u];
    }
    if (row + 4 < r1) fetch(row + 4);
    double2 a[4], bb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (LOCAL) {
        a[u] = sld<1>(sm.laddr(w[u] & 0x7FFFu));
        bb[u] = sld<1>(sm.laddr((w[u] >> 15) & 0x7FFFu));
      } else {
        a[u] = sld<CL>(sm.addr(w[u] & 0x7FFFu));
        bb[u] = sld<CL>(sm.addr((w[u] >> 15) & 0x7FFFu));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // sign bit 30 of the pair word flips f's sign bit
      const long long sgn = (long long)((w[u] >> 30) & 1u) << 63;
      const double fs = __longlong_as_double(__double_as_longlong(f[u]) ^ sgn);
      acc = fma(fs, fma(bb[u].x, a[u].x, bb[u].y * a[u].y), acc);
      if (!FR) {
        const double fis = __longlong_as_double(__double_as_longlong(fi[u]) ^ sgn);
        acc = fma(-fis, fma(bb[u].x, a[u].y, -bb[u].y * a[u].x), acc);
      }
    }
  }
  return acc;
}

// per-pair-f rows [r0, r1) (f at pf[(row - pp0) * 32 + lane], pp0 = the row of pf ordinal 0)
template <int CL, bool LOCAL>
__device__ __forceinline__ double perpair_rows(const SectorDev& sd, int r0, int r1, int pp0, int lane,
                                               const SlotMap<CL>& sm) {
  // r1 - r0 is a multiple of 4 (rows padded at compile time)
  double acc = 0.0;
  for (int row = r0; row < r1; row += 4) {
    uint32_t w[4];
    double fr[4], fi[4];
    const uint32_t* p = sd.row_pairs + (size_t)row * 32 + lane;
    const int64_t fo = (int64_t)(row - pp0) * 32 + lane;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      w[u] = __ldg(p + 32 * u);
      fr[u] = __ldg(sd.pf_re + fo + 32 * u);
      fi[u] = sd.pf_im ? __ldg(sd.pf_im + fo + 32 * u) : 0.0;
    }
    double2 a[4], bb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (LOCAL) {
        a[u] = sld<1>(sm.laddr(w[u] & 0x7FFFu));
        bb[u] = sld<1>(sm.laddr((w[u] >> 15) & 0x7FFFu));
      } else {
        a[u] = sld<CL>(sm.addr(w[u] & 0x7FFFu));
        bb[u] = sld<CL>(sm.addr((w[u] >> 15) & 0x7FFFu));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double prx = fma(bb[u].x, a[u].x, bb[u].y * a[u].y);
      const double pry = fma(bb[u].x, a[u].y, -bb[u].y * a[u].x);
      acc = fma(prx, fr[u], acc);
      acc = fma(-pry, fi[u], acc);
    }
  }
  return acc;
}

// one generator's pairs assigned to this CTA: exp(theta A) as the 2x2 rotation
// a' = c a + g F_hi b, b' = c b + g F_lo a per pair (g = +-s by the pair's sign)
template <int CL, int NT, bool MULTI, bool LOCAL, bool REALF = false>
__device__ __forceinline__ void gen_pass(const SectorDev& sd, const PlanDev& pl, int op, uint32_t t0, uint32_t t1,
                                         uint32_t w, double2 csv, double2 flo, double2 fhi, const SlotMap<CL>& sm) {
  for (uint32_t t = t0; t < t1; t += NT) {
    if (t != t0) w = __ldg(sd.gen_pairs + t);
    if (MULTI) {  // more than one active pattern pair (not UCCSD)
      const int po = pl.fused[pl.op_idx[op]].pair_off + (__ldg(sd.gen_flags + t) >> 1);
      flo = pl.pair_f[2 * po];
      fhi = pl.pair_f[2 * po + 1];
    }
    const bool neg = (w >> 30) & 1u;
    constexpr int AS = LOCAL ? 1 : CL;  // address space: shared::cta or shared::cluster
    const uint32_t pa = LOCAL ? sm.laddr(w & 0x7FFFu) : sm.addr(w & 0x7FFFu);
    const uint32_t pb = LOCAL ? sm.laddr((w >> 15) & 0x7FFFu) : sm.addr((w >> 15) & 0x7FFFu);
    const double2 a = sld<AS>(pa), bb = sld<AS>(pb);
    if (REALF) {  // F real: flo.x / fhi.x carry sin * F (sign applied here)
      const double gh = neg ? -fhi.x : fhi.x, gl = neg ? -flo.x : flo.x;
      sst<AS>(pa, make_double2(fma(gh, bb.x, csv.x * a.x), fma(gh, bb.y, csv.x * a.y)));
      sst<AS>(pb, make_double2(fma(gl, a.x, csv.x * bb.x), fma(gl, a.y, csv.x * bb.y)));
    } else {
      const double g = neg ? -csv.y : csv.y;
      const double2 hb = cmul(fhi, bb), la = cmul(flo, a);
      sst<AS>(pa, make_double2(csv.x * a.x + g * hb.x, csv.x * a.y + g * hb.y));
      sst<AS>(pb, make_double2(csv.x * bb.x + g * la.x, csv.x * bb.y + g * la.y));
    }
  }
}

template <int CL, int NT>
__global__ void __launch_bounds__(NT, 1) k_sector_eval(SectorDev sd, PlanDev pl, const double* __restrict__ theta,
                                                       int theta_stride, double* __restrict__ e_out,
                                                       double* __restrict__ im_out, int n_rows,
                                                       long long* __restrict__ phase_clk) {
  // dynamic smem: [Hmax + 1] amplitudes (the last ones of each part stay 0: the
  // zero slot of padded rows) | [n_ops] (cos, sin*scale) | [n_ops] (F_lo, F_hi)
  // of pattern pair 0 | [n_ops] this rank's pair range | [n_ops] flags
  extern __shared__ __align__(16) double2 sm_c[];
  __shared__ double2 red[NT / 32];
  __shared__ double cl_part[CL];
  const long long clk0 = clock64();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CL == 1 ? 0 : (int)cluster.block_rank();
  const int row = blockIdx.x / CL;
  if (row >= n_rows) return;  // whole clusters exit together (grid = n_rows * CL)
  uint32_t Hmax = 0;
#pragma unroll
  for (int r = 0; r < CL; ++r) Hmax = max(Hmax, sd.part_start[r + 1] - sd.part_start[r]);
  double2* cs = sm_c + Hmax + 1;
  double2* fz = cs + pl.n_ops;  // [2 * n_ops]
  uint2* gse = reinterpret_cast<uint2*>(fz + 2 * pl.n_ops);  // [n_ops]
  uint8_t* opfl = reinterpret_cast<uint8_t*>(gse + pl.n_ops);  // [n_ops]: bit 0 crosses the split, bit 1 multi-pattern
  SlotMap<CL> sm;
  {
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(sm_c);
    sm.local = local;
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      if (CL == 1) {
        sm.base[r] = local;
      } else {
        uint32_t a;
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(r));
        sm.base[r] = a;
      }
    }
  }
  for (uint32_t i = threadIdx.x; i <= Hmax; i += NT) sm_c[i] = make_double2(0.0, 0.0);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    cs[op] = make_double2(cv, sv * pl.op_sscale[op]);
    const FusedDesc& d = pl.fused[pl.op_idx[op]];
    fz[2 * op] = pl.pair_f[2 * d.pair_off];
    fz[2 * op + 1] = pl.pair_f[2 * d.pair_off + 1];
    const bool realf = d.npair == 1 && pl.pair_f[2 * d.pair_off].y == 0.0 && pl.pair_f[2 * d.pair_off + 1].y == 0.0;
    opfl[op] = (uint8_t)(sd.op_cross[op] | (d.npair > 1 ? 2 : 0) | (realf ? 4 : 0));
    gse[op] = make_uint2((uint32_t)sd.gen_off[CL * op + rank], (uint32_t)sd.gen_off[CL * op + rank + 1]);
  }
  cluster.sync();
  if (threadIdx.x == 0 && (CL == 1 || (int)(sd.hf_slot >> SlotMap<CL>::kBits) == rank))
    sst<CL>(sm.addr(sd.hf_slot), make_double2(1.0, 0.0));
  cluster.sync();
  // generators: each CTA processes the pairs assigned to it (mostly local: S is
  // split on the qubits the fewest flip masks touch); one pair per thread per
  // trip; each thread's first pair word of the next two ops is in flight
  // across the barriers
  const uint32_t tid = threadIdx.x;
  auto first_word = [&](int op) -> uint32_t {
    const uint2 se = gse[op];
    return se.x + tid < se.y ? __ldg(sd.gen_pairs + se.x + tid) : 0u;
  };
  uint32_t w0 = sd.n_ops > 0 ? first_word(0) : 0u, w1 = sd.n_ops > 1 ? first_word(1) : 0u;
  for (int op = 0; op < sd.n_ops; ++op) {
    const uint32_t w = w0;
    w0 = w1;
    w1 = op + 2 < sd.n_ops ? first_word(op + 2) : 0u;
    const uint2 se = gse[op];
    const int fl = opfl[op];
    if (se.x + tid < se.y) {
      // a CTA-local step (no pair across CTAs) addresses the shared::cta window
      const double2 csv = cs[op];
      if (fl & 2) {
        gen_pass<CL, NT, true, false>(sd, pl, op, se.x + tid, se.y, w, csv, fz[2 * op], fz[2 * op + 1], sm);
      } else if (fl & 4) {  // real F (UCCSD): sin * F folded per step
        const double2 slo = make_double2(csv.y * fz[2 * op].x, 0.0), shi = make_double2(csv.y * fz[2 * op + 1].x, 0.0);
        if (CL == 1 || !(fl & 1))
          gen_pass<CL, NT, false, true, true>(sd, pl, op, se.x + tid, se.y, w, csv, slo, shi, sm);
        else
          gen_pass<CL, NT, false, false, true>(sd, pl, op, se.x + tid, se.y, w, csv, slo, shi, sm);
      } else if (CL == 1 || !(fl & 1)) {
        gen_pass<CL, NT, false, true>(sd, pl, op, se.x + tid, se.y, w, csv, fz[2 * op], fz[2 * op + 1], sm);
      } else {
        gen_pass<CL, NT, false, false>(sd, pl, op, se.x + tid, se.y, w, csv, fz[2 * op], fz[2 * op + 1], sm);
      }
    }
    // a generator whose flip mask avoids the split qubits only touches this
    // CTA's part: a CTA barrier suffices unless it or the next one crosses
    const bool cross = (fl & 1) != 0;
    // the last one also needs the cluster barrier: the expectation reads peer parts
    const bool next_cross = op + 1 >= sd.n_ops || (opfl[op + 1] & 1) != 0;
    if (CL > 1 && (cross || next_cross)) cluster.sync(); else __syncthreads();
  }
  const long long clk1 = clock64();
  // <H>: sum over (m, m ^ X) pairs of Re(conj(psi[j]) psi[i] f), section by
  // section; a chunk section first copies the peer chunk into the buffer (the
  // generator tables behind the amplitudes are dead by now). Warp w takes an
  // equal contiguous share of each section's shared and per-pair rows.
  double acc = 0.0;
  {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int sc = sd.sec_off[rank]; sc < sd.sec_off[rank + 1]; ++sc) {
      const int32_t* es = sd.secs + 7 * sc;
      const int len = es[2];
      if (CL > 1 && len > 0) {
        const uint32_t src = ((uint32_t)es[0] << SlotMap<CL>::kBits) | (uint32_t)es[1];
        __syncthreads();  // the previous chunk's readers are done
        for (int i = threadIdx.x; i < len; i += 4 * NT) {
          double2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i + u * NT < len) v[u] = sld<CL>(sm.addr(src + i + u * NT));
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i + u * NT < len) sm_c[sd.buf_off + i + u * NT] = v[u];
        }
        __syncthreads();
      }
      // sections hold whole groups of 4 rows; warps take contiguous shares of groups
      const int sh0 = es[3], shn = (es[4] - es[3]) / 4;
      const int a0 = sh0 + 4 * (int)((int64_t)shn * warp / NW), a1 = sh0 + 4 * (int)((int64_t)shn * (warp + 1) / NW);
      if (CL == 1 || sd.buf_len > 0)  // every slot is local: own part or chunk buffer
        acc += sd.f_real ? shared_rows<CL, true, true>(sd, a0, a1, lane, sm)
                         : shared_rows<CL, false, true>(sd, a0, a1, lane, sm);
      else
        acc += sd.f_real ? shared_rows<CL, true, false>(sd, a0, a1, lane, sm)
                         : shared_rows<CL, false, false>(sd, a0, a1, lane, sm);
      const int pp0 = es[4], ppn = (es[5] - es[4]) / 4;
      if (ppn > 0) {
        const int b0 = pp0 + 4 * (int)((int64_t)ppn * warp / NW), b1 = pp0 + 4 * (int)((int64_t)ppn * (warp + 1) / NW);
        acc += CL == 1 || sd.buf_len > 0 ? perpair_rows<CL, true>(sd, b0, b1, pp0 - es[6], lane, sm)
                                         : perpair_rows<CL, false>(sd, b0, b1, pp0 - es[6], lane, sm);
      }
    }
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  // fixed-order cluster reduction: every rank writes its partial into rank 0
  if (CL == 1) {
    if (threadIdx.x == 0) cl_part[0] = tot.x;
  } else if (threadIdx.x == 0) {
    *cluster.map_shared_rank(&cl_part[rank], 0) = tot.x;
  }
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) {
    double e = 0.0;
#pragma unroll
    for (int r = 0; r < CL; ++r) e += cl_part[r];
    e_out[row] = e;
    if (im_out) im_out[row] = 0.0;
    if (phase_clk) {  // diagnostics (FFQ_PHASE_CLOCKS): generator / expectation cycles
      phase_clk[2 * row] = clk1 - clk0;
      phase_clk[2 * row + 1] = clock64() - clk1;
    }
  }
}


// ---- real-amplitude evaluator ----------------------------------------------
// When every fused generator has real F (UCCSD: F = +-1), every Hamiltonian
// class sum is real and |hf> is a basis state, psi(theta) is real for every
// theta: each step is a real 2x2 rotation and the start is real. The
// imaginary parts are then identically zero, and the complex kernel's
// arithmetic on the real parts is exactly the sequence below (fma(g, b, c a)
// per member, fma(f, b a, acc) per pair), so this kernel stores the real parts
// only: 8 B per amplitude, the 18-qubit closure (15 876 amplitudes, 127 KB)
// in ONE CTA's shared memory -- no cluster, no DSMEM, CTA barriers only.
// One anchored block unit (SectorProgram::blk_*, one lane chunk) on one warp:
// lane l holds its anchor a = psi[anchor slot] and partner base B; row r adds
// (-1)^sign * f * psi[B + O_r] to the lane's partner sum t, and the unit
// contributes a * t. A shared row is one 4-B word per lane (O_r | sign << 15 |
// f index << 16, f from the parameter-space table), streamed four rows per
// trip through two register buffers (no copies of loads in flight); per-lane
// rows carry O_r plus f per lane.
// A warp's anchored-block row stream (SectorProgram::blk_stream): its units
// back to back, four rows per trip through two register buffers of prefetched
// lane words (no copies of loads in flight), so loads run ahead across unit
// boundaries. Per lane: an anchor row loads a = psi[anchor] and the partner
// base B (closing the previous unit: acc += a * t); a shared row adds
// (-1)^sign * ftab[i] * psi[B + O] to t, f by broadcast from shared memory.
// Trips without an anchor row (the common case) take the short path.
// The lane's partner sum of a unit is kept as two chains (even and odd rows of
// the stream), added when the unit closes: two FMA chains per lane, so a warp
// running alone (split evaluations) is not bound by one chain's latency.
__device__ __forceinline__ void blk_trip(const uint32_t (&d)[4], const double* amp, const double* sft, uint32_t& bs,
                                         double& a, double (&t)[2], double& acc) {
  if (((d[0] | d[1] | d[2] | d[3]) >> 30) == 0u) {
    double v[4], f[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = amp[bs + (d[u] & 0x7FFFu)];
      f[u] = sft[d[u] >> 16];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // sign bit 15 of the word -> bit 31 of f's high word
      const uint32_t hi = (uint32_t)__double2hiint(f[u]) ^ ((d[u] << 16) & 0x80000000u);
      t[u & 1] = fma(__hiloint2double((int)hi, __double2loint(f[u])), v[u], t[u & 1]);
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t w = d[u];
    if (w >> 30) {
      acc = fma(a, t[0] + t[1], acc);
      a = amp[w & 0x7FFFu];
      bs = (w >> 15) & 0x7FFFu;
      t[0] = t[1] = 0.0;
    } else {
      const double f = sft[w >> 16];
      const uint32_t hi = (uint32_t)__double2hiint(f) ^ ((w << 16) & 0x80000000u);
      t[u & 1] = fma(__hiloint2double((int)hi, __double2loint(f)), amp[bs + (w & 0x7FFFu)], t[u & 1]);
    }
  }
}

// rows [r0, r1) of a warp's stream (one segment: starts at a unit, whole prefetch rounds)
__device__ __forceinline__ double blk_rows(const SectorDev& sd, int r0, int r1, int lane, const double* amp,
                                           const double* sft) {
  const uint32_t* rw = sd.blk_stream + lane;
  auto fetch = [&](uint32_t (&d)[4], int r) {
#pragma unroll
    for (int u = 0; u < 4; ++u) d[u] = r < r1 ? __ldg(rw + (size_t)(r + u) * 32) : 0u;
  };
  uint32_t bs = 0;
  double a = 0.0, t[2] = {0.0, 0.0}, acc = 0.0;
  // kBlkTrips trips of four rows in flight; a segment is padded to whole
  // rounds of kStreamQuantum = 4 * kBlkTrips rows
  uint32_t W[kBlkTrips][4];
#pragma unroll
  for (int k = 0; k < kBlkTrips; ++k) fetch(W[k], r0 + 4 * k);
  for (int r = r0; r < r1; r += 4 * kBlkTrips) {
#pragma unroll
    for (int k = 0; k < kBlkTrips; ++k) {
      blk_trip(W[k], amp, sft, bs, a, t, acc);
      fetch(W[k], r + 4 * (k + kBlkTrips));
    }
  }
  return fma(a, t[0] + t[1], acc);
}
// segment `seg` of warp share `warp`'s block stream (blk_warp: begin, end, cut 1, cut 2)
__device__ __forceinline__ double blk_segment(const SectorDev& sd, int warp, int seg, int lane, const double* amp,
                                              const double* sft) {
  const int4 h = __ldg(sd.blk_warp + warp);
  const int b0 = seg == 0 ? h.x : seg == 1 ? h.z : h.w, b1 = seg == 0 ? h.z : seg == 1 ? h.w : h.y;
  return b0 < b1 ? blk_rows(sd, b0, b1, lane, amp, sft) : 0.0;
}
// One warp task: lane = (Xa, clique T); returns sum_ij C_ij acc_ij (a chain from 0).
__device__ __forceinline__ double clique_task(const SectorDev& sd, int wt, int lane, const double* amp) {
  const int4 d = __ldg(sd.cq_desc + (size_t)wt * 32 + lane);
  double acc[kCliquePairs];
#pragma unroll
  for (int p = 0; p < kCliquePairs; ++p) acc[p] = 0.0;
  uint32_t rn = d.z < d.w ? __ldg(sd.cq_rows + d.z) : 0u;
  for (int k = d.z; k < d.w; ++k) {
    const uint32_t rw = rn;
    if (k + 1 < d.w) rn = __ldg(sd.cq_rows + k + 1);
    const double* ra = amp + (rw & 0x7FFFu);
    const double* rb = amp + ((rw >> 15) & 0x7FFFu);
    const int sg = (int)(rw & 0x80000000u);
    // columns stay packed (bytes of d.x, d.y): extracted per row, not held
    auto col = [&](int i) { return ((uint32_t)(i < 4 ? d.x : d.y) >> (8 * (i & 3))) & 0xFFu; };
    double u[kCliqueMax];
#pragma unroll
    for (int i = 0; i < kCliqueMax; ++i) {
      const double x = ra[col(i)];
      u[i] = __hiloint2double(__double2hiint(x) ^ sg, __double2loint(x));
    }
    // v one column at a time (register budget of the 1024-thread CTA):
    // acc_ij += u_i v_j for every i != j, pair index of (min, max)
#pragma unroll
    for (int j = 0; j < kCliqueMax; ++j) {
      const double v = rb[col(j)];
#pragma unroll
      for (int i = 0; i < kCliqueMax; ++i)
        if (i != j) {
          const int a = i < j ? i : j, b = i < j ? j : i;
          const int p = a * (2 * kCliqueMax - a - 1) / 2 + (b - a - 1);
          acc[p] = fma(u[i], v, acc[p]);
        }
    }
  }
  const double* cf = sd.cq_coef + (size_t)wt * kCliquePairs * 32 + lane;
  double tot = 0.0;
#pragma unroll
  for (int p = 0; p < kCliquePairs; ++p) tot = fma(__ldg(cf + p * 32), acc[p], tot);
  return tot;
}

// RW: role warps (a split evaluation with roles >= 2); a separate instantiation so that
// the one-CTA program carries none of the role bookkeeping (64-register cap).
template <int NT, bool RW>
__global__ void __launch_bounds__(NT, NT <= 256 ? 1024 / NT : 1) k_sector_eval_real(SectorDev sd, PlanDev pl,
                                                            const double* __restrict__ theta, int theta_stride,
                                                            double* __restrict__ e_out, double* __restrict__ im_out,
                                                            int n_rows, long long* __restrict__ phase_clk,
                                                            int split, double* __restrict__ warp_sums,
                                                            double* __restrict__ state_out, int roles,
                                                            int* __restrict__ tickets) {
  // dynamic smem: [size + 1] amplitudes (the last is the zero slot) | [n_ops]
  // (cos, sin) | [n_ops] (sin F_lo, sin F_hi) | [n_ops] pair range
  // split > 1 (small batches): `split` CTAs run one evaluation; each runs the
  // generator phase, then the warp shares w = part (mod split) of the
  // expectation, whose warp sums go to warp_sums[row][w]; k_sum_warps then
  // adds them with block_sum's second-stage tree, so the energy bits equal
  // the one-CTA kernel's.
  extern __shared__ __align__(16) unsigned char sm_raw[];
  __shared__ double2 red[NT / 32];
  // phase clocks (diagnostics) live in shared memory, not in registers of every thread
  __shared__ long long clk_s[2];
  if (threadIdx.x == 0) clk_s[0] = clock64();
  const int row = blockIdx.x / split, part = blockIdx.x % split;
  if (row >= n_rows) {
    // CTAs past the batch (role-warp launches on otherwise idle SMs): pull the table
    // ranges into L2 while the evaluations' CTAs start (k_l2_warm inside the launch)
    if constexpr (RW) {
      const uint64_t nw = gridDim.x - (uint64_t)n_rows * split, wi = blockIdx.x - (uint64_t)n_rows * split;
      for (int r = 0; r < sd.n_warm; ++r) {
        const ulonglong2 rg = __ldg(sd.warm + r);
        for (uint64_t off = (wi * NT + threadIdx.x) * 128; off < rg.y; off += nw * NT * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rg.x + off));
      }
    }
    return;
  }
  const uint32_t na = sd.n_slots + 1;
  double* amp = reinterpret_cast<double*>(sm_raw);
  // per-op record (32 B): cos phi, sin phi F_lo, sin phi F_hi, pair range in gen_pairs
  struct __align__(16) OpRec {
    double c, gh, gl;
    uint32_t s0, s1;
  };
  OpRec* opt = reinterpret_cast<OpRec*>(sm_raw + ((na * sizeof(double) + 15) & ~(size_t)15));
  double2* cs = reinterpret_cast<double2*>(opt);  // the records' bytes, reused after the generator phase
  double* sft = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(opt) +
                                          (size_t)pl.n_ops * (2 * sizeof(double2) + sizeof(uint2)));  // shared-row f table
  for (uint32_t i = threadIdx.x; i < na; i += NT) amp[i] = 0.0;
  if (sd.blk_warp)
    for (int i = threadIdx.x; i < sd.n_ftab; i += NT) sft[i] = __ldg(sd.ftab + i);
  for (int op = threadIdx.x; op < pl.n_ops; op += NT) {
    const double phi = theta[(int64_t)row * theta_stride + pl.op_gen[op]] * pl.op_cfac[op];
    double sv, cv;
    sincos(phi, &sv, &cv);
    const double sn = sv * pl.op_sscale[op];
    const FusedDesc& d = pl.fused[pl.op_idx[op]];
    OpRec r;
    r.c = cv;
    r.gl = sn * pl.pair_f[2 * d.pair_off].x;
    r.gh = sn * pl.pair_f[2 * d.pair_off + 1].x;
    r.s0 = (uint32_t)sd.gen_off[op];
    r.s1 = (uint32_t)sd.gen_off[op + 1];
    opt[op] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) amp[sd.hf_slot] = 1.0;
  __syncthreads();
  const uint32_t tid = threadIdx.x;
  // each thread's first two pair words of the next D steps are in flight
  // across the barriers (steps have up to ~2 NT pairs), read from the head
  // table at a fixed per-thread stride (no range lookup; 0xFFFFFFFF = none;
  // the table ends with empty ops, so the prefetch needs no bound). The step
  // loop is unrolled by D so the in-flight registers are never copied (a copy
  // would wait for the load).
  const uint32_t* hp = sd.gen_head + tid;
  auto first_words = [&](int op) -> uint2 {
    const uint32_t* p = hp + (size_t)op * (2 * NT);
    return make_uint2(__ldg(p), __ldg(p + NT));
  };
  auto step = [&](int op, uint2 ww) {
    if (ww.x != 0xFFFFFFFFu) {
      // (c, gh) in one 16-byte load; gl = -gh exactly (rotation block), a free operand negation
      const double2 cg = *reinterpret_cast<const double2*>(&opt[op].c);
      const double c = cg.x, gh = cg.y, gl = -cg.y;
      // one pair, slot_i | slot_j << 16 (a negative sign is a swap of the members, done by the compiler)
      auto rot = [&](uint32_t w) {
        const uint32_t i = w & 0x7FFFu, j = w >> 16;
        const double a = amp[i], b = amp[j];
        amp[i] = fma(gh, b, c * a);
        amp[j] = fma(gl, a, c * b);
      };
      rot(ww.x);
      if (ww.y != 0xFFFFFFFFu) {
        rot(ww.y);
        if (ww.y & (1u << 15)) {  // long steps (single excitations): the rest from gen_pairs
          const uint32_t s1 = opt[op].s1;
          // (the compiler unrolls this loop and issues its word loads together)
          for (uint32_t t = opt[op].s0 + tid + 2 * NT; t < s1; t += NT) rot(__ldg(sd.gen_pairs + t));
        }
      }
    }
    __syncthreads();
  };
  // D steps of pair words in flight (registers; the loop is unrolled by D so
  // a prefetched word is never copied while its load is outstanding)
  constexpr int D = 6;  // 4: 477k, 6: 465k, 8: 471k generator cycles per evaluation (config 3)
  uint2 w[D];
#pragma unroll
  for (int k = 0; k < D; ++k) w[k] = first_words(k);
  int op = 0;
  for (; op + D <= sd.n_ops; op += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      step(op + k, w[k]);
      w[k] = first_words(op + k + D);
    }
  }
#pragma unroll
  for (int k = 0; k < D - 1; ++k)
    if (op + k < sd.n_ops) step(op + k, w[k]);
  if (threadIdx.x == 0) clk_s[1] = clock64();
  if (state_out && part == 0)  // ffq_sector_state: the slots after the plan (natural gauge)
    for (uint32_t i = threadIdx.x; i < sd.n_slots; i += NT) state_out[(int64_t)row * sd.n_slots + i] = amp[i];
  if (sd.eps_flip) {  // the expectation tables are in the alpha-first gauge (compile_sector)
    for (uint32_t i = threadIdx.x; i < sd.n_slots; i += NT)
      if ((__ldg(sd.eps_flip + (i >> 5)) >> (i & 31u)) & 1u) amp[i] = -amp[i];
    __syncthreads();
  }
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31;
  // warp share `warp`: its generic rows (shared-f rows, then per-pair-f rows), one chain
  auto generic_rows = [&](int warp) -> double {
    double acc = 0.0;
    const int32_t* es = sd.secs;  // one section: every pair is local
    const int sh0 = es[3], shn = (es[4] - es[3]) / 4;
    const int r0 = sh0 + 4 * (int)((int64_t)shn * warp / NW), r1 = sh0 + 4 * (int)((int64_t)shn * (warp + 1) / NW);
    if (r0 < r1) {
      uint32_t wn[4];
      double fn[4];
      auto fetch = [&](int rw) {
        const uint32_t* p = sd.row_pairs + (size_t)rw * 32 + lane;
#pragma unroll
        for (int u = 0; u < 4; ++u) wn[u] = __ldg(p + 32 * u);
        // rw is a multiple of 4: the four f of a trip are two aligned 16-B loads
        const double2 f01 = __ldg(reinterpret_cast<const double2*>(sd.row_fre + rw));
        const double2 f23 = __ldg(reinterpret_cast<const double2*>(sd.row_fre + rw) + 1);
        fn[0] = f01.x;
        fn[1] = f01.y;
        fn[2] = f23.x;
        fn[3] = f23.y;
      };
      fetch(r0);
      for (int rw = r0; rw < r1; rw += 4) {
        uint32_t w[4];
        double f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w[u] = wn[u];
          f[u] = fn[u];
        }
        if (rw + 4 < r1) fetch(rw + 4);
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = amp[w[u] & 0x7FFFu];
          b[u] = amp[(w[u] >> 15) & 0x7FFFu];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long sgn = (long long)((w[u] >> 30) & 1u) << 63;
          const double fs = __longlong_as_double(__double_as_longlong(f[u]) ^ sgn);
          acc = fma(fs, b[u] * a[u], acc);
        }
      }
    }
    const int pp0 = es[4], ppn = (es[5] - es[4]) / 4;
    const int q0 = pp0 + 4 * (int)((int64_t)ppn * warp / NW), q1 = pp0 + 4 * (int)((int64_t)ppn * (warp + 1) / NW);
    for (int rw = q0; rw < q1; rw += 4) {
      const uint32_t* p = sd.row_pairs + (size_t)rw * 32 + lane;
      const int64_t fo = (int64_t)(rw - pp0 + es[6]) * 32 + lane;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t w = __ldg(p + 32 * u);
        const double fr = __ldg(sd.pf_re + fo + 32 * u);
        acc = fma(amp[(w >> 15) & 0x7FFFu] * amp[w & 0x7FFFu], fr, acc);
      }
    }
    return acc;
  };
  // One warp share ws of the expectation = its generic rows + the three segment sums
  // of its anchored block stream (added in order from zero) + its clique task
  // totals (added in task order from zero). A CTA running a whole evaluation, or
  // a split evaluation without role warps, has physical warp ws compute all of
  // share ws. With role warps (split > 1, roles = split >= 2) this CTA serves the
  // shares ws = part + split * si and share si gets `roles` physical warps: role 0
  // takes the generic rows; the block segments go to roles 1, 2, 3 (eight roles),
  // to roles 0, 1, 1 (three to seven roles) or all to role 0 (two roles); the
  // remaining roles take the clique tasks round robin. The pieces travel
  // through an exchange buffer that overlays the per-op records (dead after the
  // generator phase) and role 0 adds them in the order above, so the energy
  // bits do not depend on split or roles.
  constexpr bool role_mode = RW;  // (the host passes split > 1 and roles >= 2 with RW)
  const int pw = threadIdx.x >> 5;
  const int nr = role_mode ? roles : 1, si = pw / nr, role = pw - si * nr;
  const int ws = role_mode ? part + split * si : pw;
  if (!role_mode && split > 1 && pw % split != part) return;
  const int nseg = nr >= 3 ? kBlkSegments : 0;  // exchanged segment sums
  const int cq0 = nr >= 8 ? 1 + kBlkSegments : nr >= 3 ? 2 : nr - 1, ncq = nr - cq0;
  double* xs = reinterpret_cast<double*>(cs) + (size_t)si * (nseg + sd.max_warp_tasks) * 32 + lane;
  double* xt = xs + nseg * 32;
  double acc = role == 0 ? generic_rows(ws) : 0.0;
  if (sd.blk_warp) {
    double tot = 0.0;
#pragma unroll 1
    for (int seg = 0; seg < kBlkSegments; ++seg) {
      if (role != (nr >= 8 ? 1 + seg : nr >= 3 && seg > 0 ? 1 : 0)) continue;
      const double v = blk_segment(sd, ws, seg, lane, amp, sft);
      if (nseg)
        xs[seg * 32] = v;
      else
        tot += v;
    }
    if (!nseg) acc += tot;  // (role 0; other roles' acc is not used)
  }
  const int2 wr = sd.cq_warp ? __ldg(sd.cq_warp + ws) : make_int2(0, 0);
  if (role >= cq0) {
    double tot = 0.0;
#pragma unroll 1
    for (int wt = wr.x + role - cq0; wt < wr.y; wt += ncq) {
      const double v = clique_task(sd, wt, lane, amp);
      if (nr > 1)
        xt[(wt - wr.x) * 32] = v;
      else
        tot += v;
    }
    if (nr == 1) acc += tot;
  }
  if constexpr (RW) {
    __shared__ int last_cta;
    // diagnostics: cycles of every role's piece (CTA 0 of row 0) behind the per-row pairs
    if (phase_clk && blockIdx.x == 0 && lane == 0) phase_clk[2 * n_rows + pw] = clock64() - clk_s[1];
    __syncthreads();
    if (role == 0) {
      if (sd.blk_warp && nseg) {
        double tot = 0.0;
        for (int seg = 0; seg < kBlkSegments; ++seg) tot += xs[seg * 32];
        acc += tot;
      }
      double tot = 0.0;
      for (int k = 0; k < wr.y - wr.x; ++k) tot += xt[k * 32];
      if (sd.cq_warp) acc += tot;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);  // block_sum's first stage
      if (lane == 0) {
        warp_sums[(int64_t)row * NW + ws] = acc;
        __threadfence();
      }
    }
    // The evaluation's last CTA to arrive adds the 32 warp sums with block_sum's
    // second-stage tree (what k_sum_warps does after a launch without role warps)
    // and clears the ticket for the next launch.
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last_cta = atomicAdd(tickets + row, 1) == split - 1;
    }
    __syncthreads();
    if (last_cta && pw == 0) {
      __threadfence();
      double v = __ldcg(warp_sums + (int64_t)row * NW + lane);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) {
        e_out[row] = v;
        if (im_out) im_out[row] = 0.0;
        tickets[row] = 0;
      }
    }
    if (threadIdx.x == 0 && phase_clk) {
      phase_clk[2 * row] = clk_s[1] - clk_s[0];
      phase_clk[2 * row + 1] = clock64() - clk_s[1];
    }
    return;
  }
  // diagnostics: per-warp expectation cycles of row 0 behind the per-row pairs
  if (phase_clk && split == 1 && row == 0 && lane == 0) phase_clk[2 * n_rows + pw] = clock64() - clk_s[1];
  if (split > 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);  // block_sum's first stage
    if (lane == 0) warp_sums[(int64_t)row * (NT / 32) + ws] = acc;
    if (threadIdx.x == 0 && phase_clk) {
      phase_clk[2 * row] = clk_s[1] - clk_s[0];
      phase_clk[2 * row + 1] = clock64() - clk_s[1];
    }
    return;
  }
  const double2 tot = block_sum<NT>(make_double2(acc, 0.0), red);
  if (threadIdx.x == 0) {
    e_out[row] = tot.x;
    if (im_out) im_out[row] = 0.0;
    if (phase_clk) {
      phase_clk[2 * row] = clk_s[1] - clk_s[0];
      phase_clk[2 * row + 1] = clock64() - clk_s[1];
    }
  }
}

// One warp per evaluation: block_sum's second stage over the 32 warp sums
// of a split k_sector_eval_real launch.
__global__ void k_sum_warps(const double* __restrict__ warp_sums, double* __restrict__ e_out,
                            double* __restrict__ im_out) {
  double v = warp_sums[(int64_t)blockIdx.x * 32 + threadIdx.x];
  double z = 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_down_sync(0xffffffffu, v, o);
    z += __shfl_down_sync(0xffffffffu, z, o);
  }
  if (threadIdx.x == 0) {
    e_out[blockIdx.x] = v;
    if (im_out) im_out[blockIdx.x] = z;
  }
}

}  // namespace ffq

namespace ffq {

// ---- sparse row-wise matvec on a Krylov basis (lanczos_ground, energy_exact) ----
// y[r] = sum_e val[e] * (gen ? theta[gen[e]] : 1) * x[col[e]]; one warp per row,
// lanes stride the row, fixed shuffle tree (deterministic).
__global__ void k_csr_matvec(int64_t rows, const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                             const double* __restrict__ vre, const double* __restrict__ vim,
                             const int32_t* __restrict__ gen, const double* __restrict__ theta,
                             const double2* __restrict__ x, double2* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t e = rp[r] + lane; e < rp[r + 1]; e += 32) {
      double ar = vre[e], ai = vim[e];
      if (gen) {
        const double t = theta[gen[e]];
        ar *= t;
        ai *= t;
      }
      const double2 v = x[col[e]];
      acc.x = fma(ar, v.x, fma(-ai, v.y, acc.x));
      acc.y = fma(ar, v.y, fma(ai, v.x, acc.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) y[r] = acc;
  }
}

}  // namespace ffq
