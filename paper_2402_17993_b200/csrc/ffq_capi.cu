// ffq_capi.cu -- C-ABI of libfragfield_cuda.so (include/fragfield_cuda.h).
//
// Host orchestration of the sm_100a kernels in ffq_kernels.cuh: contexts own a
// device + stream, plans/Hamiltonians own their compiled device tables, and
// batched energy evaluation picks one of two execution paths:
//   * n <= kSmemMaxQubits: k_smem_eval, one CTA per evaluation;
//   * otherwise: a CUDA graph of per-op kernels over a [chunk][2^n] slab
//     (HF build -> fused/string passes -> grouped expectation -> fixed-tree
//     reduction), replayed for every chunk of the batch.
// There is no CPU fallback: without a device every call fails with
// FFQ_ENODEV / FFQ_ECUDA.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fragfield_cuda.h"
#include "ffq_compile.hpp"
#include "ffq_kernels.cuh"
#include "ffq_sparse.cuh"
#include "ffq_sector.cuh"

using namespace ffq;

namespace {

constexpr int kSmemMaxQubitsDefault = 13;
constexpr int kThreads = 256;
constexpr int kVersion = 1;

thread_local std::string g_thread_err = "no error";

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));               \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    n = count;
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// Runs of >= 2 consecutive eligible rotations whose flip masks, together with
// the low 5 qubits, lie in a set Q of t qubits (the run's tile: Q = the union
// filled up with the lowest free qubits; Q = the low t qubits is the TMA case),
// each cut into groups of consecutive rotations whose flip masks span <= 3
// dimensions (k_rotation_run). rd gets the masks in tile coordinates (pext by
// Q) and the group coordinates; group ranges are relative to the run.
struct RotRuns {
  std::vector<int> run_at;  // per rotation: index of the run starting there, else -1
  std::vector<int> len, g0, ng;
  std::vector<uint64_t> q;  // per run: its qubit set
  std::vector<RotGroup> groups;
};

inline uint64_t pext64(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (int o = 0; mask; mask &= mask - 1, ++o)
    if (v & mask & (~mask + 1)) r |= 1ULL << o;
  return r;
}

// x, z: original strings; rd[r].ny must be set by the caller
RotRuns build_rot_runs(std::vector<RotDesc>& rd, const uint64_t* x, const uint64_t* z,
                       const std::vector<char>& ok, int n, int t) {
  RotRuns R;
  const int N = (int)rd.size();
  R.run_at.assign(N, -1);
  if (t < 3 || t > 12 || n < t) return R;
  const uint64_t low = (1ULL << std::min(5, t)) - 1ULL;
  for (int i = 0; i < N;) {
    uint64_t U = low;
    int e = i;
    while (e < N && ok[e] && __builtin_popcountll(U | x[e]) <= t) U |= x[e++];
    if (e - i < 2) { i = std::max(i + 1, e); continue; }
    uint64_t Q = U;
    for (int bit = 0; __builtin_popcountll(Q) < t; ++bit) Q |= 1ULL << bit;
    R.run_at[i] = (int)R.len.size();
    R.len.push_back(e - i);
    R.q.push_back(Q);
    R.g0.push_back((int)R.groups.size());
    for (int r = i; r < e; ++r) {
      rd[r].x = pext64(x[r], Q);
      rd[r].z = pext64(z[r], Q);
      rd[r].zo = z[r] & ~Q;
    }
    for (int r = i; r < e;) {
      uint32_t b[3];
      int piv[3], d = 0, qq = r;
      for (; qq < e; ++qq) {
        uint32_t v = (uint32_t)rd[qq].x;
        for (int j = 0; j < d; ++j)
          if ((v >> piv[j]) & 1u) v ^= b[j];
        if (!v) continue;  // in the span: joins the group
        if (d == 3) break;
        const int p = 31 - __builtin_clz(v);
        for (int j = 0; j < d; ++j)
          if ((b[j] >> p) & 1u) b[j] ^= v;
        b[d] = v;
        piv[d++] = p;
      }
      for (int bit = t - 1; d < 3; --bit) {  // pad with unit vectors at the highest free bits
        bool used = false;
        for (int j = 0; j < d; ++j) used |= piv[j] == bit;
        if (used) continue;
        for (int j = 0; j < d; ++j)
          if ((b[j] >> bit) & 1u) b[j] ^= 1u << bit;
        b[d] = 1u << bit;
        piv[d++] = bit;
      }
      RotGroup G;
      int ord[3] = {0, 1, 2};
      std::sort(ord, ord + 3, [&](int a2, int b2) { return piv[a2] < piv[b2]; });
      for (int j = 0; j < 3; ++j) {
        G.b[j] = b[ord[j]];
        G.piv[j] = piv[ord[j]];
      }
      G.r0 = r - i;
      G.r1 = qq - i;
      for (int j = r; j < qq; ++j) {
        int cx = 0;
        for (int k = 0; k < 3; ++k)
          if ((rd[j].x >> G.piv[k]) & 1u) cx |= 1 << k;
        rd[j].cx = cx;
      }
      R.groups.push_back(G);
      r = qq;
    }
    R.ng.push_back((int)R.groups.size() - R.g0.back());
    i = e;
  }
  return R;
}

}  // namespace

struct ffq_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int n_sm = 148;
  size_t smem_optin = 0;
  int smem_max_qubits = kSmemMaxQubitsDefault;  // env FFQ_SMEM_MAX_QUBITS overrides
  int64_t slab_bytes = 256LL << 20;              // env FFQ_SLAB_MB: batch chunk of the graph path
  int support = 1;                               // env FFQ_SUPPORT=0: dense passes only
  int sector = 1;                                // env FFQ_SECTOR=0: no support-closure cluster evaluator
  int sector_cl = 2;                             // env FFQ_SECTOR_CL: 2, 4 or 8 CTAs per large closure
  int sector_real = 1;                           // env FFQ_SECTOR_REAL=0: no real-amplitude sector kernel
  int sector_blocks = 1;                         // env FFQ_BLOCKS=0: no anchored string blocks (product layout)
  int sector_cliques = 1;                        // env FFQ_CLIQUES=0: alpha-beta pairs in the blocks, not the cliques
  int sector_split = 16;                         // env FFQ_SPLIT: most CTAs per evaluation of the 1024-thread real program
  std::string err = "no error";
  int64_t launches = 0;
  // scratch
  DevBuf<double> theta, eout, eim, io_theta, io_e;
  DevBuf<double2> cs, partial, slab;
  DevBuf<double> compact_psi, compact_coef, compact_part, compact_io;  // compact real sector path (ffq_compact.inl)
  int compact_graph = 1;                     // env FFQ_COMPACT_GRAPH=0: small compact matrices launch by launch
  int compact_il = 8;                        // env FFQ_COMPACT_IL: most theta rows interleaved per matrix (1, 2, 4, 8)
  int sector_roles = 1;                      // env FFQ_ROLES=0: split evaluations without role warps
  int sector_warm = 1;                       // env FFQ_WARM=0: no L2 warm-up pass before small sector batches
  int compact = 1;                           // env FFQ_COMPACT=0: no compact sector path
  int compact_min_qubits = 24;               // env FFQ_COMPACT_MIN: smallest n it takes at any batch
                                             // (batches >= 8 from two qubits lower): measured
                                             // crossover against the dense support path
  DevBuf<double> warp_sums;  // split k_sector_eval_real: [batch][32] warp sums
  DevBuf<int> row_tickets;   // role-warp launches: CTAs of a row that have written their warp sums (zero between launches)
  DevBuf<RotDesc> rot;       // ffq_state_apply_pauli_rotations: fused low-qubit runs
  DevBuf<RotGroup> rot_groups;
  int rot_tile_bits = 12;    // env FFQ_ROT_TILE: tile of a fused run (0: one pass per rotation)
  DevBuf<uint32_t> slab_sup;
  bool slab_clean = false;      // support path: slab all-zero between graph replays
  double* pinned = nullptr;
  size_t pinned_n = 0;
  // ffq_energy_batch: chunk H2D copies on their own stream, so a copy overlaps
  // the previous chunk's kernels instead of sitting between them
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_done;
  cudaEvent_t copy_event(size_t k) {
    if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    while (copy_done.size() <= k) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      copy_done.push_back(e);
    }
    return copy_done[k];
  }
  void ensure_pinned(size_t n) {
    if (n <= pinned_n) return;
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    CK(cudaMallocHost(&pinned, n * sizeof(double)));
    pinned_n = n;
  }
};

// a captured graph bakes in every scratch pointer, so all of them are key parts
using GraphKey = std::vector<uintptr_t>;

struct ffq_plan_s {
  ffq_ctx_t ctx;
  CompiledPlan cp;
  DevBuf<int32_t> op_kind, op_gen, op_idx, str_ny;
  DevBuf<double> op_cfac, op_sscale;
  DevBuf<FusedDesc> fused;
  DevBuf<uint64_t> pair_bits, str_x, str_z;
  DevBuf<uint32_t> pair_low;
  DevBuf<double2> pair_f;
  DevBuf<RotDesc> rot;  // per op: the string's (x, z, ny, coset coordinate) for fused runs of string ops
  RotRuns runs;         // runs of string ops with low flip masks (context's FFQ_ROT_TILE)
  int runs_t = 0;
  DevBuf<RotGroup> rot_groups;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int64_t> graph_nodes;
  struct SectorDevBufs {
    SectorProgram prog;
    DevBuf<int64_t> gen_off;
    DevBuf<uint32_t> gen_pairs, gen_head, row_pairs;
    DevBuf<int32_t> secs;
    DevBuf<uint8_t> gen_flags, op_cross;
    DevBuf<double> row_fre, row_fim, pf_re, pf_im;
    DevBuf<int32_t> blk_warp;
    DevBuf<uint32_t> blk_stream;
    DevBuf<double> ftab;
    DevBuf<uint32_t> eps_flip, cq_rows;
    DevBuf<int32_t> cq_desc, cq_warp;
    DevBuf<double> cq_coef;
    DevBuf<ulonglong2> warm;  // (address, bytes) of every table (k_l2_warm)
    int n_warm = 0;
    bool real = false;  // real-amplitude program (k_sector_eval_real)
  };
  std::map<std::pair<uint64_t, uint64_t>, std::unique_ptr<SectorDevBufs>> sectors;  // (ham uid, hf)
  std::map<std::string, std::shared_ptr<void>> compacts;  // CompactProg per (ham, hf) (ffq_compact.inl)
  PlanDev dev() const {
    PlanDev d;
    d.n_ops = (int)cp.op_kind.size();
    d.op_kind = op_kind.p; d.op_gen = op_gen.p; d.op_idx = op_idx.p;
    d.op_cfac = op_cfac.p; d.op_sscale = op_sscale.p;
    d.fused = fused.p; d.pair_bits = pair_bits.p; d.pair_f = pair_f.p;
    d.str_x = str_x.p; d.str_z = str_z.p; d.str_ny = str_ny.p;
    return d;
  }
  ~ffq_plan_s() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  }
};

// process-unique id per uploaded Hamiltonian: the compiled-program caches key on
// it, never on the handle's address (a destroyed handle's address can be reused)
static std::atomic<uint64_t> g_ham_uid{1};

struct ffq_ham_s {
  ffq_ctx_t ctx;
  uint64_t uid = g_ham_uid.fetch_add(1);
  CompiledHam ch;
  std::vector<uint64_t> raw_x, raw_z;  // the uploaded terms (sharded path recompiles them)
  std::vector<double> raw_re, raw_im;
  DevBuf<GroupDesc> groups;
  DevBuf<uint64_t> act_bits, cls_z;
  DevBuf<double2> cls_f;
  DevBuf<int32_t> item_g, item_p;
  DevBuf<int64_t> item_u0;
  DevBuf<uint32_t> act_low;
  DevBuf<int32_t> sitem_g, sitem_p;
  DevBuf<int64_t> sitem_w0;
  int64_t n_partials(bool support) const {
    if (support) return (int64_t)ch.sitem_g.size();
    return (int64_t)ch.item_g.size();
  }
  HamDev dev() const {
    HamDev d;
    d.n_groups = (int)ch.groups.size();
    d.groups = groups.p; d.act_bits = act_bits.p; d.cls_z = cls_z.p; d.cls_f = cls_f.p;
    d.n_items = (int64_t)ch.item_g.size();
    d.item_g = item_g.p; d.item_p = item_p.p; d.item_u0 = item_u0.p;
    d.item_chunk = ch.item_chunk;
    d.sitem_words = ch.sitem_words;
    return d;
  }
};

struct ffq_state_s {
  ffq_ctx_t ctx;
  int n = 0, batch = 0;
  DevBuf<double2> psi;
  DevBuf<uint32_t> sup;   // support bitmap [batch][2^(n-5)] (support mode only)
  bool sup_valid = false; // false after a dense pass: rebuilt lazily from the data
};

namespace {

int fail(ffq_ctx_t ctx, int code, const std::string& msg) {
  g_thread_err = msg;
  if (ctx) ctx->err = msg;
  return code;
}

template <typename F>
int guarded(ffq_ctx_t ctx, F&& f) {
  try {
    if (ctx) CK(cudaSetDevice(ctx->device));
    return f();
  } catch (const BadInput& e) {
    return fail(ctx, e.code, e.what());
  } catch (const CudaError& e) {
    std::string w = e.what();
    bool oom = w.find("out of memory") != std::string::npos;
    return fail(ctx, oom ? FFQ_ENOMEM : FFQ_ECUDA, w);
  } catch (const std::bad_alloc&) {
    return fail(ctx, FFQ_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, FFQ_EINVAL, e.what());
  }
}

int grid_for(int64_t work, int n_sm, int per_sm = 8) {
  int64_t g = (work + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)n_sm * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}


bool use_support(ffq_ctx_t ctx, int n) { return ctx->support && n >= 6 && n <= 32; }

void launch_support_from_state(ffq_ctx_t ctx, const double2* psi, uint32_t* sup, int n, int batch) {
  const int64_t total = (int64_t)batch << n;
  k_support_from_state<<<grid_for(total, ctx->n_sm), kThreads, 0, ctx->stream>>>(psi, sup, total);
  CK(cudaGetLastError());
  ctx->launches++;
}

// rotation-pass dispatch for a single string (state API and plan string ops)
void launch_string(ffq_ctx_t ctx, double2* psi, int n, int batch, uint64_t x, uint64_t z, int ny,
                   const double2* cs, int cs_stride, int op) {
  int mode, hbit = 0;
  int64_t nvec;
  if (n < 2) throw BadInput("rotation kernels need n_qubits >= 2", FFQ_EINVAL);
  if (x == 0) { mode = 0; nvec = 1LL << (n - 1); }
  else if (!(x & 1ULL)) { mode = 1; hbit = __builtin_ctzll(x); nvec = 1LL << (n - 2); }
  else if (x == 1ULL) { mode = 2; nvec = 1LL << (n - 1); }
  else { mode = 3; hbit = __builtin_ctzll(x & ~1ULL); nvec = 1LL << (n - 2); }
  dim3 grid(grid_for(nvec, ctx->n_sm), batch);
  k_pauli_rotation<<<grid, kThreads, 0, ctx->stream>>>(psi, n, x, z, ny, cs, cs_stride, op, mode,
                                                        hbit);
  CK(cudaGetLastError());
  ctx->launches++;
}

// a run of rotations with flip masks below 2^t: one TMA-staged tile per CTA
// (the 64 KiB dynamic-smem and carveout attributes are set at context creation,
// so the launch can sit inside a captured graph)
constexpr int kRotRunThreads = 256;  // 3 CTAs (64 KiB tiles) per SM
void launch_rotation_run(ffq_ctx_t ctx, double2* psi, int n, int batch, int t, uint64_t q, const RotGroup* g,
                         int n_grp, const RotDesc* rd, const double2* cs, int cs_stride) {
  const size_t sb = sizeof(double2) << t;
  dim3 grid((unsigned)(1u << (n - t)), batch);
  k_rotation_run<kRotRunThreads><<<grid, kRotRunThreads, sb, ctx->stream>>>(psi, n, t, q, g, n_grp, rd, cs,
                                                                           cs_stride);
  CK(cudaGetLastError());
  ctx->launches++;
}

void launch_fused(ffq_ctx_t ctx, const ffq_plan_s* pl, double2* psi, uint32_t* sup, int n, int batch,
                  const FusedDesc& d, const double2* cs, int cs_stride, int op, int64_t rstride) {
  if (sup) {
    const int64_t work = (int64_t)d.npair << (n - 5 - d.whi);
    dim3 grid(grid_for(work, ctx->n_sm), batch);
    k_fused_gen_support<<<grid, kThreads, 0, ctx->stream>>>(psi, sup, n, d, pl->pair_bits.p, pl->pair_low.p,
                                                            pl->pair_f.p, cs, cs_stride, op, rstride);
    CK(cudaGetLastError());
    ctx->launches++;
    return;
  }
  const bool vec = !(d.x & 1ULL) && (n - d.w) >= 1;
  const int64_t work = ((int64_t)d.npair << (n - d.w)) >> (vec ? 1 : 0);
  dim3 grid(grid_for(work, ctx->n_sm), batch);
  if (vec)
    k_fused_gen<true><<<grid, kThreads, 0, ctx->stream>>>(psi, n, d, pl->pair_bits.p, pl->pair_f.p,
                                                          cs, cs_stride, op, 0);
  else
    k_fused_gen<false><<<grid, kThreads, 0, ctx->stream>>>(psi, n, d, pl->pair_bits.p,
                                                           pl->pair_f.p, cs, cs_stride, op, 0);
  CK(cudaGetLastError());
  ctx->launches++;
}

// apply every op of the plan to a [batch][2^n] slab; cs already computed
// sup != nullptr: support-tracked fused passes; string ops are dense and are
// followed by an exact support rebuild before the next support-tracked op
void run_plan_ops(ffq_ctx_t ctx, const ffq_plan_s* pl, double2* psi, uint32_t* sup, int batch,
                  const double2* cs, int64_t rstride = 0) {
  const CompiledPlan& cp = pl->cp;
  const int n = cp.n_qubits;
  const int n_ops = (int)cp.op_kind.size();
  bool stale = false;
  for (int op = 0; op < n_ops; ++op) {
    if (cp.op_kind[op] == 0) {
      if (sup && stale) {
        launch_support_from_state(ctx, psi, sup, n, batch);
        stale = false;
      }
      launch_fused(ctx, pl, psi, sup, n, batch, cp.fused[cp.op_idx[op]], cs, n_ops, op,
                   rstride ? rstride : (1LL << n));
    } else {
      // a run of >= 2 string ops with flip masks below 2^t: one tiled pass
      const int ri = pl->runs.run_at[op];
      if (ri >= 0) {
        launch_rotation_run(ctx, psi, n, batch, pl->runs_t, pl->runs.q[ri], pl->rot_groups.p + pl->runs.g0[ri],
                            pl->runs.ng[ri], pl->rot.p + op, cs + op, n_ops);
        op += pl->runs.len[ri] - 1;
      } else {
        const int si = cp.op_idx[op];
        launch_string(ctx, psi, n, batch, cp.str_x[si], cp.str_z[si], cp.str_ny[si], cs, n_ops, op);
      }
      stale = true;
    }
  }
  if (sup && stale) launch_support_from_state(ctx, psi, sup, n, batch);
}

void launch_cs(ffq_ctx_t ctx, const ffq_plan_s* pl, const double* theta, int batch, double2* cs) {
  const int n_ops = (int)pl->cp.op_kind.size();
  if (n_ops == 0) return;
  const int64_t work = (int64_t)n_ops * batch;
  k_op_cs<<<grid_for(work, ctx->n_sm), kThreads, 0, ctx->stream>>>(
      theta, pl->cp.n_gen, n_ops, pl->op_gen.p, pl->op_cfac.p, pl->op_sscale.p, cs, batch);
  CK(cudaGetLastError());
  ctx->launches++;
}

void launch_expect(ffq_ctx_t ctx, const ffq_ham_s* h, const double2* psi, const uint32_t* sup, int n,
                   int batch, double2* partial, double* e, double* im, int64_t rstride = 0) {
  const int64_t items = h->n_partials(sup != nullptr);
  if (items == 0) {
    CK(cudaMemsetAsync(e, 0, sizeof(double) * batch, ctx->stream));
    if (im) CK(cudaMemsetAsync(im, 0, sizeof(double) * batch, ctx->stream));
    return;
  }
  if (sup) {
    k_expect_support<kThreads><<<dim3((unsigned)items, batch), kThreads, 0, ctx->stream>>>(
        psi, sup, n, h->dev(), h->sitem_g.p, h->sitem_p.p, h->sitem_w0.p, h->act_low.p, partial,
        rstride ? rstride : (1LL << n));
    CK(cudaGetLastError());
    ctx->launches++;
  } else {
    dim3 grid((unsigned)items, batch);
    k_expect_items<kThreads><<<grid, kThreads, 0, ctx->stream>>>(psi, n, h->dev(), partial);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  k_reduce_partials<kThreads><<<batch, kThreads, 0, ctx->stream>>>(partial, items, e, im);
  CK(cudaGetLastError());
  ctx->launches++;
}

size_t smem_bytes(const ffq_plan_s* pl) {
  return ((size_t(1) << pl->cp.n_qubits) + pl->cp.op_kind.size()) * sizeof(double2);
}

constexpr int kSectorThreads = 768;       // per CTA of a 2/4/8-CTA cluster (measured best at 18 qubits)
constexpr int kSectorSingleThreads = 128;  // one-CTA evaluations (small closures, many CTAs per SM)
constexpr int kSectorRealThreads = 1024;   // one-CTA real-amplitude evaluations of large closures
// small closures run one CTA per evaluation (many per SM); large ones a 2^s-CTA cluster
constexpr uint32_t kSectorSingleMax = 2048;  // <= 32 KiB of amplitudes per CTA
static_assert(kSectorHeadSmall == kSectorSingleThreads && kSectorHeadLarge == kSectorRealThreads,
              "gen_head is compiled for the real program's thread counts");
constexpr uint32_t kSectorMaxSize = 32767;   // 15-bit pair indices

// cluster size for a closure of `size` amplitudes: 1 when it fits a small CTA,
// else env FFQ_SECTOR_CL (2, 4 or 8), default 2 (throughput-optimal at 18 qubits)
int sector_parts(ffq_ctx_t ctx, uint32_t size) {
  return size <= kSectorSingleMax ? 1 : ctx->sector_cl;
}

// compiled + uploaded support-closure program for (plan, Hamiltonian, hf), or
// nullptr when the closure does not fit the cluster (then other paths run)
// k_sector_eval's dynamic smem: Hmax + 1 amplitudes (zero slot), then either
// the generator tables (cs and the two F per op, this rank's pair range and
// flags per op) or, in the expectation, the peer-chunk buffer
size_t sector_smem_bytes(size_t hmax, size_t n_ops, size_t buf_len = 0) {
  const size_t tables = 3 * n_ops * sizeof(double2) + n_ops * (sizeof(uint2) + 1);
  return (hmax + 1) * sizeof(double2) + std::max(tables, buf_len * sizeof(double2)) + 16;
}

// k_sector_eval_real's dynamic smem: size + 1 real amplitudes, then (cos, sin),
// (sin F_lo, sin F_hi) and the pair range per op
size_t sector_real_smem_bytes(size_t size, size_t n_ops) {
  return (((size + 1) * sizeof(double) + 15) & ~(size_t)15) + n_ops * (2 * sizeof(double2) + sizeof(uint2)) + 16;
}

// every fused op with one pattern pair and real antisymmetric F (UCCSD: F = +-1)
bool plan_is_real(const CompiledPlan& P) {
  if (P.n_string_ops() > 0) return false;
  for (size_t op = 0; op < P.op_kind.size(); ++op) {
    const FusedDesc& d = P.fused[P.op_idx[op]];
    if (d.npair != 1 || P.pair_f[4 * d.pair_off + 1] != 0.0 || P.pair_f[4 * d.pair_off + 3] != 0.0) return false;
    // a real unitary 2x2 block with equal diagonal is a rotation: F_hi = -F_lo
    // (the real programs turn a pair's sign into a swap of its members)
    if (P.pair_f[4 * d.pair_off + 2] != -P.pair_f[4 * d.pair_off]) return false;
  }
  return true;
}

// every class sum real, so every pair's f(m) is real
bool ham_is_real(const CompiledHam& H) {
  for (size_t i = 1; i < H.cls_f.size(); i += 2)
    if (H.cls_f[i] != 0.0) return false;
  return true;
}

const SectorDev* sector_program(ffq_ctx_t ctx, ffq_plan_s* pl, ffq_ham_s* h, uint64_t hf) {
  auto key = std::make_pair(h->uid, hf);
  auto it = pl->sectors.find(key);
  if (it == pl->sectors.end()) {
    auto b = std::make_unique<ffq_plan_s::SectorDevBufs>();
    const size_t tables = sector_smem_bytes(0, pl->cp.op_kind.size());
    const uint32_t max_part =
        ctx->smem_optin > tables ? (uint32_t)((ctx->smem_optin - tables) / sizeof(double2)) : 0u;
    // real amplitudes for every theta (see k_sector_eval_real): real F on every
    // generator, real class sums, basis-state start
    const bool real_ok = ctx->sector_real && plan_is_real(pl->cp) && ham_is_real(h->ch);
    // closure size first (one part, no size limit on the part), then either the
    // one-CTA real program or the cluster split (rows padded to multiples of 4)
    // (anchored string blocks for the 1024-thread real program: FFQ_BLOCKS=0 disables them)
    b->prog = compile_sector(pl->cp, h->ch, hf, kSectorMaxSize, 0xFFFFFFFFu, 1, 0xFFFFFFFFu, 4, real_ok ? 8 : 16,
                             real_ok && ctx->sector_blocks ? kSectorRealThreads / 32 : 0, kSectorSingleMax,
                             real_ok && ctx->sector_blocks && ctx->sector_cliques);
    b->real = b->prog.ok && real_ok &&
              sector_real_smem_bytes(b->prog.n_slots, pl->cp.op_kind.size()) +
                      b->prog.ftab.size() * sizeof(double) <= ctx->smem_optin;
    // (a real-format compile that does not become the real program is redone: its
    // generator words are in the real program's format)
    if (b->prog.ok && !b->real && (real_ok || sector_parts(ctx, b->prog.size) > 1))
      b->prog = compile_sector(pl->cp, h->ch, hf, kSectorMaxSize, max_part, sector_parts(ctx, b->prog.size),
                               (uint32_t)((ctx->smem_optin - 16) / sizeof(double2)), 4);
    if (b->prog.ok) {
      b->gen_off.upload(b->prog.gen_off, ctx->stream);
      b->gen_pairs.upload(b->prog.gen_pairs, ctx->stream);
      if (!b->prog.gen_head.empty()) b->gen_head.upload(b->prog.gen_head, ctx->stream);
      b->gen_flags.upload(b->prog.gen_flags, ctx->stream);
      b->op_cross.upload(b->prog.op_cross, ctx->stream);
      b->row_pairs.upload(b->prog.row_pairs, ctx->stream);
      std::vector<int32_t> secs;
      for (const auto& es : b->prog.sections)
        secs.insert(secs.end(), {es.src_rank, es.src_off, es.len, es.sh0, es.sh1, es.pp1, es.pf_base});
      b->secs.upload(secs, ctx->stream);
      b->row_fre.upload(b->prog.row_fre, ctx->stream);
      b->pf_re.upload(b->prog.pf_re, ctx->stream);
      if (b->prog.product && !b->prog.blk_warp.empty()) {
        b->blk_warp.upload(b->prog.blk_warp, ctx->stream);
        b->blk_stream.upload(b->prog.blk_stream, ctx->stream);
        b->ftab.upload(b->prog.ftab, ctx->stream);
      }
      if (!b->prog.eps_flip.empty()) b->eps_flip.upload(b->prog.eps_flip, ctx->stream);
      if (b->prog.product && !b->prog.cq_warp.empty()) {
        b->cq_rows.upload(b->prog.cq_rows, ctx->stream);
        b->cq_desc.upload(b->prog.cq_desc, ctx->stream);
        b->cq_warp.upload(b->prog.cq_warp, ctx->stream);
        b->cq_coef.upload(b->prog.cq_coef, ctx->stream);
      }
      if (!b->prog.f_real) {
        b->row_fim.upload(b->prog.row_fim, ctx->stream);
        b->pf_im.upload(b->prog.pf_im, ctx->stream);
      }
      std::vector<ulonglong2> warm;
      auto range = [&](const void* p, size_t bytes) {
        if (p && bytes) warm.push_back(make_ulonglong2((unsigned long long)(uintptr_t)p, (unsigned long long)bytes));
      };
      range(b->gen_off.p, b->prog.gen_off.size() * sizeof(int64_t));
      range(b->gen_pairs.p, b->prog.gen_pairs.size() * sizeof(uint32_t));
      range(b->gen_head.p, b->prog.gen_head.size() * sizeof(uint32_t));
      range(b->row_pairs.p, b->prog.row_pairs.size() * sizeof(uint32_t));
      range(b->row_fre.p, b->prog.row_fre.size() * sizeof(double));
      range(b->pf_re.p, b->prog.pf_re.size() * sizeof(double));
      range(b->blk_warp.p, b->blk_warp.p ? b->prog.blk_warp.size() * sizeof(int32_t) : 0);
      range(b->blk_stream.p, b->blk_stream.p ? b->prog.blk_stream.size() * sizeof(uint32_t) : 0);
      range(b->cq_rows.p, b->cq_rows.p ? b->prog.cq_rows.size() * sizeof(uint32_t) : 0);
      range(b->cq_desc.p, b->cq_desc.p ? b->prog.cq_desc.size() * sizeof(int32_t) : 0);
      range(b->cq_coef.p, b->cq_coef.p ? b->prog.cq_coef.size() * sizeof(double) : 0);
      b->n_warm = (int)warm.size();
      b->warm.upload(warm, ctx->stream);
      CK(cudaStreamSynchronize(ctx->stream));
    }
    it = pl->sectors.emplace(key, std::move(b)).first;
  }
  auto& b = *it->second;
  if (!b.prog.ok) return nullptr;
  static thread_local SectorDev sd;
  sd = SectorDev{};
  sd.size = b.prog.size;
  for (int r = 0; r <= b.prog.n_parts; ++r) {
    sd.part_start[r] = b.prog.part_start[r];
    sd.sec_off[r] = b.prog.sec_off[r];
  }
  sd.op_cross = b.op_cross.p;
  sd.hf_slot = b.prog.hf_slot;
  sd.f_real = b.prog.f_real ? 1 : 0;
  sd.n_ops = (int)pl->cp.op_kind.size();
  sd.gen_off = b.gen_off.p;
  sd.gen_pairs = b.gen_pairs.p;
  sd.gen_head = b.gen_head.p;
  sd.gen_flags = b.gen_flags.p;
  sd.buf_off = b.prog.buf_off;
  sd.buf_len = b.prog.buf_len;
  sd.secs = b.secs.p;
  sd.row_pairs = b.row_pairs.p;
  sd.row_fre = b.row_fre.p;
  sd.row_fim = b.prog.f_real ? nullptr : b.row_fim.p;
  sd.pf_re = b.pf_re.p;
  sd.pf_im = b.prog.f_real ? nullptr : b.pf_im.p;
  sd.n_parts = b.prog.n_parts;
  sd.real = b.real ? 1 : 0;
  sd.n_slots = b.prog.n_slots;
  const bool blk = b.prog.product && !b.prog.blk_warp.empty();
  sd.blk_warp = blk ? reinterpret_cast<const int4*>(b.blk_warp.p) : nullptr;
  sd.blk_stream = blk ? b.blk_stream.p : nullptr;
  sd.ftab = blk ? b.ftab.p : nullptr;
  sd.n_ftab = blk ? (int)b.prog.ftab.size() : 0;
  const bool cq = blk && !b.prog.cq_warp.empty();
  sd.eps_flip = blk && !b.prog.eps_flip.empty() ? b.eps_flip.p : nullptr;
  sd.cq_rows = cq ? b.cq_rows.p : nullptr;
  sd.cq_desc = cq ? reinterpret_cast<const int4*>(b.cq_desc.p) : nullptr;
  sd.cq_warp = cq ? reinterpret_cast<const int2*>(b.cq_warp.p) : nullptr;
  sd.cq_coef = cq ? b.cq_coef.p : nullptr;
  sd.warm = b.warm.p;
  sd.max_warp_tasks = 0;
  for (size_t w2 = 0; w2 + 1 < b.prog.cq_warp.size(); w2 += 2)
    sd.max_warp_tasks = std::max(sd.max_warp_tasks, b.prog.cq_warp[w2 + 1] - b.prog.cq_warp[w2]);
  sd.n_warm = b.n_warm;
  return &sd;
}

template <int CL, int NT>
void launch_sector_t(ffq_ctx_t ctx, const ffq_plan_s* pl, const SectorDev& sd, const double* theta, int batch,
                     double* e, double* im, long long* clk) {
  size_t hmax = 0;
  for (int r = 0; r < CL; ++r) hmax = std::max<size_t>(hmax, sd.part_start[r + 1] - sd.part_start[r]);
  const size_t sb = sector_smem_bytes(hmax, pl->cp.op_kind.size(), sd.buf_len);
  CK(cudaFuncSetAttribute(k_sector_eval<CL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  if (CL > 1) CK(cudaFuncSetAttribute(k_sector_eval<CL, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)batch * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sb;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_sector_eval<CL, NT>, sd, pl->dev(), theta, pl->cp.n_gen, e, im, batch, clk));
  ctx->launches++;
}

template <int NT>
void launch_sector_real(ffq_ctx_t ctx, const ffq_plan_s* pl, const SectorDev& sd, const double* theta, int batch,
                        double* e, double* im, long long* clk, double* state_out = nullptr) {
  // anchored blocks keep the shared-row f table behind the per-op tables
  const size_t sb = sector_real_smem_bytes(sd.n_slots, pl->cp.op_kind.size()) + (size_t)sd.n_ftab * sizeof(double);
  CK(cudaFuncSetAttribute(k_sector_eval_real<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  if (NT == 32 * 32) CK(cudaFuncSetAttribute(k_sector_eval_real<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  // Batches smaller than the SM count: up to sector_split CTAs per evaluation
  // (1024-thread program only). Each runs the generator phase and 32 / split
  // of the warp shares of the expectation; the energies are bit-identical.
  int split = 1;
  if (NT == 32 * 32 && !state_out)
    while (split * 2 <= ctx->sector_split && (int64_t)batch * split * 2 <= ctx->n_sm) split *= 2;
  if (split > 1) ctx->warp_sums.alloc((size_t)batch * 32);
  // role warps (split evaluations of the 1024-thread program): each of the
  // 32 / split warp shares of a CTA gets `roles` warps (generic rows, block
  // stream segments, clique tasks); needs >= 2 warps per share and the exchange
  // buffer ([share][segments + tasks][32] doubles) inside the per-op tables
  int roles = 0;
  if (split > 1 && ctx->sector_roles) {
    const int r = 32 / (32 / split);
    const size_t need = (size_t)(32 / split) * ((r >= 3 ? kBlkSegments : 0) + sd.max_warp_tasks) * 32 * sizeof(double);
    if (r >= 2 && need <= pl->cp.op_kind.size() * 2 * sizeof(double2)) roles = r;
  }
  // a batch of at most one wave: all SMs pull the tables into L2 (cold tables cost
  // 14-40 us inside the serial generator phase, the pass 4 us) -- on the idle SMs
  // inside a role-warp launch (extra CTAs past the batch), else as a launch before it
  const bool warm = NT == 32 * 32 && batch * split <= ctx->n_sm && sd.n_warm > 0 && ctx->sector_warm;
  const int warm_ctas = warm && roles >= 2 ? ctx->n_sm - batch * split : 0;
  if (warm && warm_ctas == 0) {  // (small programs: KBs of tables)
    k_l2_warm<<<2 * ctx->n_sm, 256, 0, ctx->stream>>>(sd.warm, sd.n_warm);
    ctx->launches++;
  }
  if (roles >= 2) {
    // (the evaluation's last CTA adds its warp sums: one arrival ticket per row, left at zero)
    if ((size_t)batch > ctx->row_tickets.n || !ctx->row_tickets.p) {
      ctx->row_tickets.alloc((size_t)batch);
      CK(cudaMemsetAsync(ctx->row_tickets.p, 0, ctx->row_tickets.n * sizeof(int), ctx->stream));
    }
    k_sector_eval_real<NT, NT == 32 * 32><<<batch * split + warm_ctas, NT, sb, ctx->stream>>>(
        sd, pl->dev(), theta, pl->cp.n_gen, e, im, batch, clk, split, ctx->warp_sums.p, state_out, roles,
        ctx->row_tickets.p);
  } else {
    k_sector_eval_real<NT, false><<<batch * split, NT, sb, ctx->stream>>>(
        sd, pl->dev(), theta, pl->cp.n_gen, e, im, batch, clk, split, ctx->warp_sums.p, state_out, roles, nullptr);
  }
  CK(cudaGetLastError());
  ctx->launches++;
  if (split > 1 && roles < 2) {
    k_sum_warps<<<batch, 32, 0, ctx->stream>>>(ctx->warp_sums.p, e, im);
    CK(cudaGetLastError());
    ctx->launches++;
  }
}

void launch_sector(ffq_ctx_t ctx, const ffq_plan_s* pl, const SectorDev& sd, const double* theta, int batch,
                   double* e, double* im) {
  static const bool clocks = std::getenv("FFQ_PHASE_CLOCKS") != nullptr;
  DevBuf<long long> clk;
  if (clocks) {
    clk.alloc(2 * (size_t)batch + 32);
    CK(cudaMemsetAsync(clk.p, 0, (2 * (size_t)batch + 32) * sizeof(long long), ctx->stream));
  }
  long long* cp = clocks ? clk.p : nullptr;
  if (sd.real) {
    if (sd.size <= kSectorSingleMax)
      launch_sector_real<kSectorSingleThreads>(ctx, pl, sd, theta, batch, e, im, cp);
    else
      launch_sector_real<kSectorRealThreads>(ctx, pl, sd, theta, batch, e, im, cp);
  } else switch (sd.n_parts) {
    case 1: launch_sector_t<1, kSectorSingleThreads>(ctx, pl, sd, theta, batch, e, im, cp); break;
    case 2: launch_sector_t<2, kSectorThreads>(ctx, pl, sd, theta, batch, e, im, cp); break;
    case 4: launch_sector_t<4, kSectorThreads>(ctx, pl, sd, theta, batch, e, im, cp); break;
    default: launch_sector_t<8, kSectorThreads>(ctx, pl, sd, theta, batch, e, im, cp); break;
  }
  if (clocks) {
    std::vector<long long> hc(2 * (size_t)batch + 32);
    CK(cudaMemcpyAsync(hc.data(), clk.p, hc.size() * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double g = 0, x = 0;
    for (int r = 0; r < batch; ++r) { g += (double)hc[2 * r]; x += (double)hc[2 * r + 1]; }
    std::fprintf(stderr, "[ffq] sector rows=%d avg cycles: generators %.0f expectation %.0f\n", batch,
                 g / batch, x / batch);
    if (hc[2 * (size_t)batch]) {  // per-warp expectation cycles of row 0 (one-CTA real program)
      std::fprintf(stderr, "[ffq] row 0 expectation cycles per warp:");
      for (int w = 0; w < 32; ++w) std::fprintf(stderr, " %lld", hc[2 * (size_t)batch + w]);
      std::fprintf(stderr, "\n");
    }
  }
}

bool use_smem_path(ffq_ctx_t ctx, const ffq_plan_s* pl) {
  return pl->cp.n_qubits <= ctx->smem_max_qubits && smem_bytes(pl) <= ctx->smem_optin;
}

// energies of `batch` rows of theta (device) into e/im (device), async
#include "ffq_compact.inl"

void energy_device(ffq_ctx_t ctx, ffq_plan_s* pl, ffq_ham_s* h, uint64_t hf, int batch,
                   const double* theta_dev, double* e_dev, double* im_dev) {
  const int n = pl->cp.n_qubits;
  if (h->ch.n_qubits != n) throw BadInput("plan and Hamiltonian qubit counts differ", FFQ_EINVAL);
  if (n < 64 && (hf >> n) != 0) throw BadInput("hf_bits exceeds n_qubits", FFQ_EINVAL);
  if (batch <= 0) return;
  // support-closure evaluator first (FFQ_SECTOR=0 disables it); plans it cannot
  // take (non-fused generators, closures beyond 32768 amplitudes) fall through,
  // real spin-conserving ones to the compact sector layout (FFQ_COMPACT=0 disables it)
  if (ctx->sector) {
    if (const SectorDev* sd = sector_program(ctx, pl, h, hf)) {
      launch_sector(ctx, pl, *sd, theta_dev, batch, e_dev, im_dev);
      return;
    }
  }
  if (ctx->compact && (n >= ctx->compact_min_qubits || (n >= ctx->compact_min_qubits - 2 && batch >= 8)))
    if (CompactProg* cpg = compact_program(ctx, pl, h, hf)) {
      compact_energy(ctx, pl, *cpg, theta_dev, batch, e_dev, im_dev);
      return;
    }
  if (use_smem_path(ctx, pl)) {
    const size_t sb = smem_bytes(pl);
    CK(cudaFuncSetAttribute(k_smem_eval<kThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sb));
    k_smem_eval<kThreads><<<batch, kThreads, sb, ctx->stream>>>(n, pl->dev(), h->dev(), hf,
                                                                theta_dev, pl->cp.n_gen, e_dev,
                                                                im_dev);
    CK(cudaGetLastError());
    ctx->launches++;
    return;
  }
  // global path: chunk the batch so the slab stays L2-resident (<= 64 MiB)
  const int64_t dim = 1LL << n;
  const int64_t slab_cap = ctx->slab_bytes / (dim * (int64_t)sizeof(double2));
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(batch, std::max<int64_t>(1, slab_cap)));
  const int n_ops = (int)pl->cp.op_kind.size();
  const bool sp = use_support(ctx, n);
  const int64_t items = h->n_partials(sp);
  const int64_t rstride = dim;  // slab row stride (the support kernels take it explicitly)
  if (ctx->slab.n < (size_t)chunk * rstride) ctx->slab_clean = false;
  ctx->slab.alloc((size_t)chunk * rstride);
  if (sp) ctx->slab_sup.alloc((size_t)chunk * (dim >> 5));
  if (sp && !ctx->slab_clean) {
    CK(cudaMemsetAsync(ctx->slab.p, 0, sizeof(double2) * ctx->slab.n, ctx->stream));
    ctx->slab_clean = true;
  }
  uint32_t* sup = sp ? ctx->slab_sup.p : nullptr;
  ctx->cs.alloc((size_t)chunk * std::max(1, n_ops));
  ctx->partial.alloc((size_t)chunk * std::max<int64_t>(1, items));
  ctx->theta.alloc((size_t)chunk * std::max(1, pl->cp.n_gen));
  ctx->eout.alloc(chunk);
  ctx->eim.alloc(chunk);
  GraphKey key{(uintptr_t)h->uid, (uintptr_t)chunk, (uintptr_t)hf, (uintptr_t)ctx->theta.p,
               (uintptr_t)ctx->slab.p, (uintptr_t)ctx->cs.p, (uintptr_t)ctx->partial.p,
               (uintptr_t)ctx->eout.p, (uintptr_t)ctx->eim.p, (uintptr_t)sup};
  auto it = pl->graphs.find(key);
  if (it == pl->graphs.end()) {
    cudaGraph_t graph;
    const int64_t before = ctx->launches;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      if (sup) {
        // clean slab: only the HF amplitudes are written; the support is zeroed at the end
        k_set_basis_sparse<<<grid_for(chunk, ctx->n_sm), kThreads, 0, ctx->stream>>>(ctx->slab.p, n, chunk, hf,
                                                                                      rstride);
        k_support_basis<<<grid_for((dim >> 5) * chunk, ctx->n_sm), kThreads, 0, ctx->stream>>>(
            sup, dim >> 5, chunk, hf);
        ctx->launches += 2;
      } else {
        k_set_basis<<<grid_for(dim * chunk, ctx->n_sm), kThreads, 0, ctx->stream>>>(ctx->slab.p, dim,
                                                                                   chunk, hf);
        ctx->launches++;
      }
      launch_cs(ctx, pl, ctx->theta.p, chunk, ctx->cs.p);
      run_plan_ops(ctx, pl, ctx->slab.p, sup, chunk, ctx->cs.p, rstride);
      launch_expect(ctx, h, ctx->slab.p, sup, n, chunk, ctx->partial.p, ctx->eout.p, ctx->eim.p, rstride);
      if (sup) {
        k_support_zero<<<grid_for(((dim >> 5) * chunk) * 32, ctx->n_sm), kThreads, 0, ctx->stream>>>(
            ctx->slab.p, sup, n, chunk, rstride);
        ctx->launches++;
      }
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      throw;
    }
    CK(cudaStreamEndCapture(ctx->stream, &graph));
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->graph_nodes[key] = ctx->launches - before;
    ctx->launches = before;
    it = pl->graphs.emplace(key, exec).first;
  }
  const int64_t nodes = pl->graph_nodes[key];
  for (int b0 = 0; b0 < batch; b0 += chunk) {
    const int nb = std::min(chunk, batch - b0);
    CK(cudaMemcpyAsync(ctx->theta.p, theta_dev + (int64_t)b0 * pl->cp.n_gen,
                       sizeof(double) * (size_t)nb * pl->cp.n_gen, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    // rows past nb in the last chunk recompute stale theta; their outputs are dropped
    if (cudaGraphLaunch(it->second, ctx->stream) != cudaSuccess) {
      ctx->slab_clean = false;
      throw CudaError("cudaGraphLaunch failed");
    }
    ctx->launches += nodes;
    CK(cudaMemcpyAsync(e_dev + b0, ctx->eout.p, sizeof(double) * nb, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    if (im_dev)
      CK(cudaMemcpyAsync(im_dev + b0, ctx->eim.p, sizeof(double) * nb, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  }
}

}  // namespace

// support bitmap of a state, rebuilt from the data if a dense pass left it stale
uint32_t* state_support(ffq_state_s* st) {
  ffq_ctx_t ctx = st->ctx;
  if (!use_support(ctx, st->n)) return nullptr;
  st->sup.alloc((size_t)st->batch << (st->n - 5));
  if (!st->sup_valid) {
    launch_support_from_state(ctx, st->psi.p, st->sup.p, st->n, st->batch);
    st->sup_valid = true;
  }
  return st->sup.p;
}

extern "C" {

int ffq_version(void) { return kVersion; }

int ffq_device_count(int* n_out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    if (n_out) *n_out = 0;
    return fail(nullptr, FFQ_ENODEV, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  if (n_out) *n_out = n;
  return FFQ_OK;
}

int ffq_ctx_create(int device, ffq_ctx_t* out) {
  if (!out) return fail(nullptr, FFQ_EINVAL, "ffq_ctx_create: null out");
  *out = nullptr;
  int n = 0;
  if (ffq_device_count(&n) != FFQ_OK || n == 0)
    return fail(nullptr, FFQ_ENODEV, "no CUDA device available (the hot path has no CPU fallback)");
  if (device < 0 || device >= n) return fail(nullptr, FFQ_EINVAL, "device ordinal out of range");
  auto* c = new ffq_ctx_s();
  c->device = device;
  int rc = guarded(c, [&] {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device));
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    c->smem_optin = (size_t)optin - 2048;  // static smem of the reduction scratch
    if (const char* e = std::getenv("FFQ_SMEM_MAX_QUBITS")) c->smem_max_qubits = std::atoi(e);
    if (const char* e = std::getenv("FFQ_ROT_TILE")) c->rot_tile_bits = std::min(12, std::max(0, std::atoi(e)));
    CK(cudaFuncSetAttribute(k_rotation_run<kRotRunThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double2) << 12)));
    CK(cudaFuncSetAttribute(k_rotation_run<kRotRunThreads>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            (int)cudaSharedmemCarveoutMaxShared));
    if (const char* e = std::getenv("FFQ_SLAB_MB")) c->slab_bytes = std::max(1LL, std::atoll(e)) << 20;
    if (const char* e = std::getenv("FFQ_SUPPORT")) c->support = std::atoi(e);
    if (const char* e = std::getenv("FFQ_SECTOR")) c->sector = std::atoi(e);
    if (const char* e = std::getenv("FFQ_SECTOR_REAL")) c->sector_real = std::atoi(e);
    if (const char* e = std::getenv("FFQ_BLOCKS")) c->sector_blocks = std::atoi(e);
    if (const char* e = std::getenv("FFQ_CLIQUES")) c->sector_cliques = std::atoi(e);
    if (const char* e = std::getenv("FFQ_COMPACT")) c->compact = std::atoi(e);
    if (const char* e = std::getenv("FFQ_COMPACT_MIN")) c->compact_min_qubits = std::atoi(e);
    if (const char* e = std::getenv("FFQ_COMPACT_IL")) c->compact_il = std::atoi(e);
    if (const char* e = std::getenv("FFQ_COMPACT_GRAPH")) c->compact_graph = std::atoi(e);
    if (const char* e = std::getenv("FFQ_WARM")) c->sector_warm = std::atoi(e);
    if (const char* e = std::getenv("FFQ_ROLES")) c->sector_roles = std::atoi(e);
    if (const char* e = std::getenv("FFQ_SPLIT")) c->sector_split = std::min(32, std::max(1, std::atoi(e)));
    if (const char* e = std::getenv("FFQ_SECTOR_CL")) {
      const int v = std::atoi(e);
      c->sector_cl = (v == 4 || v == 8) ? v : 2;
    }
    return FFQ_OK;
  });
  if (rc != FFQ_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return FFQ_OK;
}

int ffq_ctx_destroy(ffq_ctx_t ctx) {
  if (!ctx) return FFQ_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  for (cudaEvent_t e : ctx->copy_done) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  delete ctx;
  return FFQ_OK;
}

int ffq_ctx_synchronize(ffq_ctx_t ctx) {
  if (!ctx) return fail(nullptr, FFQ_EINVAL, "null context");
  return guarded(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->stream));
    return FFQ_OK;
  });
}

const char* ffq_last_error(ffq_ctx_t ctx) { return ctx ? ctx->err.c_str() : g_thread_err.c_str(); }

int64_t ffq_ctx_kernel_launches(ffq_ctx_t ctx) { return ctx ? ctx->launches : 0; }

int ffq_ctx_stream(ffq_ctx_t ctx, void** stream) {
  if (!ctx || !stream) return fail(ctx, FFQ_EINVAL, "null argument");
  *stream = (void*)ctx->stream;
  return FFQ_OK;
}

int ffq_ham_upload(ffq_ctx_t ctx, int n_qubits, int64_t n_terms, const uint64_t* x,
                   const uint64_t* z, const double* c_re, const double* c_im, ffq_ham_t* out) {
  if (!ctx || !out || (n_terms > 0 && (!x || !z || !c_re || !c_im)))
    return fail(ctx, FFQ_EINVAL, "ffq_ham_upload: null argument");
  *out = nullptr;
  return guarded(ctx, [&] {
    auto h = std::make_unique<ffq_ham_s>();
    h->ctx = ctx;
    h->ch = compile_ham(n_qubits, n_terms, x, z, c_re, c_im);
    h->raw_x.assign(x, x + n_terms);
    h->raw_z.assign(z, z + n_terms);
    h->raw_re.assign(c_re, c_re + n_terms);
    h->raw_im.assign(c_im, c_im + n_terms);
    const auto& ch = h->ch;
    h->groups.upload(ch.groups, ctx->stream);
    h->act_bits.upload(ch.act_bits, ctx->stream);
    h->cls_z.upload(ch.cls_z, ctx->stream);
    std::vector<double2> f(ch.cls_f.size() / 2);
    for (size_t i = 0; i < f.size(); ++i) f[i] = make_double2(ch.cls_f[2 * i], ch.cls_f[2 * i + 1]);
    h->cls_f.upload(f, ctx->stream);
    h->item_g.upload(ch.item_g, ctx->stream);
    h->item_p.upload(ch.item_p, ctx->stream);
    h->item_u0.upload(ch.item_u0, ctx->stream);
    h->act_low.upload(ch.act_low, ctx->stream);
    h->sitem_g.upload(ch.sitem_g, ctx->stream);
    h->sitem_p.upload(ch.sitem_p, ctx->stream);
    h->sitem_w0.upload(ch.sitem_w0, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    *out = h.release();
    return FFQ_OK;
  });
}

int ffq_ham_destroy(ffq_ham_t ham) {
  if (ham) {
    cudaSetDevice(ham->ctx->device);
    delete ham;
  }
  return FFQ_OK;
}

int ffq_ham_info(ffq_ham_t ham, int* n_groups, int64_t* n_terms, int64_t* n_classes) {
  if (!ham) return fail(nullptr, FFQ_EINVAL, "null Hamiltonian");
  if (n_groups) *n_groups = (int)ham->ch.groups.size();
  if (n_terms) *n_terms = ham->ch.n_terms;
  if (n_classes) *n_classes = ham->ch.n_classes();
  return FFQ_OK;
}

int ffq_plan_upload(ffq_ctx_t ctx, int n_qubits, int n_gen, const int64_t* term_off,
                    const uint64_t* x, const uint64_t* z, const double* c_re, const double* c_im,
                    ffq_plan_t* out) {
  if (!ctx || !out || (n_gen > 0 && !term_off)) return fail(ctx, FFQ_EINVAL, "ffq_plan_upload: null argument");
  *out = nullptr;
  return guarded(ctx, [&] {
    if (n_gen > 0 && term_off[n_gen] > 0 && (!x || !z || !c_re || !c_im))
      throw BadInput("ffq_plan_upload: null term arrays", FFQ_EINVAL);
    auto p = std::make_unique<ffq_plan_s>();
    p->ctx = ctx;
    p->cp = compile_plan(n_qubits, n_gen, term_off, x, z, c_re, c_im);
    const auto& cp = p->cp;
    p->op_kind.upload(cp.op_kind, ctx->stream);
    p->op_gen.upload(cp.op_gen, ctx->stream);
    p->op_idx.upload(cp.op_idx, ctx->stream);
    p->op_cfac.upload(cp.op_cfac, ctx->stream);
    p->op_sscale.upload(cp.op_sscale, ctx->stream);
    p->fused.upload(cp.fused, ctx->stream);
    p->pair_bits.upload(cp.pair_bits, ctx->stream);
    p->pair_low.upload(cp.pair_low, ctx->stream);
    std::vector<double2> pf(cp.pair_f.size() / 2);
    for (size_t i = 0; i < pf.size(); ++i) pf[i] = make_double2(cp.pair_f[2 * i], cp.pair_f[2 * i + 1]);
    p->pair_f.upload(pf, ctx->stream);
    const size_t nop = cp.op_kind.size();
    std::vector<RotDesc> rd(nop, RotDesc{0, 0, 0, 0, 0});
    std::vector<uint64_t> ox(nop, 0), oz(nop, 0);
    std::vector<char> ok(nop, 0);
    for (size_t op = 0; op < nop; ++op)
      if (cp.op_kind[op] != 0) {
        const int si = cp.op_idx[op];
        ox[op] = cp.str_x[si];
        oz[op] = cp.str_z[si];
        rd[op].ny = cp.str_ny[si];
        ok[op] = 1;
      }
    p->runs_t = ctx->rot_tile_bits > 0 ? std::min(n_qubits, ctx->rot_tile_bits) : 0;
    p->runs = build_rot_runs(rd, ox.data(), oz.data(), ok, n_qubits, p->runs_t);
    p->rot_groups.upload(p->runs.groups, ctx->stream);
    p->rot.upload(rd, ctx->stream);
    p->str_x.upload(cp.str_x, ctx->stream);
    p->str_z.upload(cp.str_z, ctx->stream);
    p->str_ny.upload(cp.str_ny, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    *out = p.release();
    return FFQ_OK;
  });
}

int ffq_plan_destroy(ffq_plan_t plan) {
  if (plan) {
    cudaSetDevice(plan->ctx->device);
    delete plan;
  }
  return FFQ_OK;
}

int ffq_plan_info(ffq_plan_t plan, int* n_fused, int* n_string_ops) {
  if (!plan) return fail(nullptr, FFQ_EINVAL, "null plan");
  if (n_fused) *n_fused = plan->cp.n_fused();
  if (n_string_ops) *n_string_ops = plan->cp.n_string_ops();
  return FFQ_OK;
}

int ffq_energy_batch_device(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits,
                            int batch, const double* theta_dev, double* e_dev, double* imag_dev) {
  if (!ctx || !plan || !ham || batch < 0 || (batch > 0 && (!e_dev || (!theta_dev && plan->cp.n_gen > 0))))
    return fail(ctx, FFQ_EINVAL, "ffq_energy_batch_device: invalid argument");
  return guarded(ctx, [&] {
    energy_device(ctx, plan, ham, hf_bits, batch, theta_dev, e_dev, imag_dev);
    return FFQ_OK;
  });
}

int ffq_energy_prepare(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits) {
  if (!ctx || !plan || !ham) return fail(ctx, FFQ_EINVAL, "ffq_energy_prepare: invalid argument");
  return guarded(ctx, [&] {
    const int n = plan->cp.n_qubits;
    if (ham->ch.n_qubits != n) throw BadInput("plan and Hamiltonian qubit counts differ", FFQ_EINVAL);
    if (n < 64 && (hf_bits >> n) != 0) throw BadInput("hf_bits exceeds n_qubits", FFQ_EINVAL);
    // the same order as energy_device: sector program first, then the compact layout
    if (ctx->sector && sector_program(ctx, plan, ham, hf_bits)) return FFQ_OK;
    if (ctx->compact && n >= ctx->compact_min_qubits - 2) compact_program(ctx, plan, ham, hf_bits);
    return FFQ_OK;
  });
}

int ffq_compact_emulate(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* px, const uint64_t* pz,
                        const double* pc_re, const double* pc_im, int64_t n_terms, const uint64_t* hx,
                        const uint64_t* hz, const double* hc_re, const double* hc_im, uint64_t hf_bits,
                        const double* theta, double* out) {
  if (!out || !term_off || n_qubits < 2 || n_qubits > 32 || (n_gen > 0 && !theta))
    return fail(nullptr, FFQ_EINVAL, "ffq_compact_emulate: invalid argument");
  return guarded(nullptr, [&] {
    const CompiledPlan P = compile_plan(n_qubits, n_gen, term_off, px, pz, pc_re, pc_im);
    for (int64_t t = 0; t < n_terms; ++t)
      if (hc_im && std::abs(hc_im[t]) > 1e-12)
        return fail(nullptr, FFQ_ENONHERMITIAN, "ffq_compact_emulate: imaginary coefficient");
    CompactProg cp;
    compact_compile(P, std::vector<uint64_t>(hx, hx + n_terms), std::vector<uint64_t>(hz, hz + n_terms),
                    std::vector<double>(hc_re, hc_re + n_terms), hf_bits, &cp);
    for (int i = 0; i < 8; ++i) out[i] = 0.0;
    out[1] = cp.ok ? 1.0 : 0.0;
    if (!cp.ok) return FFQ_OK;
    int64_t bad = 0;
    out[0] = compact_emulate(P, cp, theta, &bad);
    out[2] = cp.na;
    out[3] = cp.nb;
    out[4] = (double)cp.gen_pairs;
    out[5] = (double)cp.term_pairs;
    out[6] = (double)bad;
    out[7] = (double)(cp.single.size() + cp.multi.size());
    return FFQ_OK;
  });
}

int ffq_sector_state(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, const double* theta,
                     double* psi, double* energy) {
  if (!ctx || !plan || !ham || !theta || !psi) return fail(ctx, FFQ_EINVAL, "ffq_sector_state: invalid argument");
  return guarded(ctx, [&] {
    if (!ctx->sector) return fail(ctx, FFQ_EINVAL, "ffq_sector_state: support-closure evaluator disabled (FFQ_SECTOR=0)");
    const SectorDev* sd = sector_program(ctx, plan, ham, hf_bits);
    if (!sd || !sd->real || sd->size <= kSectorSingleMax)
      return fail(ctx, FFQ_EINVAL, "ffq_sector_state: no 1024-thread real-amplitude sector program for these inputs");
    const SectorProgram& S = plan->sectors.at(std::make_pair(ham->uid, hf_bits))->prog;
    const int ng = plan->cp.n_gen;
    DevBuf<double> th, e, st;
    th.alloc((size_t)ng);
    e.alloc(1);
    st.alloc((size_t)S.n_slots);
    CK(cudaMemcpyAsync(th.p, theta, (size_t)ng * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    launch_sector_real<kSectorRealThreads>(ctx, plan, *sd, th.p, 1, e.p, nullptr, nullptr, st.p);
    std::vector<double> slots(S.n_slots);
    double eh = 0.0;
    CK(cudaMemcpyAsync(slots.data(), st.p, slots.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&eh, e.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const size_t dim = size_t(1) << plan->cp.n_qubits;
    std::memset(psi, 0, 2 * dim * sizeof(double));
    for (uint32_t i = 0; i < S.size; ++i) psi[2 * (size_t)S.basis[i]] = slots[S.slot_of[i]];
    if (energy) *energy = eh;
    return FFQ_OK;
  });
}

int ffq_sector_info(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, int64_t* out) {
  if (!ctx || !plan || !ham || !out) return fail(ctx, FFQ_EINVAL, "ffq_sector_info: invalid argument");
  return guarded(ctx, [&] {
    if (!ctx->sector) return fail(ctx, FFQ_EINVAL, "ffq_sector_info: support-closure evaluator disabled (FFQ_SECTOR=0)");
    if (!sector_program(ctx, plan, ham, hf_bits)) {
      const auto& b = *plan->sectors.at(std::make_pair(ham->uid, hf_bits));
      return fail(ctx, FFQ_EINVAL, "ffq_sector_info: no support-closure program: " + b.prog.why);
    }
    const auto& bufs = *plan->sectors.at(std::make_pair(ham->uid, hf_bits));
    const SectorProgram& S = bufs.prog;
    const int n_ops = (int)S.op_cross.size();
    int64_t cluster_steps = 0;
    for (int op = 0; op < n_ops; ++op)
      cluster_steps += S.n_parts > 1 && (S.op_cross[op] || op + 1 >= n_ops || S.op_cross[op + 1]);
    if (S.n_parts == 1) cluster_steps = 0;
    out[0] = S.size;
    out[1] = S.n_parts;
    out[2] = (int64_t)S.gen_pairs.size();
    out[3] = S.exp_pair_count;
    out[4] = (int64_t)(S.row_pairs.size() / 32 + S.blk_stream.size() / 32);
    out[5] = cluster_steps;
    out[6] = S.split_masks.empty() ? 0 : (int64_t)S.split_masks[0];
    out[7] = S.buf_len;
    out[8] = bufs.real ? 1 : 0;
    out[9] = S.blk_pairs;
    out[10] = S.n_slots;
    out[11] = S.cq_pairs;
    out[12] = (int64_t)(S.cq_desc.size() / 128);
    out[13] = S.cq_conflicts;
    int64_t lane_rows = 0;  // sum over clique lanes of their rows (12 amplitude loads each)
    for (size_t l = 0; l < S.cq_desc.size() / 4; ++l) lane_rows += S.cq_desc[4 * l + 3] - S.cq_desc[4 * l + 2];
    out[14] = lane_rows;
    return FFQ_OK;
  });
}

int ffq_energy_batch(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, int batch,
                     const double* theta, double* e_out) {
  if (!ctx || !plan || !ham || batch < 0 || (batch > 0 && (!e_out || (!theta && plan->cp.n_gen > 0))))
    return fail(ctx, FFQ_EINVAL, "ffq_energy_batch: invalid argument");
  if (batch == 0) return FFQ_OK;
  return guarded(ctx, [&] {
    const int ng = plan->cp.n_gen;
    const size_t nth = (size_t)batch * ng;
    // host -> pinned staging -> device, energies + residues back (one D2H). A
    // large batch goes in chunks of whole SM waves: the host copies chunk c + 1
    // into the staging buffer and its H2D is queued while chunk c computes
    // (energies are bitwise independent of the split).
    // theta already in page-locked host memory (cudaHostAlloc / cudaHostRegister,
    // e.g. a pinned torch tensor): the H2D copies read it in place, no staging
    cudaPointerAttributes pa{};
    const bool user_pinned = nth > 0 && cudaPointerGetAttributes(&pa, theta) == cudaSuccess &&
                             pa.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();  // (an unregistered pointer may leave a sticky-free error code on old drivers)
    ctx->ensure_pinned((user_pinned ? 0 : nth) + 2 * (size_t)batch);
    double* stage_e = ctx->pinned + (user_pinned ? 0 : nth);
    const double* src = user_pinned ? theta : ctx->pinned;
    DevBuf<double>& th = ctx->io_theta;
    DevBuf<double>& eo = ctx->io_e;
    th.alloc(std::max<size_t>(1, nth));
    eo.alloc(2 * (size_t)batch);
    // first chunk one wave (its staging is the exposed part), then 2, 4, ... waves
    // (a chunk boundary drains the SMs: few boundaries), a tail below one wave
    // joining the last chunk
    const bool piped = nth * sizeof(double) >= (size_t)(1 << 20);
    const int wave = std::max(1, ctx->n_sm);
    if (piped) {
      // the copies start after everything already queued on the context stream
      const cudaEvent_t start = ctx->copy_event(0);
      CK(cudaEventRecord(start, ctx->stream));
      CK(cudaStreamWaitEvent(ctx->copy_stream, start, 0));
    }
    for (int b0 = 0, k = 0; b0 < batch; ++k) {
      int nb = piped ? std::min((1 << std::min(k, 20)) * wave, batch - b0) : batch;
      if (piped && batch - b0 - nb < wave) nb = batch - b0;
      const size_t o = (size_t)b0 * ng, n = (size_t)nb * ng;
      if (n && piped) {
        // chunk k's copy runs on the copy stream while chunk k - 1 computes
        if (!user_pinned) std::memcpy(ctx->pinned + o, theta + o, n * sizeof(double));
        const cudaEvent_t ev = ctx->copy_event((size_t)k + 1);
        CK(cudaMemcpyAsync(th.p + o, src + o, n * sizeof(double), cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaEventRecord(ev, ctx->copy_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ev, 0));
      } else if (n) {
        if (!user_pinned) std::memcpy(ctx->pinned + o, theta + o, n * sizeof(double));
        CK(cudaMemcpyAsync(th.p + o, src + o, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      }
      energy_device(ctx, plan, ham, hf_bits, nb, th.p + o, eo.p + b0, eo.p + batch + b0);
      b0 += nb;
    }
    CK(cudaMemcpyAsync(stage_e, eo.p, 2 * sizeof(double) * batch, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::memcpy(e_out, stage_e, sizeof(double) * batch);
    for (int b = 0; b < batch; ++b)
      if (std::abs(stage_e[batch + b]) > 1e-10)
        throw BadInput("energy has imaginary residue " + std::to_string(stage_e[batch + b]) +
                           " > 1e-10 (non-Hermitian Hamiltonian?)",
                       FFQ_ENONHERMITIAN);
    return FFQ_OK;
  });
}

int ffq_state_alloc(ffq_ctx_t ctx, int n_qubits, int batch, ffq_state_t* out) {
  if (!ctx || !out || n_qubits < 2 || n_qubits > 40 || batch < 1 || batch > 65535)
    return fail(ctx, FFQ_EINVAL,
                "ffq_state_alloc: invalid argument (need n_qubits in [2,40], batch in [1,65535])");
  *out = nullptr;
  return guarded(ctx, [&] {
    auto s = std::make_unique<ffq_state_s>();
    s->ctx = ctx;
    s->n = n_qubits;
    s->batch = batch;
    s->psi.alloc((size_t)batch << n_qubits);
    *out = s.release();
    return FFQ_OK;
  });
}

int ffq_state_free(ffq_state_t st) {
  if (st) {
    cudaSetDevice(st->ctx->device);
    delete st;
  }
  return FFQ_OK;
}

int ffq_state_set_basis(ffq_state_t st, uint64_t bits) {
  if (!st) return fail(nullptr, FFQ_EINVAL, "null state");
  ffq_ctx_t ctx = st->ctx;
  if (st->n < 64 && (bits >> st->n)) return fail(ctx, FFQ_EINVAL, "basis index exceeds n_qubits");
  return guarded(ctx, [&] {
    const int64_t dim = 1LL << st->n;
    k_set_basis<<<grid_for(dim * st->batch, ctx->n_sm), kThreads, 0, ctx->stream>>>(st->psi.p, dim,
                                                                                   st->batch, bits);
    CK(cudaGetLastError());
    ctx->launches++;
    if (use_support(ctx, st->n)) {
      st->sup.alloc((size_t)st->batch << (st->n - 5));
      k_support_basis<<<grid_for((dim >> 5) * st->batch, ctx->n_sm), kThreads, 0, ctx->stream>>>(
          st->sup.p, dim >> 5, st->batch, bits);
      CK(cudaGetLastError());
      ctx->launches++;
      st->sup_valid = true;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return FFQ_OK;
  });
}

int ffq_state_upload(ffq_state_t st, const double* psi) {
  if (!st || !psi) return fail(st ? st->ctx : nullptr, FFQ_EINVAL, "null argument");
  return guarded(st->ctx, [&] {
    CK(cudaMemcpyAsync(st->psi.p, psi, sizeof(double2) * ((size_t)st->batch << st->n),
                       cudaMemcpyHostToDevice, st->ctx->stream));
    st->sup_valid = false;
    CK(cudaStreamSynchronize(st->ctx->stream));
    return FFQ_OK;
  });
}

int ffq_state_download(ffq_state_t st, double* psi) {
  if (!st || !psi) return fail(st ? st->ctx : nullptr, FFQ_EINVAL, "null argument");
  return guarded(st->ctx, [&] {
    CK(cudaMemcpyAsync(psi, st->psi.p, sizeof(double2) * ((size_t)st->batch << st->n),
                       cudaMemcpyDeviceToHost, st->ctx->stream));
    CK(cudaStreamSynchronize(st->ctx->stream));
    return FFQ_OK;
  });
}

int ffq_state_apply_pauli_rotation(ffq_state_t st, uint64_t x, uint64_t z, double theta) {
  if (!st) return fail(nullptr, FFQ_EINVAL, "null state");
  ffq_ctx_t ctx = st->ctx;
  if (st->n < 64 && ((x | z) >> st->n)) return fail(ctx, FFQ_EINVAL, "Pauli string exceeds n_qubits");
  return guarded(ctx, [&] {
    std::vector<double2> cs(st->batch, make_double2(std::cos(theta), std::sin(theta)));
    ctx->cs.upload(cs, ctx->stream);
    launch_string(ctx, st->psi.p, st->n, st->batch, x, z, __builtin_popcountll(x & z) & 3, ctx->cs.p,
                  1, 0);
    st->sup_valid = false;  // dense pass: the support is rebuilt lazily
    CK(cudaStreamSynchronize(ctx->stream));
    return FFQ_OK;
  });
}

int ffq_state_apply_pauli_rotations(ffq_state_t st, int n_rot, const uint64_t* x, const uint64_t* z,
                                    const double* theta) {
  if (!st || n_rot < 0 || (n_rot > 0 && (!x || !z || !theta))) return fail(st ? st->ctx : nullptr, FFQ_EINVAL, "null argument");
  ffq_ctx_t ctx = st->ctx;
  for (int r = 0; r < n_rot; ++r)
    if (st->n < 64 && ((x[r] | z[r]) >> st->n)) return fail(ctx, FFQ_EINVAL, "Pauli string exceeds n_qubits");
  return guarded(ctx, [&] {
    if (n_rot == 0) return FFQ_OK;
    if (st->n < 2) throw BadInput("rotation kernels need n_qubits >= 2", FFQ_EINVAL);
    // maximal runs of >= 2 consecutive rotations with flip masks below 2^t
    // are one tiled launch each; every other rotation is one pass
    const int t = ctx->rot_tile_bits > 0 ? std::min(st->n, ctx->rot_tile_bits) : 0;
    std::vector<RotDesc> rd(n_rot);
    std::vector<double2> cs(n_rot);
    std::vector<char> ok(n_rot);
    for (int r = 0; r < n_rot; ++r) {
      rd[r] = RotDesc{0, 0, 0, __builtin_popcountll(x[r] & z[r]) & 3, 0};
      cs[r] = make_double2(std::cos(theta[r]), std::sin(theta[r]));
      ok[r] = 1;
    }
    const RotRuns runs = build_rot_runs(rd, x, z, ok, st->n, t);
    ctx->rot.upload(rd, ctx->stream);
    ctx->rot_groups.upload(runs.groups, ctx->stream);
    ctx->cs.upload(cs, ctx->stream);
    for (int r = 0; r < n_rot;) {
      const int ri = runs.run_at[r];
      if (ri >= 0) {
        launch_rotation_run(ctx, st->psi.p, st->n, st->batch, t, runs.q[ri], ctx->rot_groups.p + runs.g0[ri],
                            runs.ng[ri], ctx->rot.p + r, ctx->cs.p + r, 0);
        r += runs.len[ri];
      } else {
        launch_string(ctx, st->psi.p, st->n, st->batch, x[r], z[r], rd[r].ny, ctx->cs.p, 0, r);
        ++r;
      }
    }
    st->sup_valid = false;
    CK(cudaStreamSynchronize(ctx->stream));
    return FFQ_OK;
  });
}

int ffq_rotation_groups(int n, int t, int n_rot, const uint64_t* x, int32_t* run_of, int32_t* group_of, int32_t* cx,
                        uint64_t* run_q, uint32_t* basis, int32_t* piv, int32_t* n_groups) {
  if (n_rot < 0 || n < 1 || n > 63 || t < 0 || t > 31 ||
      (n_rot > 0 && (!x || !run_of || !group_of || !cx || !run_q || !basis || !piv)) || !n_groups)
    return fail(nullptr, FFQ_EINVAL, "ffq_rotation_groups: invalid argument");
  for (int r = 0; r < n_rot; ++r)  // the same check as ffq_state_apply_pauli_rotations
    if (x[r] >> n) return fail(nullptr, FFQ_EINVAL, "ffq_rotation_groups: flip mask beyond n_qubits");
  std::vector<RotDesc> rd(n_rot, RotDesc{0, 0, 0, 0, 0});
  std::vector<char> ok(n_rot, 1);
  std::vector<uint64_t> z(n_rot, 0);
  const RotRuns R = build_rot_runs(rd, x, z.data(), ok, n, std::min(n, t));
  for (int r = 0; r < n_rot; ++r) {
    run_of[r] = group_of[r] = -1;
    run_q[r] = 0;
  }
  for (int r = 0; r < n_rot; ++r)
    if (R.run_at[r] >= 0)
      for (int q = 0; q < R.len[R.run_at[r]]; ++q) run_q[r + q] = R.q[R.run_at[r]];
  for (int r = 0; r < n_rot; ++r) {
    const int ri = R.run_at[r];
    if (ri < 0) continue;
    for (int g = R.g0[ri]; g < R.g0[ri] + R.ng[ri]; ++g)
      for (int q = R.groups[g].r0; q < R.groups[g].r1; ++q) {
        run_of[r + q] = ri;
        group_of[r + q] = g;
      }
  }
  for (int r = 0; r < n_rot; ++r) cx[r] = group_of[r] >= 0 ? rd[r].cx : 0;
  for (size_t g = 0; g < R.groups.size(); ++g)
    for (int i = 0; i < 3; ++i) {
      basis[3 * g + i] = R.groups[g].b[i];
      piv[3 * g + i] = R.groups[g].piv[i];
    }
  *n_groups = (int32_t)R.groups.size();
  return FFQ_OK;
}

int ffq_state_apply_plan(ffq_state_t st, ffq_plan_t plan, const double* theta) {
  if (!st || !plan || (!theta && plan->cp.n_gen > 0)) return fail(st ? st->ctx : nullptr, FFQ_EINVAL, "null argument");
  ffq_ctx_t ctx = st->ctx;
  if (plan->cp.n_qubits != st->n) return fail(ctx, FFQ_EINVAL, "plan and state qubit counts differ");
  return guarded(ctx, [&] {
    const int ng = plan->cp.n_gen, n_ops = (int)plan->cp.op_kind.size();
    if (n_ops == 0) return FFQ_OK;
    ctx->theta.alloc((size_t)std::max(1, ng) * st->batch);
    CK(cudaMemcpyAsync(ctx->theta.p, theta, sizeof(double) * (size_t)ng * st->batch,
                       cudaMemcpyHostToDevice, ctx->stream));
    ctx->cs.alloc((size_t)n_ops * st->batch);
    launch_cs(ctx, plan, ctx->theta.p, st->batch, ctx->cs.p);
    run_plan_ops(ctx, plan, st->psi.p, state_support(st), st->batch, ctx->cs.p);
    CK(cudaStreamSynchronize(ctx->stream));
    return FFQ_OK;
  });
}

int ffq_state_expectation(ffq_state_t st, ffq_ham_t ham, double* re_out, double* im_out) {
  if (!st || !ham || !re_out) return fail(st ? st->ctx : nullptr, FFQ_EINVAL, "null argument");
  ffq_ctx_t ctx = st->ctx;
  if (ham->ch.n_qubits != st->n) return fail(ctx, FFQ_EINVAL, "Hamiltonian and state qubit counts differ");
  return guarded(ctx, [&] {
    uint32_t* sup = state_support(st);
    const int64_t items = ham->n_partials(sup != nullptr);
    ctx->partial.alloc((size_t)std::max<int64_t>(1, items) * st->batch);
    DevBuf<double> eo;
    eo.alloc(2 * (size_t)st->batch);
    launch_expect(ctx, ham, st->psi.p, sup, st->n, st->batch, ctx->partial.p, eo.p, eo.p + st->batch);
    std::vector<double> host(2 * (size_t)st->batch);
    CK(cudaMemcpyAsync(host.data(), eo.p, sizeof(double) * host.size(), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < st->batch; ++b) {
      re_out[b] = host[b];
      if (im_out) im_out[b] = host[st->batch + b];
    }
    return FFQ_OK;
  });
}

int ffq_state_device_ptr(ffq_state_t st, void** ptr) {
  if (!st || !ptr) return fail(nullptr, FFQ_EINVAL, "null argument");
  *ptr = st->psi.p;
  return FFQ_OK;
}

int ffq_ham_compile_stats(int n_qubits, int64_t n_terms, const uint64_t* x, const uint64_t* z,
                          const double* c_re, const double* c_im, int64_t* stats) {
  if (!stats || (n_terms > 0 && (!x || !z || !c_re || !c_im))) return fail(nullptr, FFQ_EINVAL, "null argument");
  return guarded(nullptr, [&] {
    const CompiledHam H = compile_ham(n_qubits, n_terms, x, z, c_re, c_im);
    int64_t act = 0, visits = 0, cls_evals = 0;
    for (const auto& d : H.groups) {
      act += d.nact;
      const int64_t pairs = (int64_t)d.nact << (n_qubits - d.w);
      visits += pairs;
      cls_evals += pairs * d.ncls;
    }
    stats[0] = (int64_t)H.groups.size();
    stats[1] = H.n_terms;
    stats[2] = H.n_classes();
    stats[3] = act;
    stats[4] = (int64_t)H.item_g.size();
    stats[5] = visits;
    stats[6] = cls_evals;
    stats[7] = visits * 2 * (int64_t)sizeof(double2);
    return FFQ_OK;
  });
}

int ffq_plan_compile_stats(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* x,
                           const uint64_t* z, const double* c_re, const double* c_im,
                           int64_t* stats) {
  if (!stats || (n_gen > 0 && !term_off)) return fail(nullptr, FFQ_EINVAL, "null argument");
  return guarded(nullptr, [&] {
    const CompiledPlan P = compile_plan(n_qubits, n_gen, term_off, x, z, c_re, c_im);
    int64_t pairs = 0, upd = 0, bytes = 0;
    for (const auto& d : P.fused) {
      pairs += d.npair;
      const int64_t u = (int64_t)d.npair << (n_qubits - d.w);
      upd += u;
      bytes += u * 4 * (int64_t)sizeof(double2);
    }
    const int64_t string_bytes = (int64_t)P.n_string_ops() * (32LL << n_qubits);
    stats[0] = P.n_fused();
    stats[1] = P.n_string_ops();
    stats[2] = pairs;
    stats[3] = upd + (int64_t)P.n_string_ops() * (1LL << (n_qubits - 1));
    stats[4] = bytes + string_bytes;
    stats[5] = (int64_t)P.op_kind.size();
    return FFQ_OK;
  });
}

// Host emulation of the one-CTA real program's expectation (generic rows +
// anchored blocks) on a real state psi[2^n]: checks the product layout and
// the block compilation without a GPU. out[8]: energy, closure size, slots,
// product layout, block pairs, expectation pairs, generic rows, block units.
int ffq_sector_emulate(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* px, const uint64_t* pz,
                       const double* pc_re, const double* pc_im, int64_t n_terms, const uint64_t* hx,
                       const uint64_t* hz, const double* hc_re, const double* hc_im, uint64_t hf_bits,
                       const double* psi, double* out) {
  if (!out || !psi || !term_off || n_qubits < 1 || n_qubits > 26) return fail(nullptr, FFQ_EINVAL, "invalid argument");
  return guarded(nullptr, [&] {
    const CompiledPlan P = compile_plan(n_qubits, n_gen, term_off, px, pz, pc_re, pc_im);
    const CompiledHam H = compile_ham(n_qubits, n_terms, hx, hz, hc_re, hc_im);
    if (!plan_is_real(P) || !ham_is_real(H)) return fail(nullptr, FFQ_EINVAL, "ffq_sector_emulate: complex program");
    const char* cqe = std::getenv("FFQ_CLIQUES");
    const SectorProgram S = compile_sector(P, H, hf_bits, kSectorMaxSize, 0xFFFFFFFFu, 1, 0xFFFFFFFFu, 4, 8,
                                           kSectorRealThreads / 32, kSectorSingleMax, !cqe || std::atoi(cqe) != 0);
    if (!S.ok) return fail(nullptr, FFQ_EINVAL, "ffq_sector_emulate: " + S.why);
    // race freedom and bounds by construction (compute-sanitizer is not available
    // on the GPU pool): every generator step's pairs touch distinct amplitude
    // slots (the step's threads then never race; steps are barrier-separated),
    // and every slot a table can address lies in [0, n_slots] (n_slots = zero slot)
    int64_t bad = 0;
    {
      std::vector<int32_t> seen((size_t)S.n_slots + 1, -1);
      const int n_ops = (int)S.op_cross.size();
      for (int op = 0; op < n_ops; ++op)
        for (int64_t t = S.gen_off[op]; t < S.gen_off[op + 1]; ++t) {
          const uint32_t w = S.gen_pairs[t], i = w & 0x7FFFu, j = w >> 16;  // real program: i | j << 16
          if (i >= S.n_slots || j >= S.n_slots || i == j || (w & 0x8000u)) { ++bad; continue; }
          for (uint32_t k : {i, j}) {
            if (seen[k] == op) ++bad;
            seen[k] = op;
          }
        }
      // the head table repeats the first 2 head_threads words of every op (bit 15: more follow)
      const int NT = S.head_threads;
      if (NT <= 0 || S.gen_head.size() != (size_t)(n_ops + kSectorHeadPad) * 2 * NT) ++bad;
      for (int op = 0; NT > 0 && op < n_ops + kSectorHeadPad; ++op)
        for (int t = 0; t < 2 * NT; ++t) {
          const uint32_t hw = S.gen_head[(size_t)2 * op * NT + t];
          const int64_t at = op < n_ops ? S.gen_off[op] + t : -1;
          const bool have = op < n_ops && at < S.gen_off[op + 1];
          const bool more = have && t >= NT && at + NT < S.gen_off[op + 1];
          if (!have ? hw != 0xFFFFFFFFu : hw != (S.gen_pairs[at] | (more ? 1u << 15 : 0u))) ++bad;
        }
      for (uint32_t w : S.row_pairs)
        if ((w & 0x7FFFu) > S.n_slots || ((w >> 15) & 0x7FFFu) > S.n_slots) ++bad;
      for (size_t w = 0; w < S.blk_warp.size() / 4; ++w) {
        // segments: begin <= cut 1 <= cut 2 <= end, whole prefetch rounds each, an anchor row first
        const int32_t* h = &S.blk_warp[4 * w];
        const int32_t edge[kBlkSegments + 1] = {h[0], h[2], h[3], h[1]};
        for (int sg = 0; sg < kBlkSegments; ++sg) {
          if (edge[sg] > edge[sg + 1] || (edge[sg + 1] - edge[sg]) % kStreamQuantum) ++bad;
          if (edge[sg] < edge[sg + 1])
            for (int l = 0; l < 32; ++l)
              if (!(S.blk_stream[(size_t)edge[sg] * 32 + l] >> 30)) ++bad;
        }
        uint32_t bs = 0;
        for (int r = S.blk_warp[4 * w]; r < S.blk_warp[4 * w + 1]; ++r)
          for (int l = 0; l < 32; ++l) {
            const uint32_t d = S.blk_stream[(size_t)r * 32 + l];
            if (d >> 30) {
              bs = (d >> 15) & 0x7FFFu;
              if ((d & 0x7FFFu) > S.n_slots) ++bad;
            } else if (bs + (d & 0x7FFFu) > S.n_slots || (d >> 16) >= S.ftab.size()) {
              ++bad;
            }
          }
      }
      for (size_t l = 0; l < S.cq_desc.size() / 4; ++l) {
        const int32_t* d = &S.cq_desc[4 * l];
        for (int32_t k = d[2]; k < d[3]; ++k)
          for (int i = 0; i < kCliqueMax; ++i) {
            const uint32_t c = ((uint32_t)(i < 4 ? d[0] : d[1]) >> (8 * (i & 3))) & 0xFFu;
            if (c >= S.stride_b || (S.cq_rows[k] & 0x7FFFu) + c >= S.n_slots ||
                ((S.cq_rows[k] >> 15) & 0x7FFFu) + c >= S.n_slots)
              ++bad;
          }
      }
    }
    std::vector<double> amp((size_t)S.n_slots + 1, 0.0);
    for (uint32_t i = 0; i < S.size; ++i) amp[S.slot_of[i]] = psi[S.basis[i]];
    if (!S.eps_flip.empty())  // the expectation tables are in the alpha-first gauge
      for (uint32_t i = 0; i < S.n_slots; ++i)
        if ((S.eps_flip[i / 32] >> (i % 32)) & 1u) amp[i] = -amp[i];
    double e = 0.0;
    const auto& es = S.sections[0];
    for (int r = es.sh0; r < es.pp1; ++r)
      for (int l = 0; l < 32; ++l) {
        const uint32_t w = S.row_pairs[(size_t)r * 32 + l];
        double f = r < es.sh1 ? S.row_fre[r] : S.pf_re[((size_t)(es.pf_base + r - es.sh1)) * 32 + l];
        if (r < es.sh1 && ((w >> 30) & 1u)) f = -f;
        e += f * amp[w & 0x7FFFu] * amp[(w >> 15) & 0x7FFFu];
      }
    const size_t nu = S.blk_units.size() / 8;
    for (size_t w = 0; w < S.blk_warp.size() / 4; ++w) {  // the device's per-warp row streams
      const int32_t* h = &S.blk_warp[4 * w];
      for (int l = 0; l < 32; ++l) {
        double a = 0.0, t = 0.0;
        uint32_t bs = 0;
        for (int r = h[0]; r < h[1]; ++r) {
          const uint32_t d = S.blk_stream[(size_t)r * 32 + l];
          if (d >> 30) {
            e += a * t;
            a = amp.at(d & 0x7FFFu);
            bs = (d >> 15) & 0x7FFFu;
            t = 0.0;
          } else {  // (the device keeps t as two chains, even and odd rows)
            const double f = S.ftab.at(d >> 16);
            t += ((d >> 15) & 1u ? -f : f) * amp.at(bs + (d & 0x7FFFu));
          }
        }
        e += a * t;
      }
    }
    if (!S.cq_warp.empty()) {  // the device's clique phase, same arithmetic
      for (size_t w = 0; w < S.cq_warp.size() / 2; ++w)
        for (int32_t wt = S.cq_warp[2 * w]; wt < S.cq_warp[2 * w + 1]; ++wt)
          for (int l = 0; l < 32; ++l) {
            const int32_t* d = &S.cq_desc[((size_t)wt * 32 + l) * 4];
            uint32_t c[kCliqueMax];
            for (int i = 0; i < 4; ++i) c[i] = ((uint32_t)d[0] >> (8 * i)) & 0xFFu;
            c[4] = (uint32_t)d[1] & 0xFFu;
            c[5] = ((uint32_t)d[1] >> 8) & 0xFFu;
            double acc[kCliquePairs] = {0.0};
            for (int k = d[2]; k < d[3]; ++k) {
              const uint32_t rw = S.cq_rows[k];
              double u[kCliqueMax], v[kCliqueMax];
              for (int i = 0; i < kCliqueMax; ++i) {
                u[i] = amp.at((rw & 0x7FFFu) + c[i]) * ((rw >> 31) ? -1.0 : 1.0);
                v[i] = amp.at(((rw >> 15) & 0x7FFFu) + c[i]);
              }
              for (int jj = 0; jj < kCliqueMax; ++jj)
                for (int i = 0; i < kCliqueMax; ++i)
                  if (i != jj) {
                    const int a = std::min(i, jj), b = std::max(i, jj);
                    const int p = a * (2 * kCliqueMax - a - 1) / 2 + (b - a - 1);
                    acc[p] = std::fma(u[i], v[jj], acc[p]);
                  }
            }
            for (int p = 0; p < kCliquePairs; ++p) e += S.cq_coef[((size_t)wt * kCliquePairs + p) * 32 + l] * acc[p];
          }
    }
    out[0] = e;
    out[1] = S.size;
    out[2] = S.n_slots;
    out[3] = S.product ? 1 : 0;
    out[4] = (double)S.blk_pairs;
    out[5] = (double)S.exp_pair_count;
    out[6] = (double)(es.pp1 - es.sh0);
    out[7] = (double)nu;
    out[8] = (double)S.cq_pairs;
    out[9] = (double)S.cq_conflicts;
    out[10] = (double)bad;
    return FFQ_OK;
  });
}

}  // extern "C"

#include "ffq_shard.inl"
#include "ffq_krylov.inl"
#include "ffq_multi.inl"
