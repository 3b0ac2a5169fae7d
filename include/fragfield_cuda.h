/*
 * fragfield_cuda.h -- C-ABI of the B200 UCCSD state-vector hot path
 * (libfragfield_cuda.so). Plain pointers and sizes only; no torch/CUDA types.
 *
 * The reference (fragfield, /root/reference/proj) has no code or FFI for this
 * path: its simulator / vqe-uccsd modules exist only as SPEC contracts. Each
 * entry point below names the SPEC operation it replaces, so a maintainer can
 * bind it from the reference's C++ side:
 *
 *   ffq_state_set_basis            hf_state
 *   ffq_state_apply_pauli_rotation apply_pauli_rotation
 *   ffq_state_apply_pauli_rotations apply_pauli_rotation over a string list
 *                                  (Trotter step)
 *   ffq_state_expectation          expectation
 *   ffq_plan_upload                TrotterPlan
 *   ffq_state_apply_plan           energy_trotter (state) SPEC.md:508-516
 *   ffq_energy_batch               energy_trotter, batched over amplitude
 *                                  vectors (VQE objective / gradient sets /
 *                                  FMO fragments)
 *
 * Conventions: a Pauli string is a pair of bitmasks
 * (x, z) over qubits, qubit 0 = least-significant bit of the amplitude index;
 * letter X where only x is set, Z where only z is set, Y where both are set;
 * the string carries no phase (phase lives in the coefficient). State vectors
 * are complex128, interleaved (re, im), natural binary order, laid out
 * [batch][2^n].
 *
 * Errors: every call returns FFQ_OK (0) or a negative code; ffq_last_error()
 * returns a message. The C++ facade maps FFQ_EINVAL / FFQ_ENONHERMITIAN to
 * fragfield::ContractViolation (errors.hpp convention of the reference,
 * proj/core/include/fragfield/errors.hpp:23-25) and the rest to
 * std::runtime_error.
 *
 * Threading: one context per device, bound to one CUDA stream; a context is
 * not re-entrant. Distinct contexts may be driven from different host threads.
 * Determinism: energies are bitwise identical for any batch split or device
 * count (fixed work decomposition and fixed-shape reduction trees).
 */
#ifndef FRAGFIELD_CUDA_H
#define FRAGFIELD_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFQ_OK 0
#define FFQ_EINVAL (-1)
#define FFQ_ENONHERMITIAN (-2)
#define FFQ_ECUDA (-3)
#define FFQ_ENOMEM (-4)
#define FFQ_ENCCL (-5)
#define FFQ_ENODEV (-6)

typedef struct ffq_ctx_s* ffq_ctx_t;
typedef struct ffq_ham_s* ffq_ham_t;
typedef struct ffq_plan_s* ffq_plan_t;
typedef struct ffq_state_s* ffq_state_t;
typedef struct ffq_multi_s* ffq_multi_t;

/* ---- library / context ---------------------------------------------------- */
int ffq_version(void);
int ffq_device_count(int* n_out);
int ffq_ctx_create(int device, ffq_ctx_t* out);
int ffq_ctx_destroy(ffq_ctx_t ctx);
int ffq_ctx_synchronize(ffq_ctx_t ctx);
/* Message of the last failing call on this context (ctx == NULL: last failing
 * call on this host thread). Never NULL. */
const char* ffq_last_error(ffq_ctx_t ctx);
/* Number of kernels this context has launched so far (graph nodes counted). */
int64_t ffq_ctx_kernel_launches(ffq_ctx_t ctx);
/* The context's cudaStream_t, as an opaque pointer (for event timing). */
int ffq_ctx_stream(ffq_ctx_t ctx, void** stream);
/* Environment, read at ffq_ctx_create (tuning and diagnostics only; every
 * setting gives the same energies to <= 1e-12):
 *   FFQ_SECTOR (1)          support-closure evaluator first; 0 disables it
 *   FFQ_SECTOR_REAL (1)     real-amplitude one-CTA evaluator when psi is real; 0 off
 *   FFQ_SECTOR_CL (2)       CTAs per cluster for large complex closures: 2, 4 or 8
 *   FFQ_SMEM_MAX_QUBITS (13) largest state held whole in one CTA's smem
 *   FFQ_SUPPORT (1)         support-bitmap passes on the global-memory path
 *   FFQ_SLAB_MB (256)       state slab per chunk of the global path
 *   FFQ_BLOCKS (1)          anchored string blocks of the real sector program; 0 off
 *   FFQ_CLIQUES (1)         alpha-beta cliques of the real sector program; 0 off
 *   FFQ_SPLIT (16)          most CTAs per evaluation of small real-program batches
 *   FFQ_COMPACT (1), FFQ_COMPACT_MIN (27)  compact real sector layout, from n qubits
 *   FFQ_ROT_TILE (12)       tile bits of fused rotation runs; 0: one pass per rotation
 *   FFQ_PHASE_CLOCKS        print per-phase cycle counts (read once per process) */

/* ---- qubit Hamiltonian (PauliSum) ------------------------ */
/* Flat Pauli sum, any order; duplicate strings are summed. The library groups
 * the terms by flip mask x. Non-Hermitian input (|Im c| > 1e-12) is rejected
 * with FFQ_ENONHERMITIAN. */
int ffq_ham_upload(ffq_ctx_t ctx, int n_qubits, int64_t n_terms, const uint64_t* x,
                   const uint64_t* z, const double* c_re, const double* c_im, ffq_ham_t* out);
int ffq_ham_destroy(ffq_ham_t ham);
/* n_groups = distinct flip masks; n_classes = (group, z outside the flip
 * mask) classes the kernels evaluate per amplitude. */
int ffq_ham_info(ffq_ham_t ham, int* n_groups, int64_t* n_terms, int64_t* n_classes);

/* ---- Trotter plan (TrotterPlan) -------------------------- */
/* n_gen generators in EXECUTION order. Generator g is the anti-Hermitian Pauli
 * sum sum_j (c_re + i c_im)_j P_j over terms [term_off[g], term_off[g+1]),
 * normally the JW image of tau - tau^dag; it is applied as exp(theta_g * A_g)
 * (equivalently prod_j e^{i theta_g c_j P_j} in canonical term order,
 * SPEC.md:511). Real parts must vanish (|c_re| <= 1e-12) -> else FFQ_EINVAL.
 * Generators whose strings share one flip mask and commute are fused into one
 * exact rotation pass; any other generator runs string by string. */
int ffq_plan_upload(ffq_ctx_t ctx, int n_qubits, int n_gen, const int64_t* term_off,
                    const uint64_t* x, const uint64_t* z, const double* c_re,
                    const double* c_im, ffq_plan_t* out);
int ffq_plan_destroy(ffq_plan_t plan);
int ffq_plan_info(ffq_plan_t plan, int* n_fused, int* n_string_ops);

/* ---- batched energy (energy_trotter) --------------------- */
/* e_out[b] = <psi_b|H|psi_b>, psi_b = prod_g exp(theta[b][g] A_g) |hf_bits>.
 * theta is [batch][n_gen] in plan order. Host pointers; the call returns when
 * e_out is written. Imaginary residue above 1e-10 -> FFQ_ENONHERMITIAN. */
int ffq_energy_batch(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits,
                     int batch, const double* theta, double* e_out);
/* Same with device pointers (inputs resident in HBM); asynchronous on the
 * context stream; imag_dev (optional, [batch]) receives imaginary residues. */
int ffq_energy_batch_device(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits,
                            int batch, const double* theta_dev, double* e_dev,
                            double* imag_dev);
/* Compile and cache the program ffq_energy_batch(_device) runs for (plan, ham,
 * hf_bits) -- the support-closure program, or the compact sector lists from 22
 * qubits up -- without evaluating anything (otherwise compiled on the first
 * energy call: ~1-2 s of host work at 18 qubits). The one entry point that is
 * re-entrant per context: host threads may call it concurrently for DISTINCT
 * plans of one context (the VQE driver of SPEC.md:566 compiles its fragments in
 * parallel before the serial optimiser loops). */
int ffq_energy_prepare(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits);
/* Support-closure program that ffq_energy_batch(_device) runs for (plan, ham,
 * hf_bits) (compiled on first use and cached): out[0] closure size |S|,
 * out[1] CTAs per evaluation, out[2] generator pairs, out[3] expectation
 * pairs, out[4] expectation rows of 32, out[5] generator steps ending in a
 * cluster barrier, out[6] first split mask, out[7] peer-chunk buffer
 * (amplitudes), out[8] 1 when the program stores real amplitudes only (real F
 * on every generator and real class sums: psi(theta) is real for every theta),
 * out[9] expectation pairs held by anchored string blocks (product layout),
 * out[10] amplitude slots (padded product layout; = out[0] otherwise),
 * out[11] expectation pairs held by alpha-beta cliques, out[12] clique warp
 * tasks, out[13] modelled extra shared wavefronts per clique row (bank
 * conflicts summed over half-warp tasks; 0 = conflict-free), out[14] clique
 * lane-rows (12 amplitude loads each).
 * out must hold 15 values.
 * FFQ_EINVAL when the closure does not fit the sector evaluator (the other
 * paths then run) or FFQ_SECTOR=0. */
int ffq_sector_info(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, int64_t* out);
/* Amplitude-level view of the 1024-thread real-amplitude sector program (the
 * 18-qubit default): runs one evaluation of theta[n_gen] (plan order) and
 * returns the state after the plan, scattered from its product-layout slots to
 * natural order, in psi[2^n][2] (re, im; im = 0: the program holds psi's real
 * parts, which is all of psi), plus the energy of the same launch in *energy
 * (may be NULL). Replaces the state-dump side of energy_trotter (SPEC.md:459,
 * 508-516) for the sector program. FFQ_EINVAL when that program does not run
 * for these inputs. */
int ffq_sector_state(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits, const double* theta,
                     double* psi, double* energy);

/* ---- state-level operations (simulator) ------------------ */
int ffq_state_alloc(ffq_ctx_t ctx, int n_qubits, int batch, ffq_state_t* out);
int ffq_state_free(ffq_state_t st);
int ffq_state_set_basis(ffq_state_t st, uint64_t bits);
int ffq_state_upload(ffq_state_t st, const double* psi);   /* [batch][2^n][2] */
int ffq_state_download(ffq_state_t st, double* psi);       /* [batch][2^n][2] */
/* psi <- cos(theta) psi + i sin(theta) P psi  (e^{i theta P}), every batch row */
int ffq_state_apply_pauli_rotation(ffq_state_t st, uint64_t x, uint64_t z, double theta);
/* The sequence e^{i theta[n_rot-1] P_{n_rot-1}} ... e^{i theta[0] P_0}, in order
 * (apply_pauli_rotation over a Trotter string list).
 * Runs of consecutive rotations whose flip masks, with the low 5 qubits, lie in
 * 12 qubits go through one shared-memory tile pass each (TMA-staged when those
 * are the low 12; FFQ_ROT_TILE). */
int ffq_state_apply_pauli_rotations(ffq_state_t st, int n_rot, const uint64_t* x, const uint64_t* z,
                                    const double* theta);
/* Host only (no device work): how ffq_state_apply_pauli_rotations cuts a list
 * of flip masks on n qubits for tile bits t (min(n, t) used). run_of/group_of/
 * cx [n_rot]: run and group of each rotation (-1 when it is a single pass) and
 * its flip mask's coordinates in its group's basis (tile coordinates = pext by
 * the run's qubit set run_q [n_rot]); basis/piv [n_rot * 3] (first 3 * n_groups
 * used). */
int ffq_rotation_groups(int n, int t, int n_rot, const uint64_t* x, int32_t* run_of, int32_t* group_of, int32_t* cx,
                        uint64_t* run_q, uint32_t* basis, int32_t* piv, int32_t* n_groups);
/* Apply the plan with theta [batch][n_gen] (host pointer). */
int ffq_state_apply_plan(ffq_state_t st, ffq_plan_t plan, const double* theta);
/* re_out/im_out [batch] (host) */
int ffq_state_expectation(ffq_state_t st, ffq_ham_t ham, double* re_out, double* im_out);
/* Device pointer to the amplitudes (for zero-copy interop in tests/bench). */
int ffq_state_device_ptr(ffq_state_t st, void** ptr);

/* ---- sharded state (global qubits; BASELINE.json config 5) ----------------- */
/* A state of n qubits split on n_global physical qubits over R = 2^n_global
 * ranks. ffq_shard_create keeps all R shards on this context's device
 * (exchanges are device-side swaps); ffq_shard_create_nccl holds one rank's
 * shard per process and exchanges half shards over NCCL (ncclSend/ncclRecv)
 * for global-qubit swaps and whole shards per out-of-shard flip pattern in the
 * expectation; per-rank partial energies are all-gathered and summed in rank
 * order. */
typedef struct ffq_shard_s* ffq_shard_t;
int ffq_shard_create(ffq_ctx_t ctx, int n_qubits, int n_global, ffq_shard_t* out);
int ffq_nccl_unique_id(void* id128); /* ncclUniqueId bytes (128) from rank 0 */
int ffq_shard_create_nccl(ffq_ctx_t ctx, int n_qubits, int n_global, int rank, const void* id128,
                          ffq_shard_t* out);
int ffq_shard_destroy(ffq_shard_t sh);
/* One energy evaluation; theta [n_gen] in plan order (host), e_out on every rank. */
int ffq_shard_energy(ffq_shard_t sh, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits,
                     const double* theta, double* e_out);
/* Group mode only: the full state in LOGICAL order [2^n][2] after the last evaluation. */
int ffq_shard_download(ffq_shard_t sh, double* psi);
/* Swaps performed by the last evaluation and the current logical->physical map [n]. */
int ffq_shard_info(ffq_shard_t sh, int* last_swaps, int* perm);
/* Host-only: the swap schedule a plan gets (initial/final permutation, swaps). */
int ffq_shard_schedule(int n_qubits, int n_global, int n_gen, const int64_t* term_off,
                       const uint64_t* x, const uint64_t* z, const double* c_re, const double* c_im,
                       int* init_perm, int* final_perm, int* n_swaps, int* n_steps);
/* Same, plus the step list steps[4 * i] = {kind (0 swap, 1 apply), physical
 * global position, local position, generator column} for i < n_steps. */
int ffq_shard_schedule_steps(int n_qubits, int n_global, int n_gen, const int64_t* term_off,
                             const uint64_t* x, const uint64_t* z, const double* c_re,
                             const double* c_im, int* init_perm, int* final_perm, int* n_swaps,
                             int* n_steps, int* steps, int max_steps);

/* ---- exact references -------------------------- */
/* Ground energy of H in the Krylov space of |hf_bits> (CAS-CI in the HF
 * particle/spin sector): Lanczos with full reorthogonalisation, converged when
 * the lowest Ritz value moves by <= tol between iterations (lanczos_ground). */
int ffq_lanczos_ground(ffq_ctx_t ctx, ffq_ham_t ham, uint64_t hf_bits, double tol, int max_iter,
                       double* e0, int* iters, int* dim);
/* Trotter-free UCCSD energy <hf| e^{-A} H e^{A} |hf>, A = sum_g theta_g A_g
 * (energy_exact via apply_exp_antihermitian: Taylor series of sparse
 * matrix-vector products, remainder norm <= tol, at most 200 terms). */
int ffq_energy_exact(ffq_ctx_t ctx, ffq_plan_t plan, ffq_ham_t ham, uint64_t hf_bits,
                     const double* theta, double tol, double* e_out);

/* ---- host-only diagnostics (no device needed) ----------------------------- */
/* Compile a Hamiltonian / plan exactly as the upload calls do and report the
 * table shapes. ham stats[8]: groups, terms, classes, active patterns,
 * work items, pair visits per evaluation, class evaluations per evaluation,
 * amplitude bytes read per evaluation. plan stats[6]: fused ops, string ops,
 * active pattern pairs, pair updates per evaluation, bytes moved per
 * evaluation (read+write), ops. */
int ffq_ham_compile_stats(int n_qubits, int64_t n_terms, const uint64_t* x, const uint64_t* z,
                          const double* c_re, const double* c_im, int64_t* stats);
int ffq_plan_compile_stats(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* x,
                           const uint64_t* z, const double* c_re, const double* c_im,
                           int64_t* stats);
/* Test hook (host only, no GPU): compiles the one-CTA real-amplitude sector
 * program (product layout, anchored string blocks) for plan + Hamiltonian +
 * hf and evaluates its expectation tables on the real state psi[2^n] exactly
 * as k_sector_eval_real would (generic rows, blocks, then the alpha-beta
 * cliques in the alpha-first gauge). out[11]: energy, closure size, amplitude
 * slots, product layout (0/1), pairs held by blocks, expectation pairs,
 * generic rows, block units, pairs held by cliques, modelled clique bank
 * conflicts, and table violations: generator steps whose pairs share a slot
 * (a race) or any table slot outside [0, n_slots] (0 = race-free and in
 * bounds by construction). FFQ_CLIQUES=0 compiles without cliques.
 * FFQ_EINVAL when the program is complex or has no sector. */
int ffq_sector_emulate(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* px, const uint64_t* pz,
                       const double* pc_re, const double* pc_im, int64_t n_terms, const uint64_t* hx,
                       const uint64_t* hz, const double* hc_re, const double* hc_im, uint64_t hf_bits,
                       const double* psi, double* out);

/* Test hook (host only, no GPU): compiles the compact real sector program
 * (csrc/ffq_compact.inl: row / column lists per generator, Pauli-term groups)
 * for plan + Hamiltonian + hf and evaluates one theta row (plan order) on the
 * host from the same lists, with the kernels' pair arithmetic. out[8]: energy,
 * eligible (0/1: even n, <= 16 spatial orbitals, real spin-conserving fused
 * plan), alpha strings, beta strings, generator pairs, term pairs, list
 * violations (an index out of bounds, or a row / column list of one op touching
 * an index twice: 0 = in bounds and race-free by construction), term groups. */
int ffq_compact_emulate(int n_qubits, int n_gen, const int64_t* term_off, const uint64_t* px, const uint64_t* pz,
                        const double* pc_re, const double* pc_im, int64_t n_terms, const uint64_t* hx,
                        const uint64_t* hz, const double* hc_re, const double* hc_im, uint64_t hf_bits,
                        const double* theta, double* out);

/* ---- multi-GPU, independent units (BASELINE configs 2-4) ---- */
/* One context per device of `devices` (one node); every call runs one host
 * thread per device, with no data-path collective: the units (theta rows,
 * fragments) are independent, and a row's energy is bitwise the same on any
 * device and in any batch, so results equal the one-device call bit for bit
 * (SPEC.md:455-457 worker-count independence). Replaces the fragment driver's
 * concurrent per-fragment VQE evaluations (`--jobs` :621) that
 * feed FMOEnergyLedger (proj/core/src/fmo.cpp:46-48). */
int ffq_multi_create(const int* devices, int n_dev, ffq_multi_t* out);
int ffq_multi_destroy(ffq_multi_t m);
int ffq_multi_device_count(ffq_multi_t m, int* n_dev);
const char* ffq_multi_last_error(ffq_multi_t m);
/* Plan (as ffq_plan_upload) + Hamiltonian (as ffq_ham_upload) uploaded to
 * every device; *problem_out = its id for the calls below. */
int ffq_multi_problem_upload(ffq_multi_t m, int n_qubits, int n_gen, const int64_t* term_off,
                             const uint64_t* px, const uint64_t* pz, const double* pc_re,
                             const double* pc_im, int64_t n_terms, const uint64_t* hx,
                             const uint64_t* hz, const double* hc_re, const double* hc_im,
                             int* problem_out);
/* ffq_energy_batch over all devices: rows split into contiguous blocks
 * (sizes differ by at most one), written back in row order. */
int ffq_multi_energy_batch(ffq_multi_t m, int problem, uint64_t hf_bits, int batch,
                           const double* theta, double* e_out);
/* n_units independent units (problem[u], hf_bits[u], batch[u] rows of
 * theta[u] -> e_out[u]), e.g. FMO monomers and dimers with their gradient
 * sets, assigned to devices longest-first by cost 2^n x (generators + flip-
 * mask groups) x rows; device_out[u] (optional) receives the assignment. */
int ffq_multi_energy_units(ffq_multi_t m, int n_units, const int* problem, const uint64_t* hf_bits,
                           const int* batch, const double* const* theta, double* const* e_out,
                           int* device_out);

#ifdef __cplusplus
}
#endif
#endif /* FRAGFIELD_CUDA_H */
