/*
 * ffo_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * This library is the checker for the B200 hot path, never the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.
 *
 * It restates, in plain C with per-qubit loops, the contracts of the
 * reference's SPEC for the path (the reference repo has no code for it; see
 * SURVEY.md section 0):
 *   qubit-map   /root/reference/SPEC.md:325-388  (Pauli algebra, Jordan-Wigner)
 *   simulator   /root/reference/SPEC.md:390-465  (hf_state, e^{i theta P}, <H>)
 *   vqe-uccsd   /root/reference/SPEC.md:467-576  (generators, magnitude order,
 *                                                 energy_trotter)
 *   hamiltonian /root/reference/SPEC.md:261-323  (interleaved spin orbitals)
 * plus the synthetic-integral recipe of BASELINE.json configs (pinned in
 * DESIGN.md section "Synthetic inputs").
 *
 * Parity status: the reference holds no golden vectors for this path, so the
 * oracle is pinned by (i) the SPEC examples (KATs), (ii) dense numpy/scipy
 * matrices at <= 10 qubits, (iii) a second, Jordan-Wigner-free fermionic
 * evaluator inside this file, and (iv) the C++ standard's mt19937_64 KAT.
 * DESIGN.md records this as "pinned to SPEC KATs + dense oracles; no
 * reference golden vectors exist".
 */
#ifndef FFO_ORACLE_H
#define FFO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (mt19937_64, raw output; mapping pinned in DESIGN.md) ---------- */
uint64_t ffo_mt64_nth(uint64_t seed, int nth);
void ffo_uniform_array(uint64_t seed, int count, double lo, double hi, double* out);
/* h: m*m row-major symmetric; g: m^4 chemists' (pq|rs), index ((p*m+q)*m+r)*m+s */
void ffo_synthetic_integrals(int m, uint64_t seed, double sigma_h, double sigma_g,
                             double* h, double* g);

/* ---- Pauli algebra ------------------------------------------------------ */
/* Product P1*P2 = i^k P3 (phase-free strings). Returns k in 0..3. */
int ffo_pauli_mul(int n, uint64_t x1, uint64_t z1, uint64_t x2, uint64_t z2,
                  uint64_t* x3, uint64_t* z3);

typedef struct ffo_psum ffo_psum;
ffo_psum* ffo_psum_new(int n_qubits);
void ffo_psum_free(ffo_psum* s);
int ffo_psum_size(const ffo_psum* s);
int ffo_psum_nqubits(const ffo_psum* s);
void ffo_psum_get(const ffo_psum* s, uint64_t* x, uint64_t* z, double* cr, double* ci);
ffo_psum* ffo_psum_from_arrays(int n, int count, const uint64_t* x, const uint64_t* z,
                               const double* cr, const double* ci);
/* Jordan-Wigner image of coef * prod_k op_k, op_k = a^dag_{idx[k]} if dag[k]
 * else a_{idx[k]}; product applied right-to-left as written (leftmost is
 * outermost). Accumulated into s (not simplified until ffo_psum_simplify). */
void ffo_jw_add_product(ffo_psum* s, int n_ops, const int* idx, const int* dag,
                        double cr, double ci);
void ffo_psum_simplify(ffo_psum* s);

/* Spin-orbital Hamiltonian (interleaved alpha/beta) of spatial
 * integrals, JW-mapped and simplified. */
ffo_psum* ffo_hamiltonian_jw(int m, const double* h, const double* g, double e_const);

/* ---- UCCSD generators --------------------------------------------------- */
/* Writes kind[k] (1 single, 2 double) and idx[4k..4k+3] = (i, j, a, b)
 * (singles use (i, -1, a, -1)); returns the count. Pass NULL to count. */
int ffo_build_generators(int n_so, int n_e, int* kind, int* idx);
ffo_psum* ffo_generator_image(int n_so, int kind, const int* idx4);
void ffo_magnitude_order(int n_gen, const double* amps, int* order);

/* ---- state vector ------------------------------------------------------- */
/* psi is interleaved complex128: psi[2k] = Re, psi[2k+1] = Im */
void ffo_set_threads(int n);
int ffo_get_threads(void);
void ffo_hf_state(int n, uint64_t occ_bits, double* psi);
void ffo_apply_pauli_rotation(int n, double* psi, uint64_t x, uint64_t z, double theta);
void ffo_expectation(int n, const double* psi, const ffo_psum* H, double* re, double* im);

/* energy_trotter: amps indexed by canonical generator id,
 * plan = execution order of generator ids. psi_out (optional) receives the
 * final state. Returns <H> real part; *im_out the imaginary residue. */
double ffo_energy_trotter(int n_so, int n_e, int n_gen, const int* kind, const int* idx,
                          const int* plan, const double* amps, const ffo_psum* H,
                          double* psi_out, double* im_out);

/* Same energy computed without Jordan-Wigner: fermionic Givens rotations on
 * determinants and <H> from second-quantised h/g. Independent cross-check. */
double ffo_energy_fermionic(int m, int n_e, const double* h, const double* g, double e_const,
                            int n_gen, const int* kind, const int* idx, const int* plan,
                            const double* amps, double* psi_out);

/* FMO two-body assembly, fmo.cpp:28-43: sum dimers - (N_f - 2) sum monomers */
double ffo_fmo_assemble(int n_fragments, int n_mono, const double* mono, int n_dim,
                        const double* dim);

#ifdef __cplusplus
}
#endif
#endif
