// fragfield/hamiltonian.hpp -- spin-orbital Hamiltonians
// and the seeded synthetic inputs of BASELINE.json's configs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "fragfield/pauli.hpp"

namespace fragfield {

/// Spatial-orbital integrals: h (m x m, symmetric) and chemists' (pq|rs)
/// stored at ((p*m+q)*m+r)*m+s with 8-fold symmetry.
struct SpatialIntegrals {
  int m = 0;
  std::vector<double> h, g;
  double e_const = 0.0;
};

/// SPEC.md:266-270, interleaved ordering: spin orbital 2P is
/// alpha of spatial P, 2P+1 is beta.
///   H = sum h_pq a+_p a_q + 1/2 sum g_pqrs a+_p a+_q a_s a_r + E_const,
///   g_pqrs = (PR|QS) delta(sigma_p, sigma_r) delta(sigma_q, sigma_s).
struct SpinOrbitalHamiltonian {
  int n_so = 0;
  int n_elec = 0;
  std::vector<double> h;  // n_so^2
  std::vector<double> g;  // n_so^4, physicists' order [p][q][r][s]
  double e_const = 0.0;
};

/// Seeded synthetic integrals (BASELINE.json configs): h ~ N(0, sigma_h),
/// (pq|rs) ~ N(0, sigma_g); std::mt19937_64 raw output, U = (x>>11)*2^-53,
/// Box-Muller cosine branch, canonical quadruple loop -- see DESIGN.md.
SpatialIntegrals synthetic_integrals(int m, uint64_t seed, double sigma_h = 1.0,
                                     double sigma_g = 0.1);
SpinOrbitalHamiltonian to_spin_orbitals(const SpatialIntegrals& ints, int n_elec);
/// JW image of the spin-orbital Hamiltonian.
PauliSum qubit_hamiltonian(const SpinOrbitalHamiltonian& H);
/// Config 5: n_terms seeded random {I,X,Y,Z}^n strings, real c ~ N(0, sigma).
PauliSum random_pauli_hamiltonian(int n_qubits, int n_terms, uint64_t seed, double sigma = 0.1);

/// FCIDUMP interchange: spatial orbitals, chemists' (ij|kl)
/// with 8-fold symmetry written once (i >= j, k >= l, ij >= kl, 1-based),
/// then h_ij (i >= j) as "v i j 0 0", then E_const as "v 0 0 0 0"; zero
/// values are omitted; values at 17 significant digits (lossless round trip).
struct Fcidump {
  SpatialIntegrals ints;
  int n_elec = 0;
  int ms2 = 0;
};
void write_fcidump(const std::string& path, const SpatialIntegrals& ints, int n_elec, int ms2 = 0);
/// Throws ParseError (with the line number) on a malformed file.
Fcidump read_fcidump(const std::string& path);

/// AO -> MO transformation: h_mo = C^T (h_ao + V_esp) C and
/// (pq|rs)_mo = sum C_mp C_nq C_lr C_ss' (mn|ls')_ao as four quarter
/// transformations, O(N^5). ao: n AO functions (h n x n, g n^4 chemists'
/// order, v_esp n x n or empty: the embedding operator folded into the
/// one-electron part); C: n x m row-major, column j = MO j. e_const is kept.
SpatialIntegrals ao_to_mo(const SpatialIntegrals& ao, const std::vector<double>& C, int m,
                          const std::vector<double>& v_esp = {});

/// Frozen-core contraction of the n_frozen lowest MOs (the
/// first n_frozen, orbitals in energy order):
///   h_eff_pq = h_pq + sum_c [2 (pq|cc) - (pc|cq)],
///   E_frozen = sum_c 2 h_cc + sum_cd [2 (cc|dd) - (cd|dc)],
/// active integrals over MOs n_frozen .. m-1, e_const += E_frozen, and the
/// active electron count n_elec - 2 n_frozen. ContractViolation when
/// n_frozen exceeds the occupied orbitals (n_elec / 2) or is negative.
struct FrozenCore {
  SpatialIntegrals active;  // e_const includes E_frozen
  double e_frozen = 0.0;
  int n_elec_active = 0;
};
FrozenCore freeze_core(const SpatialIntegrals& mo, int n_frozen, int n_elec);

/// Uniform draws U(lo, hi) from mt19937_64(seed), same value mapping.
std::vector<double> uniform_vector(uint64_t seed, int count, double lo, double hi);

}  // namespace fragfield
