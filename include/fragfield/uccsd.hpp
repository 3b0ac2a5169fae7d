// fragfield/uccsd.hpp -- UCCSD generators and magnitude-ordered Trotter plans
// (SPEC.md:467-576).
#pragma once

#include <cstdint>
#include <vector>

#include "fragfield/pauli.hpp"

namespace fragfield {

/// One excitation: kind 1 = single (i -> a), kind 2 = double (i<j -> a<b).
/// tau_single = a+_a a_i, tau_double = a+_a a+_b a_j a_i.
struct Excitation {
  int kind = 0;
  int i = -1, j = -1, a = -1, b = -1;
};

/// A generator is t * (tau - tau^dag); `image` is the JW image of
/// (tau - tau^dag) for t = 1 (anti-Hermitian).
struct Generator {
  int id = 0;  // canonical id
  Excitation exc;
  PauliSum image;
};

/// All spin-conserving singles and doubles of n_elec electrons in the lowest
/// spin orbitals. Canonical id order: singles (i, a), then doubles (i, j, a, b).
std::vector<Generator> build_generators(int n_so, int n_elec);

/// generator ids in execution order, frozen after build.
struct TrotterPlan {
  int n_qubits = 0;
  std::vector<int> order;            // canonical generator ids, execution order
  std::vector<Generator> generators;  // indexed by canonical id
  /// theta in plan order from amplitudes indexed by canonical id
  std::vector<double> plan_theta(const std::vector<double>& amps) const;
  /// flat C-ABI arrays (term_off + terms), generators in execution order
  void flatten(std::vector<int64_t>& off, std::vector<uint64_t>& x, std::vector<uint64_t>& z,
               std::vector<double>& re, std::vector<double>& im) const;
};

/// Descending |t|, ties by canonical id.
TrotterPlan magnitude_order(const std::vector<Generator>& gens, const std::vector<double>& amps,
                            int n_qubits);

/// |HF> bits: lowest n_elec spin orbitals occupied.
uint64_t hf_bits(int n_elec);

}  // namespace fragfield
