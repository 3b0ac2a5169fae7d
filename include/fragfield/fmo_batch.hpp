// fragfield/fmo_batch.hpp -- FMO fragment batches feeding the two-body energy
// assembly of the reference (proj/core/include/fragfield/fmo.hpp:41-55,
// proj/core/src/fmo.cpp:28-48): per-fragment VQE-UCCSD energies go into the
// ledger's corr_I / corr_IJ maps and are assembled with
//   E = sum_{I>J} E_IJ - (N_f - 2) sum_I E_I,
// algebraically the FMO2 sum  sum_I E_I + sum_{I>J} (E_IJ - E_I - E_J).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "fragfield/pauli.hpp"
#include "fragfield/uccsd.hpp"

namespace fragfield {

class Device;
class DevicePlan;
class DeviceHamiltonian;

/// Label-keyed component maps, std::map order (deterministic summation).
struct FragmentLedger {
  int n_fragments = 0;
  std::map<std::string, double> corr_I;   // "1", "2", ...
  std::map<std::string, double> corr_IJ;  // "21", "31", ...
  double assemble_corr() const;
};

/// Throws ContractViolation on a missing monomer or dimer entry (fmo.cpp:30-37).
double assemble_two_body(int n_fragments, const std::map<std::string, double>& monomers,
                         const std::map<std::string, double>& dimers);

/// Dimer labels in the reference's fragment_pairs order: "JI" with J > I
/// (proj/core/src/chem.cpp:146-151).
std::vector<std::string> dimer_labels(int n_fragments);

/// One FMO unit (monomer "I" or dimer "JI") as a VQE-UCCSD energy problem.
struct FragmentProblem {
  std::string label;
  PauliSum hamiltonian;
  TrotterPlan plan;
  uint64_t hf = 0;
  std::vector<double> amplitudes;  // canonical generator order
  double e_reference = 0.0;        // subtracted to give a correlation energy (0: total)
};

/// Relative device cost of one energy evaluation: 2^n (generators + x-groups).
double fragment_cost(const FragmentProblem& f);

/// Longest-processing-time assignment of units to `world` ranks by cost; ties
/// by input order. Returns rank per unit (deterministic).
std::vector<int> shard_by_cost(const std::vector<double>& costs, int world);

/// Uploads and evaluates this rank's share of the fragments on one device;
/// returns label -> energy for the evaluated units only.
std::map<std::string, double> evaluate_fragments(Device& dev, const std::vector<FragmentProblem>& frags,
                                                 int rank = 0, int world = 1);

/// Fills a FragmentLedger (corr_I for 1-digit labels, corr_IJ otherwise) and
/// assembles it; throws ContractViolation if a unit is missing.
double assemble_fragments(int n_fragments, const std::map<std::string, double>& energies,
                          FragmentLedger* ledger = nullptr);

}  // namespace fragfield
