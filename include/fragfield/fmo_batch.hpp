// fragfield/fmo_batch.hpp -- FMO fragment batches feeding the two-body energy
// assembly of the reference (proj/core/include/fragfield/fmo.hpp:41-55,
// proj/core/src/fmo.cpp:28-48): per-fragment VQE-UCCSD energies go into the
// ledger's corr_I / corr_IJ maps and are assembled with
//   E = sum_{I>J} E_IJ - (N_f - 2) sum_I E_I,
// algebraically the FMO2 sum  sum_I E_I + sum_{I>J} (E_IJ - E_I - E_J).
#pragma once

#include <map>
#include <string>
#include <vector>

namespace fragfield {

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

}  // namespace fragfield
