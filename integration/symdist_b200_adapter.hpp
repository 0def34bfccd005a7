// Declarations of the reference-side adapter (symdist_b200_adapter.cpp). With
// SYMDIST_USE_B200 defined, the reference's distance.cpp forwards its entry points here
// (INTEGRATION.md shows the one-line switch).
#pragma once

#include "symdist/distance.hpp"

namespace symdist {

DistanceReport saved_isometry_b200(const StabilizerInstance &inst, const RunOptions &opts = {});
DistanceReport saved_1_gamma_b200(const StabilizerInstance &inst, const RunOptions &opts = {});
DistanceReport saved_2_gamma_b200(const StabilizerInstance &inst, const RunOptions &opts = {});
DistanceReport compute_distance_b200(const StabilizerInstance &inst, Algorithm alg, const RunOptions &opts = {});

}  // namespace symdist
