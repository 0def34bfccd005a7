// Host side of the tensor-core tile kernel: the per-Gamma coordinate encoding
// (device.hpp: TcGammaDev / TcPlan) and a CPU check of its weight identity.
#pragma once

#include <cstdint>
#include <vector>

#include "device.hpp"
#include "gf2.hpp"

namespace sdb {

struct TcEncoding {
    bool ok = false;          // false: some Gamma needs more than kTcMaxK coordinates
    int kmax = 0, kw = 0;     // max coordinates per row (multiple of 32), sign words per row
    std::vector<uint32_t> sign;     // [G][N][kw]
    std::vector<short> mask;        // [G][N]
    std::vector<TcGammaDev> gam;    // [G]
};

// mats: the Gamma_j (N rows each, rows beyond a matrix's own count are zero), either the
// isometry image (a | b | a^b, 3n columns; image = true) or (a | b) with 2n columns.
TcEncoding tc_encode(const std::vector<const BitMat *> &mats, int N, int n, bool image);

// CPU check of S * popc(x|z) = C0 + c_h + sum head_k tail_k on `trials` random head/tail
// splits of random row subsets of every Gamma, with the operand bytes built exactly as the
// kernel builds them. Returns the number of mismatches.
int tc_selfcheck(const TcEncoding &enc, const std::vector<const BitMat *> &mats, int N, int n, bool image,
                 uint64_t seed, int trials);

}  // namespace sdb
