// problem.cuh -- host-side synthetic problem (samg_problem of the C-ABI).
#pragma once

#include <cstdint>
#include <vector>

#include "samg_b200.h"

struct samg_problem {
    int64_t n = 0, nnodes = 0;
    std::vector<int64_t> ptr, col;   // 3x3 BSR, int64 like csr.hpp:31-33
    std::vector<double> val, rhs, xyz;
};

namespace samgb {
// validated grid, element matrices (hex8_ke) and per-element materials
struct HexSetup {
    samg_problem_params p{};
    int64_t nx = 0, ny = 0, nz = 0, mx = 0, my = 0, mz = 0, i0 = 0, kx = 0;
    int64_t nnodes_all = 0, nb = 0, ne = 0;
    double hx = 0, hy = 0, hz = 0, nodal_force = 0, traction = 0;
    bool elim = false, keep = false;
    std::vector<double> Khom, Klam, Kmu, elam, emu;
};
HexSetup hex_prepare(const samg_problem_params &p);
}  // namespace samgb
