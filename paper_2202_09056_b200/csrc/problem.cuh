// problem.cuh -- host-side synthetic problem (samg_problem of the C-ABI).
#pragma once

#include <cstdint>
#include <vector>

struct samg_problem {
    int64_t n = 0, nnodes = 0;
    std::vector<int64_t> ptr, col;   // 3x3 BSR, int64 like csr.hpp:31-33
    std::vector<double> val, rhs, xyz;
};
