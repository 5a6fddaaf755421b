// hexgen.cuh -- pieces of the synthetic hex8 elasticity generator shared by
// the host assembly (generator.cpp) and the device assembly (assemble.cu):
// the element stiffness (elasticity.hpp:57-123), the isotropic material
// matrix and the counter-based random stream.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

namespace samgb {

// hex8_stiffness (elasticity.hpp:57-123) for a given isotropic C.
inline void hex8_ke(double hx, double hy, double hz, const double C[6][6], double *Ke) {
    int off[8][3];
    for (int a = 0; a < 8; ++a) { off[a][0] = a & 1; off[a][1] = (a >> 1) & 1; off[a][2] = (a >> 2) & 1; }
    const double g = 1.0 / std::sqrt(3.0);
    const double gp[2] = {-g, g};
    const double jac[3] = {hx / 2, hy / 2, hz / 2};
    const double detJ = jac[0] * jac[1] * jac[2];
    std::fill(Ke, Ke + 576, 0.0);
    for (int qx = 0; qx < 2; ++qx)
    for (int qy = 0; qy < 2; ++qy)
    for (int qz = 0; qz < 2; ++qz) {
        const double xi = gp[qx], eta = gp[qy], zeta = gp[qz];
        double dN[8][3];
        for (int a = 0; a < 8; ++a) {
            const double sx = off[a][0] ? 1.0 : -1.0, sy = off[a][1] ? 1.0 : -1.0,
                         sz = off[a][2] ? 1.0 : -1.0;
            dN[a][0] = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) / jac[0];
            dN[a][1] = 0.125 * (1 + sx * xi) * sy * (1 + sz * zeta) / jac[1];
            dN[a][2] = 0.125 * (1 + sx * xi) * (1 + sy * eta) * sz / jac[2];
        }
        for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
            double Ba[6][3] = {}, Bb[6][3] = {};
            auto fill = [](double Bm[6][3], const double d[3]) {
                Bm[0][0] = d[0]; Bm[1][1] = d[1]; Bm[2][2] = d[2];
                Bm[3][0] = d[1]; Bm[3][1] = d[0];
                Bm[4][1] = d[2]; Bm[4][2] = d[1];
                Bm[5][0] = d[2]; Bm[5][2] = d[0];
            };
            fill(Ba, dN[a]);
            fill(Bb, dN[b]);
            for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s = 0;
                for (int p = 0; p < 6; ++p)
                for (int q = 0; q < 6; ++q) s += Ba[p][i] * C[p][q] * Bb[q][j];
                Ke[(3 * a + i) * 24 + (3 * b + j)] += s * detJ;
            }
        }
    }
}

inline void iso_C(double lambda, double mu, double C[6][6]) {
    for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i][j] = (i == j) ? lambda + 2 * mu : lambda;
    for (int i = 3; i < 6; ++i) C[i][i] = mu;
}

// counter-based uniform in [0,1): splitmix64 of (seed, stream, index);
// integer arithmetic plus one exact scaling, so host and device agree bitwise
__host__ __device__ inline double uhash(uint64_t seed, uint64_t stream, uint64_t i) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + i + 0x632BE59BD9B4E019ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
}


} // namespace samgb
