// 3x3 block arithmetic in the reference's exact operation order
// (static_block.hpp), for the bit-exact setup kernels.  Translation units
// including this are compiled with --fmad=false; the explicit _rn
// intrinsics keep the order even where a contraction would be legal.
#pragma once

// inverse (static_block.hpp:155-194); false on a singular pivot
__device__ __forceinline__ bool blk_inverse_ref(const double *a, double *inv) {
    double lu[9];
    int piv[3];
    for (int e = 0; e < 9; ++e) lu[e] = a[e];
    for (int k = 0; k < 3; ++k) {
        int p = k;
        for (int r = k + 1; r < 3; ++r)
            if (fabs(lu[r * 3 + k]) > fabs(lu[p * 3 + k])) p = r;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < 3; ++j) { const double t = lu[k * 3 + j]; lu[k * 3 + j] = lu[p * 3 + j]; lu[p * 3 + j] = t; }
        if (fabs(lu[k * 3 + k]) < 1e-300) return false;
        const double d = __ddiv_rn(1.0, lu[k * 3 + k]);
        for (int r = k + 1; r < 3; ++r) {
            const double l = __dmul_rn(lu[r * 3 + k], d);
            lu[r * 3 + k] = l;
            for (int j = k + 1; j < 3; ++j) lu[r * 3 + j] = __dsub_rn(lu[r * 3 + j], __dmul_rn(l, lu[k * 3 + j]));
        }
    }
    for (int c = 0; c < 3; ++c) {
        double x[3] = {0.0, 0.0, 0.0};
        x[c] = 1.0;
        for (int k = 0; k < 3; ++k)
            if (piv[k] != k) { const double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
        for (int r = 1; r < 3; ++r)
            for (int j = 0; j < r; ++j) x[r] = __dsub_rn(x[r], __dmul_rn(lu[r * 3 + j], x[j]));
        for (int r = 2; r >= 0; --r) {
            for (int j = r + 1; j < 3; ++j) x[r] = __dsub_rn(x[r], __dmul_rn(lu[r * 3 + j], x[j]));
            x[r] = __ddiv_rn(x[r], lu[r * 3 + r]);
        }
        for (int r = 0; r < 3; ++r) inv[r * 3 + c] = x[r];
    }
    return true;
}

// a * b (static_block.hpp:104-113): r_ij = sum_k a_ik b_kj accumulated from
// 0 in (i, k, j) order
__device__ __forceinline__ void blk_mul_ref(const double *a, const double *b, double *r) {
    for (int e = 0; e < 9; ++e) r[e] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            const double aik = a[i * 3 + k];
            for (int j = 0; j < 3; ++j) r[i * 3 + j] = __dadd_rn(r[i * 3 + j], __dmul_rn(aik, b[k * 3 + j]));
        }
}
