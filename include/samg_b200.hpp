// samg_b200.hpp -- header-only C++ shim over the C-ABI (samg_b200.h) that
// re-exposes the reference library's interface (proj/include/samg) for the
// ns_block hot path, so a reference user switches by changing a namespace:
//
//   samg::setup(A, B, samg::pipeline::ns_block, prm)   hierarchy.hpp:263-265
//   samg::vcycle(H, f, u, ws)                           hierarchy.hpp:408-409
//   samg::cg_solve(H, f, u, cg_params)                  cg.hpp:87-88
//   samg::memory_footprint(H)                           hierarchy.hpp:443
//
// become samg_b200::... with the same argument types and meaning, and the
// same exception classes (common.hpp:12-28).  Differences:
// the hierarchy lives in GPU memory (move-only handle); the default smoother
// is the reference's, ILU(0) (bit-identical results; its triangular sweeps
// are latency-bound on a GPU, smoother_kind::spai0 is the fast choice);
// one hierarchy serves one solve at a time (device workspace is internal).
#pragma once

#include <cstddef>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "samg_b200.h"

namespace samg_b200 {

using index = std::ptrdiff_t;  // common.hpp:10

// ---- errors (common.hpp:12-28) + device-side failures -----------------------
struct error : std::runtime_error {
    int code;
    explicit error(const std::string &m, int c = SAMG_ERROR) : std::runtime_error(m), code(c) {}
};
#define SAMG_B200_ERR(name, c) \
    struct name : error { explicit name(const std::string &m) : error(m, c) {} };
SAMG_B200_ERR(dimension_mismatch, SAMG_DIMENSION_MISMATCH)
SAMG_B200_ERR(not_divisible, SAMG_NOT_DIVISIBLE)
SAMG_B200_ERR(singular_block, SAMG_SINGULAR_BLOCK)
SAMG_B200_ERR(missing_diagonal, SAMG_MISSING_DIAGONAL)
SAMG_B200_ERR(zero_diagonal, SAMG_ZERO_DIAGONAL)
SAMG_B200_ERR(non_square, SAMG_NON_SQUARE)
SAMG_B200_ERR(bad_nullspace_shape, SAMG_BAD_NULLSPACE_SHAPE)
SAMG_B200_ERR(breakdown_non_spd, SAMG_BREAKDOWN_NON_SPD)
SAMG_B200_ERR(invalid_material, SAMG_INVALID_MATERIAL)
SAMG_B200_ERR(shape_mismatch, SAMG_SHAPE_MISMATCH)
SAMG_B200_ERR(cuda_error, SAMG_CUDA_ERROR)
SAMG_B200_ERR(out_of_memory, SAMG_OUT_OF_MEMORY)
SAMG_B200_ERR(no_device, SAMG_NO_DEVICE)
SAMG_B200_ERR(unsupported, SAMG_UNSUPPORTED)
SAMG_B200_ERR(invalid_argument, SAMG_INVALID_ARGUMENT)
#undef SAMG_B200_ERR

inline void check(int st) {
    if (st == SAMG_OK) return;
    const std::string m = samg_last_error();
    switch (st) {
        case SAMG_DIMENSION_MISMATCH: throw dimension_mismatch(m);
        case SAMG_NOT_DIVISIBLE: throw not_divisible(m);
        case SAMG_SINGULAR_BLOCK: throw singular_block(m);
        case SAMG_MISSING_DIAGONAL: throw missing_diagonal(m);
        case SAMG_ZERO_DIAGONAL: throw zero_diagonal(m);
        case SAMG_NON_SQUARE: throw non_square(m);
        case SAMG_BAD_NULLSPACE_SHAPE: throw bad_nullspace_shape(m);
        case SAMG_BREAKDOWN_NON_SPD: throw breakdown_non_spd(m);
        case SAMG_INVALID_MATERIAL: throw invalid_material(m);
        case SAMG_SHAPE_MISMATCH: throw shape_mismatch(m);
        case SAMG_CUDA_ERROR: throw cuda_error(m);
        case SAMG_OUT_OF_MEMORY: throw out_of_memory(m);
        case SAMG_NO_DEVICE: throw no_device(m);
        case SAMG_UNSUPPORTED: throw unsupported(m);
        case SAMG_INVALID_ARGUMENT: throw invalid_argument(m);
        default: throw error(m, st);
    }
}

// ---- containers (csr.hpp:26-55, static_block.hpp:19) --------------------------
struct block3 {  // static_block<3>: row-major 3x3
    double m[9];
    double &operator()(int i, int j) { return m[i * 3 + j]; }
    const double &operator()(int i, int j) const { return m[i * 3 + j]; }
};

template <class V>
struct csr {
    index nrows = 0, ncols = 0;
    std::vector<index> ptr{0};
    std::vector<index> col;
    std::vector<V> val;
    index nnz() const { return static_cast<index>(col.size()); }
};
using scalar_csr = csr<double>;

struct dense_columns {  // column-major
    index nrows = 0, ncols = 0;
    std::vector<double> data;
    dense_columns() = default;
    dense_columns(index r, index c) : nrows(r), ncols(c), data(static_cast<std::size_t>(r) * c, 0.0) {}
    double &operator()(index i, index j) { return data[j * nrows + i]; }
    const double &operator()(index i, index j) const { return data[j * nrows + i]; }
};

// ---- parameters (coarsening.hpp:26-31, hierarchy.hpp:30-58, cg.hpp:22-35) ------
struct coarsening_params {
    double eps_strong = 0.08;
    double omega = 2.0 / 3.0;
    int point_block_size = 1;
};

enum class pipeline { scalar, block, ns_scalar, ns_hybrid1, ns_hybrid2, ns_block };
// reference: { ilu0, jacobi }; spai0 / block_jacobi are the B200 additions
enum class smoother_kind { ilu0, jacobi, spai0, block_jacobi };

struct amg_params {
    coarsening_params coarsening;
    smoother_kind smoother = smoother_kind::ilu0;  // hierarchy.hpp:52
    double smoother_omega = 0.72;  // damped_jacobi default (relaxation.hpp:143)
    int pre_sweeps = 1;
    int post_sweeps = 1;
    index coarse_enough = 3000;
    double stagnation_ratio = 0.8;
    bool verify_galerkin = false;
    int device = 0;
    bool mixed_precision_vcycle = false;  // extension: fp32 operator copies (samg_precision)
    bool ilu_latest_last = false;         // extension: relaxed backward-sweep order (samg_ilu_order)
};

struct cg_params {
    double tol = 1e-8;
    int max_iterations = 1000;
};

struct solve_report {
    int iterations = 0;
    double relative_residual = 0;
    double setup_seconds = 0;
    double solve_seconds = 0;
    std::size_t preconditioner_bytes = 0;
    pipeline variant = pipeline::ns_block;
    bool converged = false;
};

// ---- hierarchy (hierarchy.hpp:140-163) -----------------------------------------
class hierarchy {
public:
    hierarchy() = default;
    explicit hierarchy(samg_hierarchy *h) : h_(h) {}
    hierarchy(const hierarchy &) = delete;
    hierarchy &operator=(const hierarchy &) = delete;
    hierarchy(hierarchy &&o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    hierarchy &operator=(hierarchy &&o) noexcept {
        if (this != &o) { reset(); h_ = std::exchange(o.h_, nullptr); }
        return *this;
    }
    ~hierarchy() { reset(); }

    samg_hierarchy *handle() const { return h_; }
    index nlevels() const { int n = 0; check(samg_num_levels(h_, &n)); return n; }
    index finest_dim() const { int64_t n = 0; check(samg_finest_dim(h_, &n)); return n; }
    double setup_seconds() const { double s = 0; check(samg_setup_seconds(h_, &s)); return s; }

    // parity taps: level matrices in 3x3 blocks and aggregate ids
    csr<block3> level_matrix(index level, int which = 0) const {
        int64_t nr = 0, nc = 0, nz = 0;
        check(samg_level_info(h_, static_cast<int>(level), which, &nr, &nc, &nz));
        csr<block3> M;
        M.nrows = nr;
        M.ncols = nc;
        M.ptr.resize(nr + 1);
        M.col.resize(nz);
        M.val.resize(nz);
        std::vector<int64_t> p(nr + 1), c(nz);
        check(samg_get_level(h_, static_cast<int>(level), which, p.data(), c.data(),
                             reinterpret_cast<double *>(M.val.data())));
        for (int64_t i = 0; i <= nr; ++i) M.ptr[i] = p[i];
        for (int64_t i = 0; i < nz; ++i) M.col[i] = c[i];
        return M;
    }

private:
    void reset() {
        if (h_) samg_destroy(h_);
        h_ = nullptr;
    }
    samg_hierarchy *h_ = nullptr;
};

// device workspace is owned by the hierarchy; kept for signature parity
struct vcycle_workspace {
    explicit vcycle_workspace(const hierarchy &) {}
};

namespace detail {
inline samg_amg_params to_c(const amg_params &p) {
    samg_amg_params c;
    samg_default_amg_params(&c);
    c.eps_strong = p.coarsening.eps_strong;
    c.omega = p.coarsening.omega;
    c.point_block_size = p.coarsening.point_block_size;
    switch (p.smoother) {
        case smoother_kind::ilu0: c.smoother = SAMG_SMOOTHER_ILU0; break;
        case smoother_kind::jacobi: c.smoother = SAMG_SMOOTHER_JACOBI; break;
        case smoother_kind::spai0: c.smoother = SAMG_SMOOTHER_SPAI0; break;
        case smoother_kind::block_jacobi: c.smoother = SAMG_SMOOTHER_BLOCK_JACOBI; break;
    }
    c.smoother_omega = p.smoother_omega;
    c.pre_sweeps = p.pre_sweeps;
    c.post_sweeps = p.post_sweeps;
    c.coarse_enough = p.coarse_enough;
    c.stagnation_ratio = p.stagnation_ratio;
    c.verify_galerkin = p.verify_galerkin ? 1 : 0;
    c.device = p.device;
    c.vcycle_precision = p.mixed_precision_vcycle ? SAMG_PRECISION_MIXED : SAMG_PRECISION_FP64;
    c.ilu_sweep_order = p.ilu_latest_last ? SAMG_ILU_ORDER_LATEST_LAST : SAMG_ILU_ORDER_REFERENCE;
    return c;
}
} // namespace detail

// samg::setup (hierarchy.hpp:263-405)
inline hierarchy setup(const scalar_csr &A, const std::optional<dense_columns> &B,
                       pipeline variant, const amg_params &prm) {
    if (A.nrows != A.ncols) throw non_square("setup: system matrix must be square");
    if (static_cast<index>(A.ptr.size()) != A.nrows + 1)
        throw dimension_mismatch("setup: ptr size does not match nrows");
    const samg_amg_params c = detail::to_c(prm);
    std::vector<int64_t> ptr(A.ptr.begin(), A.ptr.end()), col(A.col.begin(), A.col.end());
    samg_hierarchy *h = nullptr;
    check(samg_setup(A.nrows, ptr.data(), col.data(), A.val.data(), B ? B->data.data() : nullptr,
                     B ? B->nrows : 0, B ? B->ncols : 0, static_cast<int>(variant), &c, &h));
    return hierarchy(h);
}

// samg::vcycle (hierarchy.hpp:408-441): u is the initial approximation
inline void vcycle(const hierarchy &H, std::span<const double> f, std::span<double> u,
                   vcycle_workspace &) {
    if (static_cast<index>(f.size()) != H.finest_dim() ||
        static_cast<index>(u.size()) != H.finest_dim())
        throw dimension_mismatch("vcycle: vector sizes");
    check(samg_vcycle(H.handle(), f.data(), u.data()));
}

// samg::cg_solve (cg.hpp:87-112)
inline solve_report cg_solve(const hierarchy &H, std::span<const double> f,
                             std::span<double> u, const cg_params &prm) {
    if (static_cast<index>(f.size()) != H.finest_dim() ||
        static_cast<index>(u.size()) != H.finest_dim())
        throw dimension_mismatch("cg_solve: vector sizes");
    samg_cg_params c{prm.tol, prm.max_iterations};
    samg_solve_report r{};
    check(samg_cg_solve(H.handle(), f.data(), u.data(), &c, &r));
    solve_report rep;
    rep.iterations = r.iterations;
    rep.relative_residual = r.relative_residual;
    rep.setup_seconds = r.setup_seconds;
    rep.solve_seconds = r.solve_seconds;
    rep.preconditioner_bytes = static_cast<std::size_t>(r.preconditioner_bytes);
    rep.variant = static_cast<pipeline>(r.variant);
    rep.converged = r.converged != 0;
    return rep;
}

// samg::memory_footprint (hierarchy.hpp:443-458)
inline std::size_t memory_footprint(const hierarchy &H) {
    uint64_t b = 0;
    check(samg_memory_footprint(H.handle(), &b));
    return static_cast<std::size_t>(b);
}

} // namespace samg_b200
