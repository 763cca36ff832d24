// cg_solve / cg_solve_permuted: the device solver (ew_cg_solve*) behind the
// reference's signatures (cg.hpp:32-46 in the reference).
#include "ellwarp/cg.hpp"

#include <exception>
#include <memory>

namespace ellwarp {

namespace {

struct ClosureCtx {
    const SpmvFn* fn;
    idx n;
    std::exception_ptr error;
};

// host-memory operator callback: x, y are host arrays of length n
int closure_trampoline(void* ctx, const double* x, double* y, void*) {
    auto* c = static_cast<ClosureCtx*>(ctx);
    try {
        const std::vector<real> out = (*c->fn)(std::span<const real>(x, static_cast<size_t>(c->n)));
        require(static_cast<idx>(out.size()) == c->n, "cg: operator returned a vector of the wrong length");
        std::copy(out.begin(), out.end(), y);
        return 0;
    } catch (...) {
        c->error = std::current_exception();
        return EW_INVALID_ARGUMENT;
    }
}

ew_cg_config to_c(const CgConfig& cfg) {
    return ew_cg_config{cfg.rel_tolerance, cfg.max_iterations,
                        cfg.preconditioner == CgConfig::Precond::jacobi ? 1 : 0, cfg.recompute_interval,
                        cfg.divergence_limit};
}

void check_diag(const CgConfig& cfg, idx n, std::span<const real> diag) {
    if (cfg.preconditioner == CgConfig::Precond::jacobi)
        require(static_cast<idx>(diag.size()) == n, "cg: jacobi preconditioner needs the diagonal");
}

CgResult finish(std::vector<real> x, const std::vector<real>& hist, const ew_cg_result& r) {
    CgResult res;
    res.solution = std::move(x);
    res.iterations = r.iterations;
    res.converged = r.converged != 0;
    res.spmv_calls = r.spmv_calls;
    res.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
    return res;
}

}  // namespace

CgResult cg_solve(const SpmvFn& apply_A, std::span<const real> b, const CgConfig& cfg, std::span<const real> diag) {
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    const idx n = static_cast<idx>(b.size());
    check_diag(cfg, n, diag);
    const ew_cg_config c = to_c(cfg);
    ClosureCtx ctx{&apply_A, n, nullptr};
    std::vector<real> x(n), hist(std::max<idx>(cfg.max_iterations, 0) + 1);
    ew_cg_result r{};
    const ew_status st = ew_cg_solve_operator(closure_trampoline, &ctx, EW_MEM_HOST, b.data(),
                                              diag.empty() ? nullptr : diag.data(), n, &c, EW_MEM_HOST,
                                              x.data(), hist.data(), &r, nullptr);
    if (ctx.error) std::rethrow_exception(ctx.error);
    device::check(st);
    return finish(std::move(x), hist, r);
}

CgResult cg_solve_permuted(const SpmvFn& apply_A_perm, std::span<const real> b, const Permutation& p,
                           const CgConfig& cfg, std::span<const real> diag) {
    // b and diag permuted once on entry, the solution once on exit (device gathers)
    const auto b_perm = apply_forward(p, b);
    std::vector<real> diag_perm;
    if (!diag.empty()) diag_perm = apply_forward(p, diag);
    CgResult res = cg_solve(apply_A_perm, b_perm, cfg, diag_perm);
    res.solution = apply_inverse(p, res.solution);
    return res;
}

static CgResult kernel_cg(const PreparedKernel& k, std::span<const real> b, const CgConfig& cfg,
                          std::span<const real> diag, bool permuted) {
    require(k.device != nullptr, "cg: kernel has no device handle");
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    const idx n = static_cast<idx>(b.size());
    check_diag(cfg, n, diag);
    const ew_cg_config c = to_c(cfg);
    std::vector<real> x(n), hist(std::max<idx>(cfg.max_iterations, 0) + 1);
    ew_cg_result r{};
    auto fn = permuted ? ew_cg_solve_permuted : ew_cg_solve;
    device::check(fn(k.device.get(), b.data(), diag.empty() ? nullptr : diag.data(), n, &c, EW_MEM_HOST, x.data(),
                     hist.data(), &r, nullptr));
    return finish(std::move(x), hist, r);
}

CgResult cg_solve(const PreparedKernel& k, std::span<const real> b, const CgConfig& cfg,
                  std::span<const real> diag) {
    return kernel_cg(k, b, cfg, diag, false);
}

CgResult cg_solve_permuted(const PreparedKernel& k, std::span<const real> b, const CgConfig& cfg,
                           std::span<const real> diag) {
    return kernel_cg(k, b, cfg, diag, true);
}

CgResult cg_solve_multi_gpu(const SparseCsr& a, std::span<const real> b, const CgConfig& cfg,
                            std::span<const real> diag, int ngpus, const std::string& kernel,
                            std::span<const int> devices) {
    require(a.square(), "cg: operator must be square");
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    const idx n = a.nrows;
    require(static_cast<idx>(b.size()) == n, "cg: operator must be square and match b");
    check_diag(cfg, n, diag);
    require(devices.empty() || static_cast<int>(devices.size()) == ngpus, "cg: one device per partition");
    std::vector<int32_t> dev(devices.begin(), devices.end());
    ew_mgpu h = nullptr;
    device::check(ew_mgpu_create(n, a.row_offsets.data(), a.col_indices.data(), a.values.data(), ngpus,
                                 dev.empty() ? nullptr : dev.data(), kernel.c_str(), nullptr, nullptr, &h));
    std::unique_ptr<ew_mgpu_t, ew_status (*)(ew_mgpu)> guard(h, ew_mgpu_destroy);
    const ew_cg_config c = to_c(cfg);
    std::vector<real> x(n), hist(std::max<idx>(cfg.max_iterations, 0) + 1);
    ew_cg_result r{};
    device::check(ew_mgpu_cg_solve(h, b.data(), diag.empty() ? nullptr : diag.data(), &c, x.data(), hist.data(), &r));
    return finish(std::move(x), hist, r);
}

AlphaAnalysis compute_alpha(real t_reorder, real t_kernel, real t_base) {
    AlphaAnalysis a;
    a.t_reorder = t_reorder;
    a.t_kernel = t_kernel;
    a.t_base = t_base;
    int64_t alpha = 0;
    int32_t finite = 0;
    device::check(ew_compute_alpha(t_reorder, t_kernel, t_base, &alpha, &finite));
    if (finite) a.alpha = alpha;
    return a;
}

}  // namespace ellwarp
