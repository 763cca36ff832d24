// prepare_kernel (kernels.cpp:59-125 in the reference) over ew_kernel_prepare.
#include "ellwarp/kernels.hpp"

namespace ellwarp {

const std::vector<std::string>& kernel_ids() {
    static const std::vector<std::string> ids = [] {
        std::vector<std::string> v;
        for (int32_t i = 0; i < ew_kernel_id_count(); ++i) v.emplace_back(ew_kernel_id(i));
        return v;
    }();
    return ids;
}

PreparedKernel prepare_kernel(const std::string& id, const SparseCsr& m, const WarpModelConfig& cfg,
                              KernelOptions opts) {
    cfg.validate();
    auto h = device::upload(m);
    const ew_warp_config c = device::to_c(cfg);
    const ew_kernel_options o{opts.k2_threshold, opts.hyb_k_ell, static_cast<int64_t>(opts.row_order)};
    ew_kernel k = nullptr;
    device::check(ew_kernel_prepare(id.c_str(), h.get(), &c, &o, &k));
    device::KernelHandle kh(k, [](ew_kernel p) { ew_kernel_destroy(p); });
    ew_kernel_info info{};
    device::check(ew_kernel_get_info(k, &info));

    PreparedKernel pk;
    pk.id = id;
    pk.nnz = info.nnz;
    pk.stored_slots = info.stored_slots;
    pk.device = kh;
    const idx nrows = info.nrows, ncols = info.ncols;
    auto call = [kh, nrows, ncols](bool permuted) {
        return [kh, nrows, ncols, permuted](std::span<const real> x, WarpTracer* t) {
            device::no_tracer(t);
            require(static_cast<idx>(x.size()) == ncols, "spmv dimension mismatch");
            std::vector<real> y(nrows);
            auto fn = permuted ? ew_kernel_apply_permuted : ew_kernel_apply;
            device::check(fn(kh.get(), x.data(), ncols, y.data(), nrows, EW_MEM_HOST, nullptr));
            return y;
        };
    };
    pk.apply = call(false);
    if (info.has_perm) {
        pk.apply_permuted = call(true);
        Permutation p;
        p.forward.resize(nrows);
        p.inverse.resize(nrows);
        device::check(ew_kernel_get_perm(k, p.forward.data(), p.inverse.data()));
        pk.perm = std::make_shared<const Permutation>(std::move(p));
    }
    return pk;
}

}  // namespace ellwarp
