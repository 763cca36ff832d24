// spmv_k1 / spmv_k1_sorted / spmv_k2 / spmv_k2_sorted on the device for a
// host layout (imported per call; prepared kernels keep theirs resident).
#include "ellwarp/warp_spmv.hpp"

#include "ellwarp/device.hpp"

namespace ellwarp {

namespace {

template <typename L>
std::vector<real> run(const L& l, std::span<const real> x, bool scatter, WarpTracer* tracer, const char* what) {
    device::no_tracer(tracer);
    require(static_cast<idx>(x.size()) == l.ncols, std::string(what) + ": dimension mismatch");
    auto h = device::import(l);
    std::vector<real> y(l.nrows);
    device::check(ew_layout_spmv(h.get(), x.data(), l.ncols, y.data(), l.nrows, scatter ? 1 : 0, EW_MEM_HOST,
                                 nullptr));
    return y;
}

}  // namespace

std::vector<real> spmv_k1(const WarpLayoutK1& l, std::span<const real> x, WarpTracer* t) {
    return run(l, x, true, t, "spmv_k1");
}
std::vector<real> spmv_k1_sorted(const WarpLayoutK1& l, std::span<const real> x, WarpTracer* t) {
    return run(l, x, false, t, "spmv_k1");
}
std::vector<real> spmv_k2(const WarpLayoutK2& l, std::span<const real> x, WarpTracer* t) {
    return run(l, x, true, t, "spmv_k2");
}
std::vector<real> spmv_k2_sorted(const WarpLayoutK2& l, std::span<const real> x, WarpTracer* t) {
    return run(l, x, false, t, "spmv_k2");
}

}  // namespace ellwarp
