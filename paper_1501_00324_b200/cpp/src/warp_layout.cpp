// build_k1 / build_k2 on the device, exported into the reference's host
// structures; value_slot_map on the device; dump_layout / padding_report
// are presentation over the host structure.
#include "ellwarp/warp_layout.hpp"

#include <sstream>

#include "ellwarp/device.hpp"

namespace ellwarp {

idx WarpLayoutK1::stored_slots() const {
    idx t = 0;
    for (idx w = 0; w < nwarps(); ++w) t += maxrows[w] * rows_in_warp[w];
    return t;
}

idx WarpLayoutK2::stored_slots() const {
    idx t = 0;
    for (idx w = 0; w < nwarps(); ++w) t += maxrows[w] * reduction[w] * rows_in_warp[w];
    return t;
}

namespace {

using LayoutHandle = std::shared_ptr<ew_layout_t>;

LayoutHandle build(const SparseCsr& m, int kind, const WarpModelConfig& cfg, idx threshold,
                   BuildOptions opts) {
    cfg.validate();
    auto h = device::upload(m);
    const ew_warp_config c = device::to_c(cfg);
    ew_layout l = nullptr;
    device::check(ew_layout_build(h.get(), kind, &c, threshold, opts.sort_rows ? 1 : 0, opts.row_major ? 1 : 0,
                                  &l));
    return LayoutHandle(l, [](ew_layout p) { ew_layout_destroy(p); });
}

template <typename L>
void export_common(const LayoutHandle& h, L& out, ew_layout_info& info, ew_layout_arrays& a) {
    device::check(ew_layout_get_info(h.get(), &info));
    out.warp_size = info.warp_size;
    out.nrows = info.nrows;
    out.ncols = info.ncols;
    out.nnz = info.nnz;
    out.values.resize(info.nslots);
    out.col_indices.resize(info.nslots);
    out.warp_offset.resize(info.nwarps);
    out.maxrows.resize(info.nwarps);
    out.rows_in_warp.resize(info.nwarps);
    out.row_perm.forward.resize(info.nrows);
    out.row_perm.inverse.resize(info.nrows);
    out.sorted_row_length.resize(info.nrows);
    a = ew_layout_arrays{out.values.data(),           out.col_indices.data(),  out.warp_offset.data(),
                         out.maxrows.data(),          out.rows_in_warp.data(), nullptr,
                         nullptr,                     out.row_perm.forward.data(), out.row_perm.inverse.data(),
                         out.sorted_row_length.data()};
}

std::shared_ptr<ew_layout_t> import_impl(int kind, int ws, bool row_major, idx nrows, idx ncols, idx nnz,
                                         idx threshold, const std::vector<real>& values,
                                         const std::vector<idx>& cols, const std::vector<idx>& woff,
                                         const std::vector<idx>& maxrows, const std::vector<idx>& riw,
                                         const std::vector<idx>* red, const std::vector<idx>* row,
                                         const Permutation& perm, const std::vector<idx>& slen) {
    require(values.size() == cols.size(), "layout values/col_indices length mismatch");
    require(maxrows.size() == woff.size() && riw.size() == woff.size(), "layout per-warp arrays mismatch");
    require(static_cast<idx>(perm.forward.size()) == nrows && static_cast<idx>(slen.size()) == nrows,
            "layout per-row arrays mismatch");
    ew_layout_desc d{};
    d.kind = kind;
    d.warp_size = ws;
    d.row_major = row_major ? 1 : 0;
    d.nrows = nrows;
    d.ncols = ncols;
    d.nnz = nnz;
    d.nwarps = static_cast<int64_t>(woff.size());
    d.nslots = static_cast<int64_t>(values.size());
    d.threshold = threshold;
    d.values = values.data();
    d.col_indices = cols.data();
    d.warp_offset = woff.data();
    d.maxrows = maxrows.data();
    d.rows_in_warp = riw.data();
    d.reduction = red ? red->data() : nullptr;
    d.rows_offset_warp = row ? row->data() : nullptr;
    d.forward = perm.forward.data();
    d.sorted_row_length = slen.data();
    ew_layout l = nullptr;
    device::check(ew_layout_import(&d, &l));
    return std::shared_ptr<ew_layout_t>(l, [](ew_layout p) { ew_layout_destroy(p); });
}

std::vector<idx> slot_map(const std::shared_ptr<ew_layout_t>& l, const SparseCsr& m) {
    auto h = device::upload(m);
    std::vector<idx> map(m.nnz());
    device::check(ew_layout_value_slot_map(l.get(), h.get(), map.data()));
    return map;
}

}  // namespace

WarpLayoutK1 build_k1(const SparseCsr& m, const WarpModelConfig& cfg, BuildOptions opts) {
    auto h = build(m, EW_LAYOUT_K1, cfg, 0, opts);
    WarpLayoutK1 out;
    ew_layout_info info{};
    ew_layout_arrays a{};
    export_common(h, out, info, a);
    out.row_major = info.row_major != 0;
    device::check(ew_layout_export(h.get(), &a));
    return out;
}

idx compute_k2_lanes(idx nnz_row, idx threshold, idx warp_size) {
    int64_t lanes = 0;
    device::check(ew_compute_k2_lanes(nnz_row, threshold, warp_size, &lanes));
    return lanes;
}

WarpLayoutK2 build_k2(const SparseCsr& m, const WarpModelConfig& cfg, idx threshold, BuildOptions opts) {
    cfg.validate();
    require(threshold >= 1, "build_k2: threshold must be >= 1");
    auto h = build(m, EW_LAYOUT_K2, cfg, threshold, opts);
    WarpLayoutK2 out;
    ew_layout_info info{};
    ew_layout_arrays a{};
    export_common(h, out, info, a);
    out.threshold = info.threshold;
    out.reduction.resize(info.nwarps);
    out.rows_offset_warp.resize(info.nwarps);
    a.reduction = out.reduction.data();
    a.rows_offset_warp = out.rows_offset_warp.data();
    device::check(ew_layout_export(h.get(), &a));
    return out;
}

namespace device {

std::shared_ptr<ew_layout_t> import(const WarpLayoutK1& l) {
    return import_impl(EW_LAYOUT_K1, l.warp_size, l.row_major, l.nrows, l.ncols, l.nnz, 0, l.values,
                       l.col_indices, l.warp_offset, l.maxrows, l.rows_in_warp, nullptr, nullptr, l.row_perm,
                       l.sorted_row_length);
}

std::shared_ptr<ew_layout_t> import(const WarpLayoutK2& l) {
    return import_impl(EW_LAYOUT_K2, l.warp_size, false, l.nrows, l.ncols, l.nnz, l.threshold, l.values,
                       l.col_indices, l.warp_offset, l.maxrows, l.rows_in_warp, &l.reduction,
                       &l.rows_offset_warp, l.row_perm, l.sorted_row_length);
}

}  // namespace device

std::vector<idx> value_slot_map(const WarpLayoutK1& l, const SparseCsr& m) {
    return slot_map(device::import(l), m);
}

std::vector<idx> value_slot_map(const WarpLayoutK2& l, const SparseCsr& m) {
    return slot_map(device::import(l), m);
}

PaddingReport padding_report(idx stored_slots, idx nnz) {
    PaddingReport r;
    r.stored_slots = stored_slots;
    r.padded_slots = stored_slots - nnz;
    r.padding_fraction = stored_slots > 0 ? static_cast<real>(r.padded_slots) / static_cast<real>(stored_slots) : 0.0;
    return r;
}

std::string dump_layout(const WarpLayoutK1& l) {
    std::ostringstream os;
    os << "k1 warp_size=" << l.warp_size << " nrows=" << l.nrows << " nnz=" << l.nnz << " nwarps=" << l.nwarps()
       << "\n";
    for (idx w = 0; w < l.nwarps(); ++w) {
        const idx first = w * l.warp_size;
        os << "warp " << w << ": offset=" << l.warp_offset[w] << " maxrows=" << l.maxrows[w]
           << " reduction=1 rows=[" << first << "," << first + l.rows_in_warp[w] << ")\n";
    }
    return os.str();
}

std::string dump_layout(const WarpLayoutK2& l) {
    std::ostringstream os;
    os << "k2 warp_size=" << l.warp_size << " nrows=" << l.nrows << " nnz=" << l.nnz
       << " threshold=" << l.threshold << " nwarps=" << l.nwarps() << "\n";
    for (idx w = 0; w < l.nwarps(); ++w) {
        os << "warp " << w << ": offset=" << l.warp_offset[w] << " maxrows=" << l.maxrows[w]
           << " reduction=" << l.reduction[w] << " rows=[" << l.rows_offset_warp[w] << ","
           << l.rows_offset_warp[w] + l.rows_in_warp[w] << ")\n";
    }
    return os.str();
}

}  // namespace ellwarp
