// ctypes-facing C wrapper around the REAL reference library (compiled from
// /root/reference/proj/src by oracle/Makefile with -Dellwarp=ellwarp_ref).
//
// TEST INFRASTRUCTURE ONLY. Nothing in paper_1501_00324_b200/ links or loads
// this; it is the checker the parity tests, smoke() and bench.py's
// cpu_baseline / --impl reference legs use.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for CgDivergenceError, 3 for any other exception; the message is in
// refw_last_error().

#include <cstdint>
#include <cstring>
#include <string>
#include <memory>

#include "ellwarp/cg.hpp"
#include "ellwarp/fem/assembly.hpp"
#include "ellwarp/fem/mesh.hpp"
#include "ellwarp/kernels.hpp"
#include "ellwarp/synth.hpp"
#include "test_support.hpp"  // the reference's own test corpus (random_case, random_vector)

using namespace ellwarp;  // expands to ellwarp_ref

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const CgDivergenceError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

SparseCsr make_csr(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                   const double* v) {
    SparseCsr m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.row_offsets.assign(ro, ro + nrows + 1);
    const int64_t nnz = ro[nrows];
    m.col_indices.assign(ci, ci + nnz);
    m.values.assign(v, v + nnz);
    return m;
}

WarpModelConfig make_cfg(int ws, int seg, int align) {
    WarpModelConfig cfg;
    cfg.warp_size = ws;
    cfg.block_size = std::max(32, ws);
    cfg.segment_bytes = seg;
    cfg.align_warp_offsets = align != 0;
    return cfg;
}

// A bag of exported arrays so Python can pull results with two calls
// (length, then copy).
struct Bag {
    std::vector<std::vector<int64_t>> i;
    std::vector<std::vector<double>> d;
    std::string s;
    int64_t scalars[8] = {0};
};
}  // namespace

extern "C" {

const char* refw_last_error() { return g_err.c_str(); }

void refw_bag_free(Bag* b) { delete b; }
int64_t refw_bag_ilen(Bag* b, int k) { return k < (int)b->i.size() ? (int64_t)b->i[k].size() : -1; }
int64_t refw_bag_dlen(Bag* b, int k) { return k < (int)b->d.size() ? (int64_t)b->d[k].size() : -1; }
void refw_bag_icopy(Bag* b, int k, int64_t* out) { std::memcpy(out, b->i[k].data(), b->i[k].size() * 8); }
void refw_bag_dcopy(Bag* b, int k, double* out) { std::memcpy(out, b->d[k].data(), b->d[k].size() * 8); }
const char* refw_bag_str(Bag* b) { return b->s.c_str(); }
int64_t refw_bag_scalar(Bag* b, int k) { return b->scalars[k]; }

// CSR bag layout: i[0]=row_offsets, i[1]=col_indices, d[0]=values, scalars {nrows, ncols}
static Bag* csr_bag(const SparseCsr& m) {
    auto* b = new Bag;
    b->i = {m.row_offsets, m.col_indices};
    b->d = {m.values};
    b->scalars[0] = m.nrows;
    b->scalars[1] = m.ncols;
    return b;
}

int refw_generate(const char* spec, uint64_t seed, Bag** out) {
    return guard([&] { *out = csr_bag(generate_synthetic(spec, seed)); });
}
int refw_laplacian3d(int64_t nx, int64_t ny, int64_t nz, Bag** out) {
    return guard([&] { *out = csr_bag(laplacian3d(nx, ny, nz)); });
}
int refw_fem_tet_graph(int64_t n, int64_t minrow, int64_t maxrow, uint64_t seed, Bag** out) {
    return guard([&] { *out = csr_bag(fem_tet_graph(n, minrow, maxrow, seed)); });
}
int refw_powerlaw_rows(int64_t nrows, double alpha, int64_t maxrow, uint64_t seed, int64_t ncols,
                       Bag** out) {
    return guard([&] { *out = csr_bag(powerlaw_rows(nrows, alpha, maxrow, seed, ncols)); });
}
int refw_uniform_band(int64_t n, int64_t row_len, Bag** out) {
    return guard([&] { *out = csr_bag(uniform_band(n, row_len)); });
}
// tests/test_support.hpp:29-50
int refw_random_case(int64_t i, Bag** out) {
    return guard([&] { *out = csr_bag(testing::random_case(i)); });
}
int refw_random_csr(int64_t nrows, int64_t ncols, double density, uint64_t seed, double empty,
                    Bag** out) {
    return guard([&] { *out = csr_bag(testing::random_csr(nrows, ncols, density, seed, empty)); });
}
// tests/test_support.hpp:52-57
void refw_random_vector(int64_t n, uint64_t seed, double* out) {
    auto v = testing::random_vector(n, seed);
    std::memcpy(out, v.data(), n * 8);
}
int refw_from_coo(int64_t nrows, int64_t ncols, int64_t n, const int64_t* rows,
                  const int64_t* cols, const double* vals, Bag** out) {
    return guard([&] {
        SparseCoo coo;
        coo.nrows = nrows;
        coo.ncols = ncols;
        for (int64_t k = 0; k < n; ++k) coo.entries.push_back({rows[k], cols[k], vals[k]});
        canonicalize(coo);
        *out = csr_bag(coo_to_csr(coo));
    });
}
int refw_validate(int64_t nrows, int64_t ncols, int64_t nro, const int64_t* ro, int64_t nnz,
                  const int64_t* ci, const double* v) {
    return guard([&] {
        SparseCsr m;
        m.nrows = nrows;
        m.ncols = ncols;
        m.row_offsets.assign(ro, ro + nro);
        m.col_indices.assign(ci, ci + nnz);
        m.values.assign(v, v + nnz);
        validate_csr(m);
    });
}

int refw_spmv_reference(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                        const double* v, const double* x, double* y) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        auto r = spmv_csr_reference(m, std::span<const double>(x, ncols));
        std::memcpy(y, r.data(), nrows * 8);
    });
}

int refw_extract_diagonal(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                          const double* v, double* d) {
    return guard([&] {
        auto r = extract_diagonal(make_csr(nrows, ncols, ro, ci, v));
        std::memcpy(d, r.data(), nrows * 8);
    });
}

int refw_sort_rows_desc(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                        const double* v, int64_t* fwd, int64_t* inv) {
    return guard([&] {
        auto p = sort_rows_desc(make_csr(nrows, ncols, ro, ci, v));
        std::memcpy(fwd, p.forward.data(), nrows * 8);
        std::memcpy(inv, p.inverse.data(), nrows * 8);
    });
}

int64_t refw_compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t ws, int* status) {
    int64_t r = 0;
    *status = guard([&] { r = compute_k2_lanes(nnz_row, threshold, ws); });
    return r;
}

// Layout bag: i[0]=col_indices, d[0]=values, i[1]=warp_offset, i[2]=maxrows,
// i[3]=rows_in_warp, i[4]=row_perm.forward, i[5]=sorted_row_length,
// i[6]=reduction (k2), i[7]=rows_offset_warp (k2), i[8]=value_slot_map;
// s = dump_layout; scalars {stored_slots, padded_slots, nwarps}
int refw_build_layout(int kind, int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                      const double* v, int ws, int seg, int align, int64_t threshold,
                      int sort_rows, int row_major, Bag** out) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        const auto cfg = make_cfg(ws, seg, align);
        BuildOptions o;
        o.sort_rows = sort_rows != 0;
        o.row_major = row_major != 0;
        auto* b = new Bag;
        if (kind == 1) {
            const auto l = build_k1(m, cfg, o);
            b->i = {l.col_indices, l.warp_offset, l.maxrows, l.rows_in_warp, l.row_perm.forward,
                    l.sorted_row_length, {}, {}, value_slot_map(l, m)};
            b->d = {l.values};
            b->s = dump_layout(l);
            b->scalars[0] = l.stored_slots();
            b->scalars[1] = l.padded_slots();
            b->scalars[2] = l.nwarps();
        } else {
            const auto l = build_k2(m, cfg, threshold, o);
            b->i = {l.col_indices,      l.warp_offset, l.maxrows,   l.rows_in_warp,
                    l.row_perm.forward, l.sorted_row_length, l.reduction, l.rows_offset_warp,
                    value_slot_map(l, m)};
            b->d = {l.values};
            b->s = dump_layout(l);
            b->scalars[0] = l.stored_slots();
            b->scalars[1] = l.padded_slots();
            b->scalars[2] = l.nwarps();
        }
        *out = b;
    });
}

// reorder bag: CSR of the r / rs operand plus i[2] = forward
int refw_reorder(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, int sort_within_rows, Bag** out) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        const Permutation p = sort_rows_desc(m);
        ReorderedOperand op = make_reordered_r(m, p);
        if (sort_within_rows) op = make_reordered_rs(op);
        auto* b = csr_bag(op.matrix);
        b->i.push_back(p.forward);
        *out = b;
    });
}

// prepare_kernel(id).apply / apply_permuted; kernels.cpp:59-125
int refw_prepared_apply(const char* id, int64_t nrows, int64_t ncols, const int64_t* ro,
                        const int64_t* ci, const double* v, int ws, int seg, int align,
                        int64_t threshold, int64_t hyb_k_ell, int permuted, const double* x,
                        double* y, int64_t* stored_slots) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        KernelOptions o;
        o.k2_threshold = threshold;
        o.hyb_k_ell = hyb_k_ell;
        const PreparedKernel k = prepare_kernel(id, m, make_cfg(ws, seg, align), o);
        const auto& fn = permuted ? k.apply_permuted : k.apply;
        require(static_cast<bool>(fn), "apply_permuted is only set for r/rs kernels");
        auto r = fn(std::span<const double>(x, ncols), nullptr);
        std::memcpy(y, r.data(), nrows * 8);
        if (stored_slots) *stored_slots = k.stored_slots;
    });
}

// A prepared kernel kept alive so bench.py can time repeated apply() calls
// without the layout build (bench.cpp:71-84 times apply only).
struct RefPrepared {
    PreparedKernel k;
};
int refw_prepare(const char* id, int64_t nrows, int64_t ncols, const int64_t* ro,
                 const int64_t* ci, const double* v, int ws, int64_t threshold,
                 RefPrepared** out) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        KernelOptions o;
        o.k2_threshold = threshold;
        *out = new RefPrepared{prepare_kernel(id, m, make_cfg(ws, 128, 1), o)};
    });
}
int refw_prepared_run(RefPrepared* p, int permuted, const double* x, int64_t nx, double* y,
                      int64_t ny) {
    return guard([&] {
        const auto& fn = permuted ? p->k.apply_permuted : p->k.apply;
        auto r = fn(std::span<const double>(x, nx), nullptr);
        std::memcpy(y, r.data(), ny * 8);
    });
}
void refw_prepared_free(RefPrepared* p) { delete p; }

// cg_solve / cg_solve_permuted through prepare_kernel(id); cg.cpp:25-119.
// Result bag: d[0]=solution, d[1]=residual_history,
// scalars {iterations, converged, spmv_calls}
int refw_cg(const char* id, int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
            const double* v, const double* b, double tol, int64_t max_it, int jacobi,
            int64_t recompute, double divergence, int permuted, int ws, int64_t threshold,
            Bag** out) {
    return guard([&] {
        const auto m = make_csr(nrows, ncols, ro, ci, v);
        KernelOptions o;
        o.k2_threshold = threshold;
        const PreparedKernel k = prepare_kernel(id, m, make_cfg(ws, 128, 1), o);
        CgConfig c;
        c.rel_tolerance = tol;
        c.max_iterations = max_it;
        c.preconditioner = jacobi ? CgConfig::Precond::jacobi : CgConfig::Precond::none;
        c.recompute_interval = recompute;
        c.divergence_limit = divergence;
        const auto diag = extract_diagonal(m);
        std::span<const double> dspan = jacobi ? std::span<const double>(diag)
                                               : std::span<const double>{};
        std::span<const double> bspan(b, nrows);
        CgResult res;
        if (permuted) {
            require(static_cast<bool>(k.perm), "permuted CG needs an r/rs kernel");
            SpmvFn op = [&](std::span<const double> x) { return k.apply_permuted(x, nullptr); };
            res = cg_solve_permuted(op, bspan, *k.perm, c, dspan);
        } else {
            SpmvFn op = [&](std::span<const double> x) { return k.apply(x, nullptr); };
            res = cg_solve(op, bspan, c, dspan);
        }
        auto* bag = new Bag;
        bag->d = {res.solution, res.residual_history};
        bag->scalars[0] = res.iterations;
        bag->scalars[1] = res.converged ? 1 : 0;
        bag->scalars[2] = res.spmv_calls;
        *out = bag;
    });
}

// fem::box_mesh connectivity (fem/mesh.cpp:33-71): i[0] = elements (ne x 4),
// scalars {nnodes, nelements}
int refw_box_elements(int64_t nx, int64_t ny, int64_t nz, Bag** out) {
    return guard([&] {
        const auto mesh = fem::box_mesh(nx, ny, nz);
        auto* b = new Bag;
        std::vector<int64_t> e;
        e.reserve(mesh.elements.size() * 4);
        for (const auto& t : mesh.elements) e.insert(e.end(), t.begin(), t.end());
        b->i = {e};
        b->scalars[0] = mesh.nnodes();
        b->scalars[1] = mesh.nelements();
        *out = b;
    });
}

// assemble_spmv (fem/assembly.cpp:140-159) of given element outputs on
// box_mesh(nx, ny, nz): i[0] = pattern row_offsets, i[1] = pattern columns,
// d[0] = tangent values, d[1] = residual
int refw_box_assemble(int64_t nx, int64_t ny, int64_t nz, int ws, const double* ke, const double* re, Bag** out) {
    return guard([&] {
        const auto mesh = fem::box_mesh(nx, ny, nz);
        const auto map = fem::build_assembly_map(mesh, make_cfg(ws, 128, 1));
        std::vector<fem::ElementOutput> outs(mesh.nelements());
        for (int64_t e = 0; e < mesh.nelements(); ++e) {
            for (int i = 0; i < 4; ++i) {
                outs[e].Re[i] = re[4 * e + i];
                for (int j = 0; j < 4; ++j) outs[e].Ke[i][j] = ke[16 * e + 4 * i + j];
            }
        }
        const auto sys = fem::assemble_spmv(map, outs);
        auto* b = new Bag;
        b->i = {map.pattern.row_offsets, map.pattern.col_indices};
        b->d = {sys.tangent_values, sys.residual};
        *out = b;
    });
}

int refw_compute_alpha(double tr, double tk, double tb, int64_t* alpha, int* finite) {
    return guard([&] {
        const auto a = compute_alpha(tr, tk, tb);
        *finite = a.alpha.has_value() ? 1 : 0;
        *alpha = a.alpha.value_or(-1);
    });
}

}  // extern "C"
