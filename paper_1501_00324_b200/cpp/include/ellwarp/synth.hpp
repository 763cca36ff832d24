// Drop-in for proj/include/ellwarp/synth.hpp (synth.hpp:13-36): seeded
// host-side input generators. Same distributions in the same draw order as
// the reference, so the matrices are identical for a given seed
// (tests/test_cpp_api.py checks every family against oracle/_ref).
#pragma once

#include <cstdint>

#include "ellwarp/csr.hpp"

namespace ellwarp {

SparseCsr laplacian3d(idx nx, idx ny, idx nz);
SparseCsr fem_tet_graph(idx n, idx minrow, idx maxrow, std::uint64_t seed);
SparseCsr powerlaw_rows(idx nrows, real alpha, idx maxrow, std::uint64_t seed, idx ncols = 0);
SparseCsr uniform_band(idx n, idx row_len);

struct SyntheticSpec {
    std::string kind;
    std::vector<std::pair<std::string, std::string>> params;
};

// "kind:k=v,..." or positional "laplacian3d:4,4,4".
SparseCsr generate_synthetic(const std::string& spec, std::uint64_t default_seed = 1);

}  // namespace ellwarp
