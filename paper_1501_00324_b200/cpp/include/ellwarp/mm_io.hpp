// Drop-in for proj/include/ellwarp/mm_io.hpp: Matrix Market coordinate
// ingest (host-side input, not the hot path).
// real / integer / pattern fields, general / symmetric storage, 1-based
// indices, plain or gzip files.
#pragma once

#include <iosfwd>

#include "ellwarp/csr.hpp"

namespace ellwarp {

struct MatrixMarketError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

SparseCoo parse_matrix_market(std::istream& in);
SparseCoo parse_matrix_market_string(const std::string& text);
// plain or gzip (detected by zlib's gzread)
SparseCoo read_matrix_market_file(const std::string& path);

}  // namespace ellwarp
