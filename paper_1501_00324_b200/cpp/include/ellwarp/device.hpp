// Glue between the reference-shaped C++ API and the C ABI of the B200
// library (include/ellwarp_b200.h). Not part of the reference's API.
#pragma once

#include <memory>

#include "ellwarp/csr.hpp"
#include "ellwarp/warp_model.hpp"
#include "ellwarp_b200.h"

namespace ellwarp {

// EW_UNSUPPORTED: inputs the device path rejects (tracer, > 2^31-1 rows).
struct UnsupportedError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// EW_CUDA / EW_OUT_OF_MEMORY.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace device {

// Maps a status to the reference's exception types.
void check(ew_status s);

using CsrHandle = std::shared_ptr<ew_csr_t>;
using LayoutHandle = std::shared_ptr<ew_layout_t>;
using KernelHandle = std::shared_ptr<ew_kernel_t>;

// Row offsets and column ranges are always checked (memory safety); the
// strictly-increasing column check of validate_csr only when canonical --
// the reference's kernels accept r operands with unsorted columns.
CsrHandle upload(const SparseCsr& m, bool canonical = false);
inline CsrHandle upload_unsorted(const SparseCsr& m) { return upload(m, false); }
SparseCsr download(const CsrHandle& h);
ew_warp_config to_c(const WarpModelConfig& cfg);
void no_tracer(const WarpTracer* t);

}  // namespace device
}  // namespace ellwarp
