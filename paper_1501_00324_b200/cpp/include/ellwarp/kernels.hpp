// Drop-in for proj/include/ellwarp/kernels.hpp (kernels.hpp:16-43): the
// operator boundary. prepare_kernel builds the layout on the device once;
// apply / apply_permuted run the sm_100a kernels (host vectors in and out,
// as the reference). `device` exposes the handle for device-resident use
// through the C ABI (ew_kernel_apply with EW_MEM_DEVICE, ew_cg_solve).
#pragma once

#include <functional>
#include <memory>

#include "ellwarp/device.hpp"
#include "ellwarp/formats.hpp"
#include "ellwarp/reorder.hpp"
#include "ellwarp/warp_spmv.hpp"

namespace ellwarp {

struct PreparedKernel {
    std::string id;
    std::function<std::vector<real>(std::span<const real>, WarpTracer*)> apply;
    std::function<std::vector<real>(std::span<const real>, WarpTracer*)> apply_permuted;  // r/rs only
    std::shared_ptr<const Permutation> perm;                                              // r/rs only
    idx nnz = 0;
    idx stored_slots = 0;
    device::KernelHandle device;  // not in the reference: the B200 handle
};

// csr_ref, csr_vector, coo, ell, hyb, k1, k1r, k1rs, k2, k2r, k2rs
const std::vector<std::string>& kernel_ids();

enum class RowOrder : idx { reference = 0, locality = 1 };

struct KernelOptions {
    idx k2_threshold = 0;  // <= 0: max row length
    idx hyb_k_ell = -1;    // < 0: 2/3-coverage heuristic
    // not in the reference: r / rs kernels may group rows by a Cuthill-McKee
    // order under the longest-first sort (same row sums; perm = that order)
    RowOrder row_order = RowOrder::reference;
};

PreparedKernel prepare_kernel(const std::string& id, const SparseCsr& m, const WarpModelConfig& cfg,
                              KernelOptions opts = {});

}  // namespace ellwarp
