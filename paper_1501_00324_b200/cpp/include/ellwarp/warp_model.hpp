// Drop-in for proj/include/ellwarp/warp_model.hpp: only the configuration
// survives on the device path. The lockstep transaction tracer is a CPU
// stand-in for coalescing (warp_model.hpp:12-14) and is out of scope here:
// its type exists so the reference signatures compile, and passing a
// non-null tracer throws ellwarp::UnsupportedError (real traffic comes from
// ncu, see profiles/).
#pragma once

#include "ellwarp/types.hpp"

namespace ellwarp {

struct WarpModelConfig {
    int warp_size = 32;              // power of two
    int block_size = 128;            // multiple of warp_size; no effect on results
    int segment_bytes = 128;         // alignment unit is segment_bytes / 4 slots
    bool align_warp_offsets = true;  // each warp's slab starts on a segment boundary
    bool ideal_cache = false;        // model-only; validated, ignored
    int cache_lines = 64;            // model-only; validated, ignored

    void validate() const;
};

class WarpTracer;          // not provided on the device path
struct TransactionReport;  // not provided on the device path

}  // namespace ellwarp
