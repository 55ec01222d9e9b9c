// difform_b200.hpp — the few controls the B200 C++ drop-in adds to the
// reference's API.  The API itself is the reference's own headers
// (proj/include/difform/*.hpp): callers keep including those and relink
// against libdifform_b200.so (paper_2404_01249_b200/cpp/difform_b200.cpp),
// which defines every function of core.hpp, interp.hpp, similarity.hpp,
// optim.hpp, diffeo.hpp and pipeline.hpp over the C-ABI (difform_gpu.h).
// Nothing here redefines a reference type, so this header can share a
// translation unit with any reference header.
#pragma once

#include <vector>

#include "difform_gpu.h"

namespace difform {
namespace gpu {

// Precision of the calling thread's device context: DFM_PREC_F64 (default,
// the reference's arithmetic type) or DFM_PREC_F32 (the benchmarked mode).
void set_precision(int precision);
int precision();
// register_images with the reference's arithmetic, bit-identical to it
// (DFM_OPT_EXACT; fp64 only, unfused): parity checks on chaotic inputs.
void set_exact(bool on);
// Devices the sweep's workers are spread over (default {0}).
void set_sweep_devices(const std::vector<int>& devices);
// The calling thread's context (created on first use on device 0) and the
// status -> exception mapping used by every drop-in function.
dfm_ctx* ctx();
void check(dfm_status s);

}  // namespace gpu
}  // namespace difform
