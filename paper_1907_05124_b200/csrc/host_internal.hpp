// host_internal.hpp -- what the multi-device driver (multi.cpp) needs from the single-device
// host (mars_host.cpp): the error channel, a problem replica, and the device-resident records
// of an executed staged batch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/mars_b200.h"

namespace marsb200 {

// sets mars_last_error() on the calling thread, returns `code`
int host_fail(int code, const std::string& msg);

// "; mbarrier wait timed out in block .. thread .. (smem .., parity ..)" once the tcgen05
// kernel's hang detector has fired in this process, else ""
std::string hang_note();

// Device-resident records of an executed batch (mars_batch_execute), shard-local indexing.
struct BatchDevView {
    int device;
    cudaStream_t stream;
    int n;
    std::int64_t first, count;
    std::uint8_t* status;
    double* energy;
    double* cut;
    long long* iters;
    double* elapsed;
    std::int8_t* spins;     // [count][n]
    long long* best;        // [1] shard-local best index (first strict minimum), -1 if none
};
int batch_device_view(mars_batch_t* b, BatchDevView* out);

// The problem's start temperatures / iteration counts are per-run host data the records keep;
// the plan is recomputed here for the whole batch (cheap, exact).
int plan_start_temps(const mars_params_t* prm, std::uint64_t base_seed, std::int64_t total, double* out);

}  // namespace marsb200
