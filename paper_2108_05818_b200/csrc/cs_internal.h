// Internal helpers shared by the libchunkstar_b200 translation units.
#pragma once

#include <stdint.h>

#include "chunkstar_b200.h"

namespace cs {

// Thread-local last-error text (cs_last_error) and a process-wide launch
// counter (cs_launch_count) — defined in capi.cpp.
void set_error(const char* fmt, ...);
void note_launches(int64_t n);

// OpenMP team size of a host kernel: `requested` if > 0, else this
// process's share of the host cores (cs_host_threads) -- defined in capi.cpp.
int host_threads(int requested);

// Work-list batching: one launch carries at most kMaxBatch items in its
// (large) kernel-parameter block; longer lists are split into launches.
constexpr int kMaxBatch = 256;

}  // namespace cs
