// Library-level C ABI: version, last-error text, launch counter, and the
// host-thread share of this process.
#include <sched.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "cs_internal.h"

namespace {
thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};
}  // namespace

namespace cs {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void note_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// One process per GPU shares the host's cores with its node-local peers.
// omp_get_max_threads() is no answer: torchrun exports OMP_NUM_THREADS=1
// (every host kernel would run single-threaded), and without it each of the
// p local ranks would start a team as wide as the whole machine.  The share
// is the cores this process may run on (its affinity mask, which the Python
// side narrows to the GPU's NUMA node when it binds) divided by the local
// ranks that share that mask: all of them unless the mask was already
// narrowed to this rank (CS_HOST_BOUND=1), never fewer than one.
int host_threads(int requested) {
  if (requested > 0) return requested;
  cpu_set_t set;
  int cores = 1;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) cores = CPU_COUNT(&set);
  int local = 1;
  const char* bound = std::getenv("CS_HOST_BOUND");
  if (!(bound && bound[0] == '1')) {
    const char* lw = std::getenv("LOCAL_WORLD_SIZE");
    if (lw) local = std::atoi(lw);
    if (local < 1) local = 1;
  }
  const int share = cores / local;
  return share > 0 ? share : 1;
}
}  // namespace cs

extern "C" const char* cs_version(void) { return "chunkstar_b200 0.1.0 sm_100a"; }
extern "C" const char* cs_last_error(void) { return g_err; }
extern "C" int64_t cs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
extern "C" int cs_host_threads(int requested) { return cs::host_threads(requested); }
