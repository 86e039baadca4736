// Library-level C ABI: version, last-error text, launch counter.
#include <atomic>
#include <cstdarg>
#include <cstdio>

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
}  // namespace cs

extern "C" const char* cs_version(void) { return "chunkstar_b200 0.1.0 sm_100a"; }
extern "C" const char* cs_last_error(void) { return g_err; }
extern "C" int64_t cs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
