// Error state, launch counter, version.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>

#include "skx_common.cuh"

namespace skx {
std::atomic<long long> g_launches{0};
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace skx

extern "C" {
const char* skx_last_error(void) { return skx::g_err; }
long long skx_launch_count(void) { return skx::g_launches.load(); }
int skx_version(void) { return 1; }
}
