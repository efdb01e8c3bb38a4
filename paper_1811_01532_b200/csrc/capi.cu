// Library-level C ABI: version, thread-local error string, launch counter.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"
#include "../../include/wap_b200.h"

std::atomic<long long> g_wap_launches{0};

static thread_local char g_err[1024] = "";

extern "C" void wap_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* wap_last_error(void) { return g_err; }

extern "C" const char* wap_version(void) { return "wap-b200 0.1.0 (sm_100a, tcgen05 tf32/3xtf32)"; }

extern "C" long long wap_launch_count(void) { return g_wap_launches.load(); }
