// Error reporting and version for the l4 C ABI (include/l4.h).
#include <cstdarg>
#include <cstdio>

#include <nvtx3/nvToolsExt.h>

#include "l4_internal.h"

namespace l4 {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

void clear_error() { g_last_error[0] = '\0'; }

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

}  // namespace l4

extern "C" const char* l4_last_error(void) { return l4::g_last_error; }

extern "C" const char* l4_version(void) { return "l4-b200 0.1.0 sm_100a"; }
