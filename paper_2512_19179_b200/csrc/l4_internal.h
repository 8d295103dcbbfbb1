// Internal helpers shared by the l4 host and CUDA sources (not part of the ABI).
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "l4.h"

namespace l4 {

// Thread-local last-error string (the only mutable library state besides pools).
void set_error(const char* fmt, ...);
void clear_error();

inline l4_status fail(l4_status s, const char* msg) {
  set_error("%s", msg);
  return s;
}

// NVTX range for the duration of a C-ABI call (tracing): header-only NVTX v3, a few
// ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};

}  // namespace l4

#define L4_CHECK_ARG(cond, msg)                              \
  do {                                                       \
    if (!(cond)) return ::l4::fail(L4_ERR_INVALID_ARG, msg); \
  } while (0)
