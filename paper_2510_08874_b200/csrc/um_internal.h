// Internal helpers shared by the C-ABI translation units (host side).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/unimul_b200.h"

namespace um {

// Thread-local last error (um_last_error).
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

inline int64_t esize(int32_t dtype) { return dtype == UM_BF16 ? 2 : 4; }
inline int64_t view_rows(const um_view& v) { return v.row_hi - v.row_lo; }
inline int64_t view_cols(const um_view& v) { return v.col_hi - v.col_lo; }

// Restores the calling thread's current device on scope exit (the CUDA current
// device is per-thread driver state shared with torch's runtime).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device);
  ~DeviceGuard();
};

// Validates the basic invariants of a view (non-negative slice, TMA pitch).
int check_view(const um_view* v, const char* name, bool need_tma_pitch);

}  // namespace um

#define UM_CUDA_CHECK(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess)                                                    \
      return ::um::fail(UM_ECUDA, std::string(#expr " failed: ") +            \
                                      cudaGetErrorString(_e));                \
  } while (0)
