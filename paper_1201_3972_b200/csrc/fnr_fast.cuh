// Specialised tile kernels (dispatch stub; filled in by the TMA kernels).
#pragma once
#include "fnr_common.cuh"

namespace irdn {
void note_launch();
namespace fast {

inline const char* last_error() { return ""; }
inline uint64_t window_mask(int32_t) { return 0; }

template <typename T>
inline bool try_launch(const T*, T*, const PassGeom&, int, int, unsigned long long*, cudaStream_t,
                       int*) {
  return false;
}

}  // namespace fast
}  // namespace irdn
