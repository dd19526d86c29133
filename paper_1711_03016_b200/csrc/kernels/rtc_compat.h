// Definitions the kernels need that NVRTC (runtime compilation of
// specialised kernels, csrc/jit.cpp) does not provide from the host C++
// library: fixed-width integers and two type traits.
#pragma once

#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#else
#include <cstdint>
#endif

namespace dlvm {
template <bool B, class T, class F>
struct cond_s {
  using type = T;
};
template <class T, class F>
struct cond_s<false, T, F> {
  using type = F;
};
template <bool B, class T, class F>
using cond_t = typename cond_s<B, T, F>::type;
template <class T>
struct is_void_s {
  static constexpr bool value = false;
};
template <>
struct is_void_s<void> {
  static constexpr bool value = true;
};
template <class T>
constexpr bool is_void_v = is_void_s<T>::value;
}  // namespace dlvm
