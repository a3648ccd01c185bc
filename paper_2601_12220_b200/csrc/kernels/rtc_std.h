// <cstdint> for headers that are also compiled at plan time by NVRTC (which
// has no host standard library): the fixed-width types the kernels use.
#pragma once
#ifdef __CUDACC_RTC__
typedef decltype(sizeof(0)) size_t;
namespace std {
using ::size_t;
typedef signed char int8_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
}  // namespace std
#else
#include <cstdint>
#endif
