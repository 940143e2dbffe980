// stream_read.cuh — read-only HBM streaming micro-benchmark (measurement
// instrumentation for bench.py: "a read-only streaming
// micro-benchmark peak measured in the same run: 128-bit loads over 2 GiB with
// a trivial reduction").  Not part of the attention step.
#pragma once
#include "common.cuh"

namespace ba {

BA_DEVINL uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Every thread XOR-folds a grid-strided run of 16-byte vectors, four loads in
// flight per iteration; one word per thread reaches `sink` only when the fold
// hits a magic value (practically never), so the loads cannot be elided.
__global__ void __launch_bounds__(512) stream_read_kernel(const uint4* __restrict__ p, size_t n16,
                                                          unsigned* sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = ld_stream_u4(p + i);
    const uint4 b = ld_stream_u4(p + i + stride);
    const uint4 c = ld_stream_u4(p + i + 2 * stride);
    const uint4 d = ld_stream_u4(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    acc ^= c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) {
    const uint4 a = ld_stream_u4(p + i);
    acc ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;
}

}  // namespace ba
