// common.cuh — small device helpers shared by the bifattn kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define BA_DEVINL __device__ __forceinline__

// Device-side bounds checks of a -DBIFATTN_CHECKS variant build (the GPU test
// suite runs against it: BIFATTN_TEST_LIB, tests/conftest.py; a failed check
// prints its line and traps).  Compiled out of the product library.
#ifdef BIFATTN_CHECKS
#include <cstdio>
#define BA_CHECK(c)                                                               \
  do {                                                                            \
    if (!(c)) {                                                                   \
      printf("BA_CHECK failed: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                  \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define BA_CHECK(c) \
  do {              \
  } while (0)
#endif

namespace ba {

BA_DEVINL uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kNegInf = -__builtin_huge_valf();  // -inf

// ---------------------------------------------------------------------------
// element conversion
// ---------------------------------------------------------------------------
BA_DEVINL float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
BA_DEVINL float bf16hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

// Round two fp32 to bf16 (RNE) and pack (lo in the low half).
BA_DEVINL uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Round two fp32 to f16 (RNE) and pack (lo in the low half).
BA_DEVINL uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Two FP8 E4M3 codes (bits [0,8) and [8,16) of `two`) -> two f16 (exact:
// every E4M3 value is an f16 normal or zero), packed lo | hi << 16.
BA_DEVINL uint32_t e4m3x2_to_f16x2(uint32_t two) {
  uint32_t h2;
  asm("{\n .reg .b16 a;\n cvt.u16.u32 a, %1;\n cvt.rn.f16x2.e4m3x2 %0, a;\n}"
      : "=r"(h2)
      : "r"(two));
  return h2;
}

// 16-byte shared-memory load / store that the compiler keeps in program order
// with other memory operations (in-place conversions).
BA_DEVINL uint4 lds128(const void* p) {
  uint4 v;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
BA_DEVINL void sts128(void* p, uint4 v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Truncate two fp32 to bf16 and pack (lo in the low half): one byte permute
// on the integer pipe instead of a conversion on the XU pipe, which the ex2 of
// the softmax already loads.  Used for the split P = P_hi + P_lo (reading
// R13): P_hi = trunc(P), P_lo = trunc(P - P_hi) (the difference is exact in
// fp32), so |P - P_hi - P_lo| < 2^-14 |P|.
BA_DEVINL uint32_t pack_bf16x2_trunc(float lo, float hi) {
  return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x7632);
}

// Packed fp32 pair arithmetic (sm_100: FFMA2 / FADD2, one instruction for
// two lanes of a pair; same IEEE rounding as the scalar operations)
BA_DEVINL unsigned long long f2_pack(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
BA_DEVINL float2 f2_unpack(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
// a * b + c
BA_DEVINL float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
  return f2_unpack(d);
}
BA_DEVINL float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(d);
}
// acc += a * b
BA_DEVINL void ffma2(float2& acc, float2 a, float2 b) { acc = fma2(a, b, acc); }

BA_DEVINL float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

BA_DEVINL float lg2(float x) {
  float y;
  asm("lg2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16-byte streaming load that does not allocate in L1 (KV is read once).
BA_DEVINL uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
BA_DEVINL uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
BA_DEVINL uint32_t ldg_stream4(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL)
// ---------------------------------------------------------------------------
BA_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
BA_DEVINL void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace ba
