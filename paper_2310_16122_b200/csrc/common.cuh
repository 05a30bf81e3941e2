// common.cuh — device helpers shared by the kernels of libcrksr.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.h"

namespace crk {

// ---------------------------------------------------------------- error plumbing
crk_status fail(crk_ctx* c, crk_status s, const char* what);
crk_status cuda_check(crk_ctx* c, cudaError_t e, const char* what);
crk_status grow(crk_ctx* c, Buf& b, size_t bytes, cudaStream_t st);

#define CRK_TRY(expr)                         \
    do {                                      \
        crk_status _s = (expr);               \
        if (_s != CRK_OK) return _s;          \
    } while (0)

#define CRK_LAUNCHED(ctx, what)                                            \
    do {                                                                   \
        (ctx)->launches++;                                                 \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::crk::cuda_check((ctx), _e, what);  \
    } while (0)

template <class T>
inline T* P(const Buf& b) { return reinterpret_cast<T*>(b.p); }

// Small device -> host readbacks (list sizes, counts) through the ctx's mapped pinned
// buffer, written by a one-thread kernel: a cudaMemcpyAsync D2H would queue on the copy
// engine behind the caller's bulk transfers on other streams (e.g. the previous step's
// results going down), stalling the build behind them.  `dst` are byte offsets into the
// pinned buffer; sizes are 4 or 8 bytes.
struct Readback {
    const void* src[8];
    int dst[8];
    int bytes[8];
    int n = 0;
    void add(const void* s, int off, int b) { src[n] = s; dst[n] = off; bytes[n] = b; ++n; }
};
crk_status readback(crk_ctx* c, const Readback& r, cudaStream_t st);
// zero `bytes` of device memory with a kernel (cudaMemsetAsync may be carried out by a copy
// engine and then queue behind the caller's bulk transfers on other streams)
cudaError_t zero_async(void* p, size_t bytes, cudaStream_t st, crk_ctx* c = nullptr);  // counts launches in c

// ---------------------------------------------------------------- Morton
__host__ __device__ inline uint64_t spread3(uint64_t v) {  // 21 bits -> every 3rd bit
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__host__ __device__ inline uint32_t compact3(uint64_t v) {  // inverse of spread3
    v &= 0x1249249249249249ull;
    v = (v | (v >> 2)) & 0x10c30c30c30c30c3ull;
    v = (v | (v >> 4)) & 0x100f00f00f00f00full;
    v = (v | (v >> 8)) & 0x1f0000ff0000ffull;
    v = (v | (v >> 16)) & 0x1f00000000ffffull;
    v = (v | (v >> 32)) & 0x1fffffull;
    return (uint32_t)v;
}

__host__ __device__ inline uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
    return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}

// shift code (sx+1) + 3(sy+1) + 9(sz+1)  ->  sx, sy, sz in {-1, 0, 1}
__device__ __forceinline__ void decode_shift(int code, int& sx, int& sy, int& sz) {
    sx = code % 3 - 1;
    sy = (code / 3) % 3 - 1;
    sz = code / 9 - 1;
}

// ---------------------------------------------------------------- O2 predicate
// s32 = fmaf(dz,dz, fmaf(dy,dy, dx*dx)) with every op rounded to nearest even; the
// explicit intrinsics keep the compiler from re-associating (bit-exact with the oracle).
__device__ __forceinline__ float s32_of(float dx, float dy, float dz) {
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// sum across the j-slots of a warp.  G > 0: lanes l, l+G, l+2G, ... hold partial sums of
// one i (i = l % G); G = -S < 0: runs of S consecutive lanes hold one i (i = l / S)
template <int G>
__device__ __forceinline__ float slot_sum(float v) {
    if constexpr (G > 0) {
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    } else {
#pragma unroll
        for (int o = 1; o < -G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}
template <int G>
__device__ __forceinline__ int slot_sum_i(int v) {
    if constexpr (G > 0) {
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    } else {
#pragma unroll
        for (int o = 1; o < -G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

// squared distance of a point to an axis-aligned box (0 inside), fp32
__device__ __forceinline__ float box_dist2(float x, float y, float z, const float lo[3], const float hi[3]) {
    float gx = fmaxf(fmaxf(lo[0] - x, x - hi[0]), 0.f);
    float gy = fmaxf(fmaxf(lo[1] - y, y - hi[1]), 0.f);
    float gz = fmaxf(fmaxf(lo[2] - z, z - hi[2]), 0.f);
    return fmaf(gz, gz, fmaf(gy, gy, gx * gx));
}

// Slack that makes fp32 culling tests a superset of the O2 predicate (|rel err| <= 2^-22).
constexpr float CULL_SLACK = 1.0f + 1.0f / 1048576.0f * 4.0f;

// ---------------------------------------------------------------- Wendland C4 (O6)
// W(r,H)   = sigma/H^3 * wt(q),  wt(q) = (1-q)^6 (1 + 6q + 35q^2/3)
// grad W   = sigma/H^3 * gt(q) * x_ij,  gt(q) = -(56/3)/H^2 (1-q)^5 (1+5q)
constexpr float SIGMA_W = 4.92385626f;  // 495 / (32 pi), fp32-rounded

__device__ __forceinline__ void wendland_t(float s, float invH, float& wt, float& gt_h2) {
    // gt_h2 = -(56/3) (1-q)^5 (1+5q)   (caller multiplies by 1/H^2)
    float r = sqrtf(s);
    float q = r * invH;
    float t = fmaxf(1.f - q, 0.f);
    float t2 = t * t;
    float t4 = t2 * t2;
    float t5 = t4 * t;
    wt = t5 * t * fmaf(q, fmaf(q, 35.f / 3.f, 6.f), 1.f);
    gt_h2 = (-56.f / 3.f) * t5 * fmaf(5.f, q, 1.f);
}

}  // namespace crk

namespace crk {
// ---------------------------------------------------------------- TMA bulk copies + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D TMA: global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Ampere-style async copies (LDGSTS): global -> shared without registers, per-thread groups
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// order this thread's generic-proxy shared-memory writes before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// shared-memory stores through 32-bit shared addresses (a base kept in a register instead of
// the generic->shared window conversion the compiler rematerialises under register pressure)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm("mov.b32 %0, %1;" : "=r"(v) : "r"(v));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const float4& v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// fire-and-forget vector atomic add (REDG.E.ADD.F32x4)
__device__ __forceinline__ void red_add_v4(float4* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
// packed list entry: x = first | (count - 1) << 29, y = leaf | shift << 26
__device__ __forceinline__ void unpack_entry(int2 r, int& first, int& count, int& leaf, int& code) {
    first = r.x & 0x1fffffff;
    count = ((unsigned)r.x >> 29) + 1;
    leaf = r.y & 0x03ffffff;
    code = (unsigned)r.y >> 26;
}
// Row staging in runs: consecutive list entries that are consecutive full j-leaves of the
// same cell under the same shift are contiguous in memory (and their slots contiguous in
// the staged tile), so one bulk copy serves the whole run.  Returns the run length of
// the run starting at entry e (e must be a run start) and whether e starts a run.
__device__ __forceinline__ bool entry_continues(int2 prev, int2 cur) {
    int pf, pc, pl, ps, cf, cc, cl, cx;
    unpack_entry(prev, pf, pc, pl, ps);
    unpack_entry(cur, cf, cc, cl, cx);
    return pc == JMAX && ps == cx && cl == pl + 1 && cf == pf + JMAX;
}
__device__ __forceinline__ int run_length(const int2* erec, int e, int end) {
    int len = 1;
    int2 prev = __ldg(erec + e);
    while (e + len < end) {
        const int2 cur = __ldg(erec + e + len);
        if (!entry_continues(prev, cur)) break;
        prev = cur;
        ++len;
    }
    return len;
}
}  // namespace crk
