// Persistent row-band pipeline: TMA bulk copies (cp.async.bulk) into a ring
// of shared-memory stages, completed on mbarriers, consumed by all threads.
//
// A plane of the time-major slab is m x m doubles, rows contiguous; a band of
// rows [r0, r1) of plane q is therefore one contiguous range of the slab and
// moves with a single cp.async.bulk (1D TMA) per array and stage.  Bulk copies
// need 16-byte aligned source/destination and sizes: the range is widened to
// even element indices (at most one extra double on each side; the library
// allocates 16 spare bytes after every slab) and the consumer indexes the
// stage with the resulting 0/1 element offset.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pint {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Waits suspend in hardware until the phase completes (suspend-time hint
// PINT_MBAR_SUSPEND_NS) instead of re-polling: ncu showed the polling loops
// (try_wait + nanosleep + branch) at 20-30 % of the issued instructions of
// the band kernels, taken from the compute warps' issue slots.
#ifndef PINT_MBAR_SUSPEND_NS
#define PINT_MBAR_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(phase), "n"(PINT_MBAR_SUSPEND_NS)
        : "memory");
}

// producer-side wait (same suspend-until-complete wait)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    mbar_wait(bar, phase);
}

// global -> shared bulk copy completing `bytes` of transaction on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier 1 over the NT consumer threads (the producer warp is excluded)
template <int NT>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// deterministic sum over the NT consumer threads; valid in consumer thread 0
template <int NT>
__device__ __forceinline__ double consumer_sum(double v, double* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int tid = threadIdx.x;
    if ((tid & 31) == 0) scratch[tid >> 5] = v;
    consumer_sync<NT>();
    double s = 0.0;
    if (tid == 0)
        for (int w = 0; w < NT / 32; ++w) s += scratch[w];
    return s;
}

// Contiguous element range [e0, e1) of a slab, widened to 16-byte alignment.
struct Span {
    long long g0;      // first copied element (even)
    uint32_t bytes;    // copied bytes (multiple of 16)
    int off;           // e0 - g0 (0 or 1)
};

__device__ __forceinline__ Span span_of(long long e0, long long e1) {
    Span s;
    s.g0 = e0 & ~1LL;
    const long long g1 = (e1 + 1) & ~1LL;
    s.bytes = (uint32_t)((g1 - s.g0) * 8);
    s.off = (int)(e0 - s.g0);
    return s;
}

// issue one array's band copy into `dst` (a 16-byte aligned stage region);
// returns the element offset of the first wanted element inside dst
__device__ __forceinline__ int load_rows(double* dst, const double* slab, long long plane_base,
                                         int m, int r0, int r1, uint64_t* bar, uint32_t& tx) {
    if (r1 <= r0) return 0;
    const Span s = span_of(plane_base + (long long)r0 * m, plane_base + (long long)r1 * m);
    bulk_g2s(dst, slab + s.g0, s.bytes, bar);
    tx += s.bytes;
    return s.off;
}

// shared-memory words reserved for a band of `rows` rows of width m
__host__ __device__ constexpr int band_words(int rows, int m) {
    return ((rows * m + 2 + 1) / 2) * 2 + 2;  // +1 alignment element, keep 16 B multiples
}

}  // namespace pint
