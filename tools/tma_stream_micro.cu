// Microbenchmark: HBM streaming throughput of persistent CTAs that pull
// contiguous chunks with cp.async.bulk (1D TMA) into an S-stage shared-memory
// ring, versus plain coalesced loads.  Guides the band-kernel design
// (csrc/band.cuh).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tma_stream_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1802_08126_b200/csrc/band.cuh"

using namespace pint;

__global__ void k_tma(const double* src, long long nchunks, int chunk_words, int S, double* sink) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[8];
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_barrier_init(); }
    __syncthreads();
    double acc = 0.0;
    long long k = 0;
    long long c0 = blockIdx.x;
    // prologue: S-1 chunks
    if (threadIdx.x == 0)
        for (int s = 0; s < S - 1; ++s) {
            long long c = c0 + (long long)s * gridDim.x;
            if (c < nchunks) { mbar_expect_tx(&bars[s], chunk_words * 8);
                bulk_g2s(sm + s * chunk_words, src + c * chunk_words, chunk_words * 8, &bars[s]); }
        }
    for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % S;
        if (threadIdx.x == 0) {
            long long cn = c + (long long)(S - 1) * gridDim.x;
            int sn = (k + S - 1) % S;
            if (cn < nchunks) { mbar_expect_tx(&bars[sn], chunk_words * 8);
                bulk_g2s(sm + sn * chunk_words, src + cn * chunk_words, chunk_words * 8, &bars[sn]); }
        }
        {
            uint32_t ok = 0;
            while (true) {
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&bars[s])), "r"((uint32_t)((k / S) & 1)) : "memory");
                if (ok) break;
                __nanosleep(64);
            }
        }
        if (S > 100) __syncthreads();
        for (int i = threadIdx.x; i < chunk_words; i += blockDim.x) acc += sm[s * chunk_words + i];
        __syncthreads();
    }
    if (acc == 123.456) sink[0] = acc;
}

// each chunk split into `nsplit` sub-copies issued by lane 0 of warps 0..nsplit-1
// (mode 1) or all by thread 0 (mode 0)
__global__ void k_tma_split(const double* src, long long nchunks, int chunk_words, int S,
                            int nsplit, int mode, double* sink) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[8];
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_barrier_init(); }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = chunk_words / nsplit;
    auto issue = [&](long long c, int s) {
        if (mode == 1) {
            if (lane == 0 && warp < nsplit) {
                if (warp == 0) mbar_expect_tx(&bars[s], chunk_words * 8);
                bulk_g2s(sm + s * chunk_words + warp * sub, src + c * chunk_words + warp * sub, sub * 8, &bars[s]);
            }
        } else if (threadIdx.x == 0) {
            mbar_expect_tx(&bars[s], chunk_words * 8);
            for (int w = 0; w < nsplit; ++w)
                bulk_g2s(sm + s * chunk_words + w * sub, src + c * chunk_words + w * sub, sub * 8, &bars[s]);
        }
    };
    double acc = 0.0;
    long long k = 0;
    long long c0 = blockIdx.x;
    for (int s = 0; s < S - 1; ++s) {
        long long c = c0 + (long long)s * gridDim.x;
        if (c < nchunks) issue(c, s);
    }
    for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % S;
        long long cn = c + (long long)(S - 1) * gridDim.x;
        if (cn < nchunks) issue(cn, (k + S - 1) % S);
        mbar_wait(&bars[s], (k / S) & 1);
        for (int i = threadIdx.x; i < chunk_words; i += blockDim.x) acc += sm[s * chunk_words + i];
        __syncthreads();
    }
    if (acc == 123.456) sink[0] = acc;
}

// cp.async (LDGSTS) 8-byte copies by all threads, S-stage ring, commit groups
__global__ void k_cpasync(const double* src, long long nchunks, int chunk_words, int S, double* sink) {
    extern __shared__ __align__(16) double sm[];
    double acc = 0.0;
    long long k = 0;
    long long c0 = blockIdx.x;
    auto issue = [&](long long c, int s) {
        for (int i = threadIdx.x; i < chunk_words; i += blockDim.x) {
            unsigned dst = (unsigned)__cvta_generic_to_shared(sm + s * chunk_words + i);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + c * chunk_words + i));
        }
    };
    for (int s = 0; s < S - 1; ++s) {
        long long c = c0 + (long long)s * gridDim.x;
        if (c < nchunks) issue(c, s);
        asm volatile("cp.async.commit_group;");
    }
    for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % S;
        long long cn = c + (long long)(S - 1) * gridDim.x;
        if (cn < nchunks) issue(cn, (k + S - 1) % S);
        asm volatile("cp.async.commit_group;");
        // wait until at most S-1 groups pending -> group k complete
        if (S == 2) asm volatile("cp.async.wait_group 1;");
        else if (S == 3) asm volatile("cp.async.wait_group 2;");
        else asm volatile("cp.async.wait_group 3;");
        __syncthreads();
        for (int i = threadIdx.x; i < chunk_words; i += blockDim.x) acc += sm[s * chunk_words + i];
        __syncthreads();
    }
    if (acc == 123.456) sink[0] = acc;
}

// TMA with a trivial consumer (wait only)
__global__ void k_tma_noconsume(const double* src, long long nchunks, int chunk_words, int S, double* sink) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[8];
    if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_barrier_init(); }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    long long k = 0;
    long long c0 = blockIdx.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < S - 1; ++s) {
            long long c = c0 + (long long)s * gridDim.x;
            if (c < nchunks) { mbar_expect_tx(&bars[s], chunk_words * 8);
                bulk_g2s(sm + s * chunk_words, src + c * chunk_words, chunk_words * 8, &bars[s]); }
        }
    double acc = 0.0;
    for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % S;
        if (threadIdx.x == 0) {
            long long cn = c + (long long)(S - 1) * gridDim.x;
            int sn = (k + S - 1) % S;
            if (cn < nchunks) { mbar_expect_tx(&bars[sn], chunk_words * 8);
                bulk_g2s(sm + sn * chunk_words, src + cn * chunk_words, chunk_words * 8, &bars[sn]); }
        }
        mbar_wait(&bars[s], (k / S) & 1);
        acc += sm[s * chunk_words + threadIdx.x];
        __syncwarp();
    }
    if (acc == 123.456) sink[0] = acc;
}

// warp-specialised: warp 0 lane 0 produces (full/empty mbarriers), warps 1.. consume
__global__ void k_tma_ws(const double* src, long long nchunks, int chunk_words, int S, double* sink) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t full[8], empty[8];
    const int nthr = blockDim.x - 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nthr); }
        fence_barrier_init();
    }
    __syncthreads();
    const long long c0 = blockIdx.x;
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            long long k = 0;
            for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
                mbar_expect_tx(&full[s], chunk_words * 8);
                bulk_g2s(sm + s * chunk_words, src + c * chunk_words, chunk_words * 8, &full[s]);
            }
        }
        return;
    }
    double acc = 0.0;
    long long k = 0;
    const int t = threadIdx.x - 32;
    for (long long c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % S;
        mbar_wait(&full[s], (k / S) & 1);
        for (int i = t; i < chunk_words; i += nthr) acc += sm[s * chunk_words + i];
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    if (acc == 123.456) sink[0] = acc;
}

__global__ void k_plain(const double* src, long long n, double* sink) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc += __ldg(src + i);
    if (acc == 123.456) sink[0] = acc;
}

int main() {
    const long long bytes = 2LL << 30;  // 2 GiB
    const long long words = bytes / 8;
    double *src, *sink;
    cudaMalloc(&src, bytes + 64); cudaMalloc(&sink, 64);
    cudaMemset(src, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); k_plain<<<sms * 8, 256>>>(src, words, sink); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("plain ldg            : %7.1f GB/s\n", bytes / ms / 1e6);
    }
    int sizes[] = {2048, 4096, 8192, 16384, 32768};  // bytes 16K..256K? words
    for (int kb : {8, 16, 32, 64}) {
        int cw = kb * 1024 / 8;
        for (int S : {2, 3, 4, 6}) {
            for (int cps : {1, 2, 3}) {
                size_t smem = (size_t)S * cw * 8;
                if (smem * cps > 220 * 1024) continue;
                long long nch = words / cw;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    k_tma<<<sms * cps, 256, smem>>>(src, nch, cw, S, sink);
                    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                }
                cudaError_t e = cudaGetLastError();
                printf("tma chunk %3d KB stages %d ctas/sm %d : %7.1f GB/s %s\n", kb, S, cps,
                       nch * cw * 8.0 / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    (void)sizes;
    cudaFuncSetAttribute(k_tma_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int kb : {8, 16, 32})
        for (int S : {2, 3, 4, 6})
            for (int cps : {1, 2}) {
                int cw = kb * 1024 / 8;
                size_t smem = (size_t)S * cw * 8;
                if (smem * cps > 220 * 1024) continue;
                long long nch = words / cw;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    k_tma_ws<<<sms * cps, 288, smem>>>(src, nch, cw, S, sink);
                    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                }
                printf("tma-ws chunk %2d KB stages %d ctas/sm %d: %7.1f GB/s %s\n", kb, S, cps,
                       nch * cw * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
    cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_tma_noconsume, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int kb : {8})
        for (int S : {2})
            for (int cps : {1}) {
                int cw = kb * 1024 / 8;
                size_t smem = (size_t)S * cw * 8;
                if (smem * cps > 220 * 1024) continue;
                long long nch = words / cw;
                for (int variant = 0; variant < 2; ++variant) {
                    for (int rep = 0; rep < 2; ++rep) {
                        cudaEventRecord(a);
                        if (variant == 0) k_cpasync<<<sms * cps, 256, smem>>>(src, nch, cw, S, sink);
                        else k_tma_noconsume<<<sms * cps, 256, smem>>>(src, nch, cw, S, sink);
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                    }
                    printf("%s chunk %2d KB stages %d ctas/sm %d: %7.1f GB/s %s\n",
                           variant == 0 ? "cpasync8 " : "tma-nocon", kb, S, cps,
                           nch * cw * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
                }
            }
    cudaFuncSetAttribute(k_tma_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int mode : {9}) if (mode != 9)
        for (int kb : {16, 32}) {
            int cw = kb * 1024 / 8;
            for (int S : {2, 4})
                for (int ns : {1, 4, 8}) {
                    size_t smem = (size_t)S * cw * 8;
                    long long nch = words / cw;
                    for (int rep = 0; rep < 2; ++rep) {
                        cudaEventRecord(a);
                        k_tma_split<<<sms, 256, smem>>>(src, nch, cw, S, ns, mode, sink);
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                    }
                    printf("split mode %d chunk %2d KB stages %d nsplit %d (1 cta/sm): %7.1f GB/s %s\n", mode, kb, S, ns,
                           nch * cw * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
                }
        }
    return 0;
}
