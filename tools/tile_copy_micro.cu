// Microbenchmark: column-tile copy of a time-major slab [N][n] (the DST's
// access pattern): each CTA moves W adjacent columns x N rows, row segments
// of W doubles at a stride of n doubles.  Measures achieved GB/s vs W.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int W, int LB>
__global__ void __launch_bounds__(256) k_copy(const double* __restrict__ in, double* __restrict__ out,
                                              int N, int n) {
    const int c0 = blockIdx.x * W;
    const int total = N * W;
    for (int base = threadIdx.x; base < total; base += 256 * LB) {
        double v[LB];
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * 256;
            const int j = idx / W, cc = idx % W;
            v[i] = (idx < total && c0 + cc < n) ? __ldg(in + (size_t)j * n + c0 + cc) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * 256;
            const int j = idx / W, cc = idx % W;
            if (idx < total && c0 + cc < n) out[(size_t)j * n + c0 + cc] = v[i];
        }
    }
}

// same with 16-byte vector accesses (column pairs)
template <int W, int LB>
__global__ void __launch_bounds__(256) k_copy2(const double2* __restrict__ in, double2* __restrict__ out,
                                               int N, int n2) {
    constexpr int W2 = W / 2;
    const int c0 = blockIdx.x * W2;
    const int total = N * W2;
    for (int base = threadIdx.x; base < total; base += 256 * LB) {
        double2 v[LB];
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * 256;
            const int j = idx / W2, cc = idx % W2;
            v[i] = (idx < total && c0 + cc < n2) ? __ldg(in + (size_t)j * n2 + c0 + cc) : make_double2(0, 0);
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * 256;
            const int j = idx / W2, cc = idx % W2;
            if (idx < total && c0 + cc < n2) out[(size_t)j * n2 + c0 + cc] = v[i];
        }
    }
}

template <int W>
void run2(const double* a, double* b, int N, int n) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n2 = n / 2;
    const int grid = (n2 + W / 2 - 1) / (W / 2);
    for (int it = 0; it < 3; ++it) k_copy2<W, 8><<<grid, 256>>>((const double2*)a, (double2*)b, N, n2);
    cudaEventRecord(e0);
    const int R = 10;
    for (int it = 0; it < R; ++it) k_copy2<W, 8><<<grid, 256>>>((const double2*)a, (double2*)b, N, n2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    const double bytes = 2.0 * 16.0 * N * (double)n2;
    printf("v2 W=%3d  %.3f ms  %.0f GB/s\n", W, ms, bytes / ms / 1e6);
}

template <int W>
void run(const double* a, double* b, int N, int n) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = (n + W - 1) / W;
    for (int it = 0; it < 3; ++it) k_copy<W, 16><<<grid, 256>>>(a, b, N, n);
    cudaEventRecord(e0);
    const int R = 10;
    for (int it = 0; it < R; ++it) k_copy<W, 16><<<grid, 256>>>(a, b, N, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    const double bytes = 2.0 * 8.0 * N * (double)n;
    printf("W=%3d  %.3f ms  %.0f GB/s\n", W, ms, bytes / ms / 1e6);
}

int main(int argc, char** argv) {
    // usage: tile_copy_micro [row pitch in doubles ...]; default: the c2 slab (odd pitch)
    // and the same slab padded to a multiple of 32 doubles
    const int N = 1024;
    int pitches[8] = {65025, 65056}, np = 2;
    if (argc > 1) {
        np = 0;
        for (int i = 1; i < argc && np < 8; ++i) pitches[np++] = atoi(argv[i]);
    }
    double *a, *b;
    cudaMalloc(&a, sizeof(double) * (size_t)N * 66000);
    cudaMalloc(&b, sizeof(double) * (size_t)N * 66000);
    cudaMemset(a, 0, sizeof(double) * (size_t)N * 66000);
    for (int k = 0; k < np; ++k) {
        const int n = pitches[k];
        printf("== row pitch %d doubles (%s)\n", n, n % 32 == 0 ? "256-byte aligned rows" : "unaligned rows");
        run<4>(a, b, N, n);
        run<8>(a, b, N, n);
        run<16>(a, b, N, n);
        run<32>(a, b, N, n);
        run<64>(a, b, N, n);
        run<128>(a, b, N, n);
        run<512>(a, b, N, n);
        if (n % 2 == 0) {
            run2<8>(a, b, N, n);
            run2<16>(a, b, N, n);
            run2<32>(a, b, N, n);
            run2<64>(a, b, N, n);
        }
        run<1024>(a, b, N, n);
    }
    return 0;
}
