// Sine transforms along the time axis, batched over all spatial nodes.
//
// Reference: DstPlan.inverse / inverse_transpose / forward /
// forward_transpose (dst.py:57-93), i.e. products with the kernel
//   S[k][n] = sin((2k-1) n pi / 2N),  k, n = 1..N
// (inverse = S^T, inverse_transpose = S).  The reference calls scipy.fft.dst
// for power-of-two N and a dense tensordot otherwise (dst.py:60-93).
//
// B200 design: the transform runs down time columns of the time-major slab.
// A CTA owns 2P adjacent spatial columns (all N rows), so its global reads
// and writes are row segments of 2P contiguous doubles.  Two real columns
// are packed into one complex column and S / S^T are evaluated with one
// N-point complex FFT per pair:
//   S^T u : x_j = (-1)^j u_j; v = Makhoul permutation of x; C = FFT(v);
//           split C into the two real-input spectra; X_m = Re(e^{-i pi m/2N} V_m);
//           out_{N-1-m} = X_m                       (DST-II = reversed DCT-II)
//   S r   : Z_k = r_{N-1-k}; Q = Hermitian part of e^{-i pi k/2N} Z;  D = FFT(Q);
//           x = inverse Makhoul permutation of (Re D | Im D); out_j = (-1)^j x_j
// The FFT is an in-place radix-4 (+ one radix-2) decimation-in-frequency
// network in shared memory; the digit-reversed output order is undone by the
// `rev` table at the final read.  The transform is an fp64 reassociation of
// the reference's (scipy/ducc) FFT, so it agrees to rounding (~1e-15
// relative), not bitwise; the parity tests bound it at the reference's own
// 1e-13 (tests/test_dst.py:28-41 of the reference).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "pint_internal.cuh"

namespace pint {

constexpr int DST_THREADS = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}

// Output position of DFT index k after the DIF stages (radix-2 first when
// log2 N is odd, then radix-4): base-4 digit reversal = bit reversal with
// the two bits of every digit swapped back.
__device__ __forceinline__ int dif_pos(int k, int lgN) {
    if (lgN == 0) return 0;
    if (lgN & 1) {
        const int lg4 = lgN - 1;
        int t = lg4 ? (int)(__brev((unsigned)(k >> 1)) >> (32 - lg4)) : 0;
        t = ((t & 0x55555555) << 1) | ((t >> 1) & 0x55555555);
        return ((k & 1) << (lgN - 1)) | t;
    }
    int t = (int)(__brev((unsigned)k) >> (32 - lgN));
    return ((t & 0x55555555) << 1) | ((t >> 1) & 0x55555555);
}

// in-place DIF FFT (forward, e^{-2 pi i jk/N}) of P columns of length N in
// smem, pair-interleaved layout buf[pos * P + pair] (a warp touches
// consecutive double2s: no bank conflicts except on the last radix-4 stage)
template <int P>
__device__ __forceinline__ void fft_dif(double2* buf, int lgN, const double2* __restrict__ tw) {
    constexpr int lgP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : 3;
    const int tid = threadIdx.x;
    int lgL = lgN;
    if (lgN & 1) {
        const int lgs = lgN - 1, s = 1 << lgs;
        for (int item = tid; item < (P << lgs); item += DST_THREADS) {
            const int pr = item & (P - 1), j = item >> lgP;
            double2* p = buf + ((size_t)j << lgP) + pr;
            const double2 a = p[0], b = p[(size_t)s << lgP];
            p[0] = cadd(a, b);
            p[(size_t)s << lgP] = cmul(csub(a, b), __ldg(tw + j));
        }
        __syncthreads();
        lgL = lgs;
    }
    const int lgq = lgN - 2;  // quarter = N/4 butterflies per column
    while (lgL >= 2) {
        const int lgs = lgL - 2, s = 1 << lgs;
        const int lgstride = lgN - lgL;
#pragma unroll 4
        for (int item = tid; item < (P << lgq); item += DST_THREADS) {
            const int pr = item & (P - 1), t = item >> lgP;
            const int blk = t >> lgs, j = t & (s - 1);
            double2* p = buf + ((size_t)((blk << lgL) + j) << lgP) + pr;
            const int sp = s << lgP;
            const double2 x0 = p[0], x1 = p[sp], x2 = p[2 * sp], x3 = p[3 * sp];
            const double2 a0 = cadd(x0, x2), a1 = csub(x0, x2);
            const double2 b0 = cadd(x1, x3), b1 = csub(x1, x3);
            // y1 = a1 - i b1 ; y3 = a1 + i b1
            const double2 y0 = cadd(a0, b0);
            const double2 y2 = csub(a0, b0);
            const double2 y1 = make_double2(a1.x + b1.y, a1.y - b1.x);
            const double2 y3 = make_double2(a1.x - b1.y, a1.y + b1.x);
            p[0] = y0;
            if (j == 0) {
                p[sp] = y1;
                p[2 * sp] = y2;
                p[3 * sp] = y3;
            } else {
                const int js = j << lgstride;
                p[sp] = cmul(y1, __ldg(tw + js));
                p[2 * sp] = cmul(y2, __ldg(tw + 2 * js));
                p[3 * sp] = cmul(y3, __ldg(tw + 3 * js));
            }
        }
        __syncthreads();
        lgL = lgs;
    }
}

struct DstArgs {
    int N, lgN, n;
    int debug;  // diagnostic: 1 skip FFT, 2 skip FFT and fold
    const double2* tw;
    const double2* tq;
    const double* in;
    double* out;
    const double* base;   // out = base + alpha*T(in) when non-null
    double alpha;
    double in_last;       // factor on input row N-1
    double out_last;      // factor on output row N-1
};

// KIND 0: out = S^T in (dst.py:67-73);  KIND 1: out = S in (dst.py:86-93).
// P column pairs (W = 2P spatial columns) per CTA; all index math is shifts.
template <int KIND, int P>
__global__ void __launch_bounds__(DST_THREADS, 3) k_dst_fft(DstArgs a) {
    extern __shared__ double2 buf[];
    constexpr int W = 2 * P;
    constexpr int lgW = P == 1 ? 1 : P == 2 ? 2 : P == 4 ? 3 : P == 8 ? 4 : 5;
    const int lgN = a.lgN, N = 1 << lgN, n = a.n;
    const int c0 = blockIdx.x * W;
    const int ncol = min(W, n - c0);
    const int tid = threadIdx.x;
    // ---- load (+ pre-processing) ----
    // batches of LB independent loads per thread keep LB requests in flight
    constexpr int LB = 8;
    const int total = N << lgW;
    for (int base = tid; base < total; base += DST_THREADS * LB) {
        double v[LB];
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * DST_THREADS;
            const int j = idx >> lgW, cc = idx & (W - 1);
            v[i] = (idx < total && cc < ncol) ? __ldg(a.in + (size_t)j * n + c0 + cc) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * DST_THREADS;
            if (idx >= total) continue;
            const int j = idx >> lgW, cc = idx & (W - 1);
            double x = v[i];
            if (j == N - 1) x *= a.in_last;
            int pos;
            if (KIND == 0) {
                if (j & 1) {
                    x = -x;
                    pos = N - 1 - (j >> 1);
                } else {
                    pos = j >> 1;
                }
            } else {
                pos = N - 1 - j;
            }
            reinterpret_cast<double*>(buf + (size_t)pos * P + (cc >> 1))[cc & 1] = x;
        }
    }
    __syncthreads();
    if (KIND == 1 && a.debug < 2) {
        // Q_k = (t_k Z_k + conj(t_k') Z_k') / 2,  k' = (N - k) mod N,  t_k = e^{-i pi k / 2N}
        for (int item = tid; item < P * ((N >> 1) + 1); item += DST_THREADS) {
            const int pr = item % P, k = item / P;
            const int kp = (N - k) & (N - 1);
            const double2 zk = buf[(size_t)k * P + pr], zp = buf[(size_t)kp * P + pr];
            const double2 q = __ldg(a.tq + k), qp = __ldg(a.tq + kp);
            const double2 tk = make_double2(q.x, -q.y), tp = make_double2(qp.x, -qp.y);
            const double2 u1 = cadd(cmul(tk, zk), cmul(qp, zp));
            const double2 u2 = cadd(cmul(tp, zp), cmul(q, zk));
            buf[(size_t)k * P + pr] = make_double2(0.5 * u1.x, 0.5 * u1.y);
            if (kp != k) buf[(size_t)kp * P + pr] = make_double2(0.5 * u2.x, 0.5 * u2.y);
        }
        __syncthreads();
    }
    if (a.debug == 0) fft_dif<P>(buf, lgN, a.tw);
    // ---- post-processing + store ----
    for (int base = tid; base < total; base += DST_THREADS * LB) {
        double bv[LB];
        if (a.base) {
#pragma unroll
            for (int i = 0; i < LB; ++i) {
                const int idx = base + i * DST_THREADS;
                const int j = idx >> lgW, cc = idx & (W - 1);
                bv[i] = (idx < total && cc < ncol) ? __ldg(a.base + (size_t)j * n + c0 + cc) : 0.0;
            }
        }
#pragma unroll
        for (int i = 0; i < LB; ++i) {
            const int idx = base + i * DST_THREADS;
            const int j = idx >> lgW, cc = idx & (W - 1);
            if (idx >= total || cc >= ncol) continue;
            const double2* col = buf + (cc >> 1);
            double v;
            if (KIND == 0) {
                const int mm = N - 1 - j;  // out_{N-1-m} = X_m
                const double2 C = col[(size_t)dif_pos(mm, lgN) * P];
                const double2 D = col[(size_t)dif_pos((N - mm) & (N - 1), lgN) * P];
                const double2 q = __ldg(a.tq + mm);
                if ((cc & 1) == 0)
                    v = 0.5 * (q.x * (C.x + D.x) + q.y * (C.y - D.y));
                else
                    v = 0.5 * (q.x * (C.y + D.y) - q.y * (C.x - D.x));
            } else {
                const int pos = (j & 1) ? N - 1 - (j >> 1) : (j >> 1);
                const double2 Dv = col[(size_t)dif_pos(pos, lgN) * P];
                v = (cc & 1) ? Dv.y : Dv.x;
                if (j & 1) v = -v;
            }
            v = a.alpha * v;
            if (j == N - 1) v *= a.out_last;
            a.out[(size_t)j * n + c0 + cc] = a.base ? bv[i] + v : v;
        }
    }
}

// dense fallback (non power of two N): kernel[k][t] = sin((2k+1)(t+1) pi / 2N), 0-based
template <int KIND>
__global__ void __launch_bounds__(256) k_dst_dense(DstArgs a, const double* __restrict__ kern) {
    const int col = blockIdx.x * 256 + threadIdx.x;
    const int row = blockIdx.y;
    if (col >= a.n) return;
    const int N = a.N;
    double s = 0.0;
    for (int t = 0; t < N; ++t) {
        const double w = KIND == 0 ? __ldg(kern + (size_t)t * N + row)   // S^T: sum_k S[k][row] in_k
                                   : __ldg(kern + (size_t)row * N + t);  // S:   sum_t S[row][t] in_t
        double v = __ldg(a.in + (size_t)t * a.n + col);
        if (t == N - 1) v *= a.in_last;
        s += w * v;
    }
    double v = a.alpha * s;
    if (row == N - 1) v *= a.out_last;
    const size_t gi = (size_t)row * a.n + col;
    a.out[gi] = a.base ? __ldg(a.base + gi) + v : v;
}

void dst_plan_free(DstPlan& d) {
    cudaFree(d.tw);
    cudaFree(d.tq);
    cudaFree(d.rev);
    cudaFree(d.dense);
    d = DstPlan{};
}

void dst_plan_build(DstPlan& d, int N) {
    dst_plan_free(d);
    d.N = N;
    d.fast = N >= 1 && (N & (N - 1)) == 0;
    const long double PI = 3.141592653589793238462643383279502884L;
    std::vector<double2> tq(N);
    for (int k = 0; k < N; ++k) {
        const long double ang = PI * k / (2.0L * N);
        tq[k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    PINT_CUDA_CHECK(cudaMalloc(&d.tq, N * sizeof(double2)));
    PINT_CUDA_CHECK(cudaMemcpy(d.tq, tq.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
    if (d.fast) {
        std::vector<double2> tw(N);
        for (int j = 0; j < N; ++j) {
            const long double ang = -2.0L * PI * j / N;
            tw[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        int lg = 0;
        while ((1 << lg) < N) ++lg;
        d.radix2_first = lg & 1;
        // radix schedule, first stage first
        std::vector<int> radix;
        if (d.radix2_first) radix.push_back(2);
        for (int L = d.radix2_first ? N / 2 : N; L >= 4; L /= 4) radix.push_back(4);
        // DIF output position of DFT index k:
        // pos(k; L, r0, rest) = (k mod r0) * (L / r0) + pos(k / r0; L / r0, rest)
        std::vector<int> rev(N);
        for (int k = 0; k < N; ++k) {
            int pos = 0, L = N, kk = k;
            for (int r : radix) {
                pos += (kk % r) * (L / r);
                kk /= r;
                L /= r;
            }
            rev[k] = pos;
        }
        PINT_CUDA_CHECK(cudaMalloc(&d.tw, N * sizeof(double2)));
        PINT_CUDA_CHECK(cudaMalloc(&d.rev, N * sizeof(int)));
        PINT_CUDA_CHECK(cudaMemcpy(d.tw, tw.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
        PINT_CUDA_CHECK(cudaMemcpy(d.rev, rev.data(), N * sizeof(int), cudaMemcpyHostToDevice));
        int P = 65536 / (16 * N);
        if (P < 1) P = 1;
        if (P > 8) P = 8;
        if (const char* e = getenv("PINT_DST_P")) P = std::max(1, std::min(8, atoi(e)));
        if ((size_t)P * N * 16 > 200 * 1024)
            pint_throw(PINT_INPUT, "time axis too long for the single-CTA sine transform");
        d.pairs = P;
        // the attribute is per function, shared by every plan in the process:
        // allow the largest plan once instead of the current one
        static const int kMaxSmem = 200 * 1024;
#define PINT_DSTATTR(K, PP) \
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_dst_fft<K, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        PINT_DSTATTR(0, 1) PINT_DSTATTR(0, 2) PINT_DSTATTR(0, 4) PINT_DSTATTR(0, 8)
        PINT_DSTATTR(1, 1) PINT_DSTATTR(1, 2) PINT_DSTATTR(1, 4) PINT_DSTATTR(1, 8)
#undef PINT_DSTATTR
    } else {
        std::vector<double> kern((size_t)N * N);
        for (int k = 0; k < N; ++k)
            for (int t = 0; t < N; ++t)
                kern[(size_t)k * N + t] =
                    (double)sinl((2.0L * k + 1.0L) * (t + 1.0L) * PI / (2.0L * N));
        PINT_CUDA_CHECK(cudaMalloc(&d.dense, kern.size() * sizeof(double)));
        PINT_CUDA_CHECK(cudaMemcpy(d.dense, kern.data(), kern.size() * sizeof(double),
                                   cudaMemcpyHostToDevice));
    }
}

void dst_apply(pint_ctx* c, int kind, const double* in, double* out, const double* base,
               double alpha) {
    if (c->dst.N != c->N) pint_throw(PINT_DIMENSION, "transform plan does not match problem");
    dst_run(c, c->dst, kind, c->n, in, out, base, alpha);
}

void dst_run(pint_ctx* c, const DstPlan& d, int kind, long long ncols, const double* in,
             double* out, const double* base, double alpha) {
    if (ncols > 0x7fffffffLL) pint_throw(PINT_INPUT, "too many columns");
    DstArgs a{};
    a.N = d.N;
    {
        int lg = 0;
        while ((1 << lg) < d.N) ++lg;
        a.lgN = lg;
    }
    a.n = (int)ncols;
    a.tw = d.tw;
    a.tq = d.tq;
    a.in = in;
    a.out = out;
    a.base = base;
    a.alpha = alpha;
    a.in_last = 1.0;
    a.out_last = 1.0;
    a.debug = getenv("PINT_DST_DEBUG") ? atoi(getenv("PINT_DST_DEBUG")) : 0;
    int K;
    switch (kind) {
        case 0: K = 0; break;
        case 1: K = 1; break;
        case 2: K = 1; a.in_last = 0.5; a.alpha *= 2.0 / d.N; break;
        case 3: K = 0; a.out_last = 0.5; a.alpha *= 2.0 / d.N; break;
        default: pint_throw(PINT_INPUT, "unknown transform kind");
    }
    ProfScope prof(c, K == 0 ? K_DST : K_DST_T,
                   8.0 * (double)d.N * (double)ncols * (base ? 3.0 : 2.0));
    if (d.fast) {
        const int W = 2 * d.pairs;
        const dim3 g((unsigned)((ncols + W - 1) / W));
        const size_t smem = (size_t)d.pairs * d.N * 16;
#define PINT_DSTL(K, PP) k_dst_fft<K, PP><<<g, DST_THREADS, smem, c->stream>>>(a)
        if (K == 0) {
            switch (d.pairs) {
                case 1: PINT_DSTL(0, 1); break;
                case 2: PINT_DSTL(0, 2); break;
                case 4: PINT_DSTL(0, 4); break;
                default: PINT_DSTL(0, 8); break;
            }
        } else {
            switch (d.pairs) {
                case 1: PINT_DSTL(1, 1); break;
                case 2: PINT_DSTL(1, 2); break;
                case 4: PINT_DSTL(1, 4); break;
                default: PINT_DSTL(1, 8); break;
            }
        }
#undef PINT_DSTL
    } else {
        const dim3 g((unsigned)((ncols + 255) / 256), d.N);
        if (K == 0)
            k_dst_dense<0><<<g, 256, 0, c->stream>>>(a, d.dense);
        else
            k_dst_dense<1><<<g, 256, 0, c->stream>>>(a, d.dense);
    }
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
