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

#include <cooperative_groups.h>

#include "band.cuh"
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
    const double2* twp[3];  // k_dst_reg: per-pass twiddles, [s-1][j] contiguous in j
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

// ---------------------------------------------------------------------------
// Register-radix transform (N = 2^LG, 8 <= LG <= 13): the same S / S^T
// algebra as k_dst_fft, restructured so the tile crosses shared memory only
// between radix passes.  ncu on k_dst_fft (profiles/r1_v2_ncu_dst.txt) showed
// it L1/shared-pipe bound (L1 80 %, DRAM 24 %): ~14 shared-memory sweeps of the
// tile per transform.  Here:
//   pass 1  (radix 16, length N): global -> registers (Makhoul permutation /
//           Hermitian pre-twiddle applied on the fly) -> DFT-16 -> twiddle -> smem
//   middle  (radix 16/8/4): smem -> registers -> DFT -> twiddle -> smem (in place)
//   final   (radix 4, length 4): smem -> registers -> DFT-4 -> post-processing
//           (spectrum split / inverse permutation, alpha, base) -> global
// i.e. 1 + 2*(middle passes) + 1 shared-memory sweeps (4 for N = 1024).
// Digit-reversed order is never materialised: the final pass maps its group
// index to the frequency base by a mixed-radix digit reversal.  S^T needs the
// spectra at k and N-k together; one final-pass work unit owns both partner
// groups so the split happens in registers.
// Shared layout: double2 buf[pos * P + pair].  Every per-thread access set is
// an arithmetic progression in pos, so all shared/global offsets are
// compile-time multiples of one per-thread base address.
// ---------------------------------------------------------------------------

// column pairs per CTA: 64 KB tiles up to N = 1024; 128 KB tiles (one CTA per SM)
// for N = 2048 / 4096, where wider row segments beat the lost CTA overlap
// (N = 4096: 1.26 -> 1.45 TB/s, N = 2048: 1.64 -> 1.70 TB/s); N = 8192: one pair
__host__ __device__ constexpr int dst_reg_pairs(int lg) {
    return lg >= 13 ? 1 : lg >= 11 ? 8192 >> lg : 4096 >> lg;
}

namespace dstreg {

constexpr int T = 256;

__device__ __forceinline__ constexpr int swz(int pos) { return pos; }

// e^{-2 pi i k / 16}
template <int K>
__device__ __forceinline__ double2 w16(double2 a) {
    constexpr int k = K & 15;
    constexpr double C = 0.92387953251128673848, S = 0.38268343236508978178,
                     Q = 0.70710678118654752440;
    if constexpr (k == 0) return a;
    else if constexpr (k == 4) return make_double2(a.y, -a.x);
    else if constexpr (k == 8) return make_double2(-a.x, -a.y);
    else if constexpr (k == 12) return make_double2(-a.y, a.x);
    else if constexpr (k == 2) return make_double2(Q * (a.x + a.y), Q * (a.y - a.x));
    else if constexpr (k == 6) return make_double2(Q * (a.y - a.x), -Q * (a.x + a.y));
    else if constexpr (k == 10) return make_double2(-Q * (a.x + a.y), Q * (a.x - a.y));
    else if constexpr (k == 14) return make_double2(Q * (a.x - a.y), Q * (a.x + a.y));
    else {
        constexpr double cs[16][2] = {{1, 0}, {C, -S}, {Q, -Q}, {S, -C}, {0, -1}, {-S, -C},
                                      {-Q, -Q}, {-C, -S}, {-1, 0}, {-C, S}, {-Q, Q},
                                      {-S, C}, {0, 1}, {S, C}, {Q, Q}, {C, S}};
        return make_double2(cs[k][0] * a.x - cs[k][1] * a.y, cs[k][0] * a.y + cs[k][1] * a.x);
    }
}

__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 a0 = cadd(x0, x2), a1 = csub(x0, x2);
    const double2 b0 = cadd(x1, x3), b1 = csub(x1, x3);
    x0 = cadd(a0, b0);
    x2 = csub(a0, b0);
    x1 = make_double2(a1.x + b1.y, a1.y - b1.x);
    x3 = make_double2(a1.x - b1.y, a1.y + b1.x);
}

// in-register forward DFT of R = 4, 8 or 16 points, natural order in and out
template <int R>
__device__ __forceinline__ void dft(double2* x) {
    if constexpr (R == 4) {
        dft4(x[0], x[1], x[2], x[3]);
    } else if constexpr (R == 8) {
        // n = q + 2 n1 (q < 2, n1 < 4), k = t + 4 u
        double2 a[8];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            double2 y0 = x[q], y1 = x[q + 2], y2 = x[q + 4], y3 = x[q + 6];
            dft4(y0, y1, y2, y3);
            a[q * 4 + 0] = y0;
            a[q * 4 + 1] = y1;
            a[q * 4 + 2] = y2;
            a[q * 4 + 3] = y3;
        }
        // twiddle W8^{q t} = W16^{2 q t}
        a[5] = w16<2>(a[5]);
        a[6] = w16<4>(a[6]);
        a[7] = w16<6>(a[7]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const double2 p = a[t], r = a[4 + t];
            x[t] = cadd(p, r);
            x[t + 4] = csub(p, r);
        }
    } else {
        // n = q + 4 n1, k = t + 4 u:  X[t + 4u] = sum_q W4^{qu} W16^{qt} sum_n1 x[q + 4 n1] W4^{n1 t}
        double2 a[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double2 y0 = x[q], y1 = x[q + 4], y2 = x[q + 8], y3 = x[q + 12];
            dft4(y0, y1, y2, y3);
            a[q * 4 + 0] = y0;
            a[q * 4 + 1] = y1;
            a[q * 4 + 2] = y2;
            a[q * 4 + 3] = y3;
        }
        a[5] = w16<1>(a[5]);
        a[6] = w16<2>(a[6]);
        a[7] = w16<3>(a[7]);
        a[9] = w16<2>(a[9]);
        a[10] = w16<4>(a[10]);
        a[11] = w16<6>(a[11]);
        a[13] = w16<3>(a[13]);
        a[14] = w16<6>(a[14]);
        a[15] = w16<9>(a[15]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            double2 y0 = a[t], y1 = a[4 + t], y2 = a[8 + t], y3 = a[12 + t];
            dft4(y0, y1, y2, y3);
            x[t] = y0;
            x[t + 4] = y1;
            x[t + 8] = y2;
            x[t + 12] = y3;
        }
    }
}

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// The 15 twiddles W^{j s}, s = 1..15, of a radix-16 butterfly from the four
// table entries s = 1, 2, 4, 8 (binary composition, at most three complex
// products deep).  ncu (profiles/r2_dst_bigN_traffic.txt): the streamed tile
// (cp.async.ca) evicts the tables from what L1 the shared-memory carve-out
// leaves, so every table read is an L2 round trip -- 3.6x the data's own L2
// sectors at N = 4096; computing 11 of the 15 costs 44 fp64 instructions per
// butterfly on a pipe that is 25 % busy.
//   t: table [s-1][j] with row stride B (entries), already offset by j
__device__ __forceinline__ void twiddle16(const double2* __restrict__ t, int B, double2* w) {
    w[1] = __ldg(t);
    w[2] = __ldg(t + B);
    w[4] = __ldg(t + 3 * B);
    w[8] = __ldg(t + 7 * B);
    w[3] = cmul(w[1], w[2]);
    w[5] = cmul(w[4], w[1]);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
    w[9] = cmul(w[8], w[1]);
    w[10] = cmul(w[8], w[2]);
    w[11] = cmul(w[8], w[3]);
    w[12] = cmul(w[8], w[4]);
    w[13] = cmul(w[8], w[5]);
    w[14] = cmul(w[8], w[6]);
    w[15] = cmul(w[8], w[7]);
}

// (cos, sin)(pi s / 32), s = 0..15: q_{j + s N/16} = q_j * this  (tq[k] = (cos, sin)(pi k / 2N))
__device__ __forceinline__ double2 rot32(int s) {
    constexpr double c[16][2] = {
        {1.0, 0.0},
        {0.995184726672196886245, 0.0980171403295606019942},
        {0.980785280403230449126, 0.195090322016128267848},
        {0.956940335732208864936, 0.290284677254462367636},
        {0.923879532511286756128, 0.382683432365089771728},
        {0.881921264348355029713, 0.471396736825997648556},
        {0.831469612302545237079, 0.555570233019602224743},
        {0.773010453362736960811, 0.634393284163645498215},
        {0.707106781186547524401, 0.707106781186547524401},
        {0.634393284163645498215, 0.773010453362736960811},
        {0.555570233019602224743, 0.831469612302545237079},
        {0.471396736825997648556, 0.881921264348355029713},
        {0.382683432365089771728, 0.923879532511286756128},
        {0.290284677254462367636, 0.956940335732208864936},
        {0.195090322016128267848, 0.980785280403230449126},
        {0.0980171403295606019942, 0.995184726672196886245}};
    return make_double2(c[s][0], c[s][1]);
}

// radix schedule: pass 1 radix 16, final radix 4, middle passes in between
//   2^8: 16.4.4  2^9: 16.8.4  2^10: 16.16.4  2^11: 16.8.4.4  2^12: 16.16.4.4  2^13: 16.16.8.4
__host__ __device__ constexpr int sched_np(int lg) { return lg <= 10 ? 3 : 4; }
__host__ __device__ constexpr int sched_r(int lg, int i) {
    return i == 0 ? 16
         : i == sched_np(lg) - 1 ? 4
         : lg == 8 ? 4 : lg == 9 ? 8 : lg == 10 ? 16 : lg == 11 ? (i == 1 ? 8 : 4)
         : lg == 12 ? (i == 1 ? 16 : 4) : (i == 1 ? 16 : 8);
}
template <int LG>
struct Sched {
    static constexpr int np = sched_np(LG);
    static constexpr int r1 = sched_r(LG, 1), r2 = sched_r(LG, 2);
};

// frequency base r (k mod N/4) of final-pass group g: mixed-radix digit reversal
template <int LG>
__device__ __forceinline__ int group_freq(int g) {
    using S = Sched<LG>;
    int r = 0, mul = 1, rem = 1 << (LG - 2);
#pragma unroll
    for (int i = 0; i + 1 < S::np; ++i) {
        const int ri = sched_r(LG, i);
        rem >>= ilog2(ri);
        const int d = (g / rem) & (ri - 1);
        r += d * mul;
        mul *= ri;
    }
    return r;
}
template <int LG>
__device__ __forceinline__ int freq_group(int r) {
    using S = Sched<LG>;
    int g = 0, rem = 1 << (LG - 2);
#pragma unroll
    for (int i = 0; i + 1 < S::np; ++i) {
        const int ri = sched_r(LG, i);
        rem >>= ilog2(ri);
        g += (r & (ri - 1)) * rem;
        r >>= ilog2(ri);
    }
    return g;
}

// middle pass: radix R on sub-blocks of length 2^LGL, in place in smem
template <int R, int LGL, int LG, int P, int NT>
__device__ __forceinline__ void mid_pass(double2* buf, const double2* __restrict__ tw) {
    constexpr int lgR = ilog2(R), lgP = ilog2(P);
    constexpr int items = P << (LG - lgR);
    constexpr int lgB = LGL - lgR;  // butterflies per sub-block
#pragma unroll 1
    for (int item = threadIdx.x; item < items; item += NT) {
        const int pr = item & (P - 1), t = item >> lgP;
        const int blk = t >> lgB, j = t & ((1 << lgB) - 1);
        double2* p = buf + ((((blk << LGL) + j) << lgP) + pr);
        double2 x[R];
#pragma unroll
        for (int s = 0; s < R; ++s) x[s] = p[(s << lgB) << lgP];
        dft<R>(x);
        p[0] = x[0];
        if (j == 0) {
#pragma unroll
            for (int s = 1; s < R; ++s) p[(s << lgB) << lgP] = x[s];
        } else {
            // table [s-1][j]: a warp's lanes read consecutive j (one sector run);
            // radix 16 / 8 read the rows s = 1, 2, 4 (, 8) and compose the rest
            const double2* w = tw + j;
            if constexpr (R == 16) {
                double2 wv[16];
                twiddle16(w, 1 << lgB, wv);
#pragma unroll
                for (int s = 1; s < R; ++s) p[(s << lgB) << lgP] = cmul(x[s], wv[s]);
            } else if constexpr (R == 8) {
                double2 wv[8];
                wv[1] = __ldg(w);
                wv[2] = __ldg(w + (1 << lgB));
                wv[4] = __ldg(w + (3 << lgB));
                wv[3] = cmul(wv[1], wv[2]);
                wv[5] = cmul(wv[4], wv[1]);
                wv[6] = cmul(wv[4], wv[2]);
                wv[7] = cmul(wv[4], wv[3]);
#pragma unroll
                for (int s = 1; s < R; ++s) p[(s << lgB) << lgP] = cmul(x[s], wv[s]);
            } else {
#pragma unroll
                for (int s = 1; s < R; ++s) p[(s << lgB) << lgP] = cmul(x[s], __ldg(w + ((s - 1) << lgB)));
            }
        }
    }
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// threads per CTA: pass 1 has exactly one radix-16 butterfly per thread
template <int LG, int P>
__host__ __device__ constexpr int reg_threads() {
    return P << (LG - 4);
}

template <int KIND, int LG, int P>
__global__ void __launch_bounds__(reg_threads<LG, P>(), reg_threads<LG, P>() >= 512 ? 1 : 512 / reg_threads<LG, P>())
    k_dst_reg(DstArgs a) {
    extern __shared__ double2 buf[];
    using S = Sched<LG>;
    constexpr int NT = reg_threads<LG, P>();
    constexpr int N = 1 << LG, W = 2 * P, lgP = ilog2(P), lgW = lgP + 1;
    static_assert((P << (LG - 4)) == NT, "one pass-1 butterfly per thread");
    const int n = a.n, tid = threadIdx.x;
    const long long c0 = (long long)blockIdx.x * W;
    const int ncol = (int)min((long long)W, (long long)n - c0);
    double* sd = reinterpret_cast<double*>(buf);
    // ---- stage: coalesced row segments -> smem (pass-1 input order) ----
    // KIND 0: v[pos] <- u[row] with pos = row/2 (even rows), N-1-row/2 (odd rows);
    // KIND 1: Z_k <- r[N-1-k].  Signs and in_last are applied in pass 1.
    // A thread keeps one column and rows row0 + i*DR (DR even), so its source,
    // position and swizzled smem offsets are all linear in i.
    constexpr int DR = NT >> lgW;
    static_assert(DR % 8 == 0, "row step must keep swizzle bit 2");
    const int cc = tid & (W - 1), row0 = tid >> lgW;
    const bool cok = cc < ncol;
    {
        const double* src = a.in + c0 + (cok ? (long long)row0 * n + cc : 0);
        const long long sstep = cok ? (long long)DR * n : 0;
        int pos0, dpos;
        if (KIND == 0) {
            pos0 = (row0 & 1) ? N - 1 - (row0 >> 1) : (row0 >> 1);
            dpos = (row0 & 1) ? -(DR / 2) : DR / 2;
        } else {
            pos0 = N - 1 - row0;
            dpos = -DR;
        }
        double* dst = sd + ((swz(pos0) << lgP) + (cc >> 1)) * 2 + (cc & 1);
        const int dstep = (dpos << lgP) * 2;
#pragma unroll 16
        for (int i = 0; i < N / DR; ++i) {
            cp_async8(dst, src, cok);
            src += sstep;
            dst += dstep;
        }
        cp_async_wait_all();
        __syncthreads();
    }
    // ---- pass 1: radix 16 over the whole column, one butterfly per thread ----
    // thread (pr, j) owns positions j + s N/16; position < N/2 <=> s < 8
    {
        constexpr int lgB = LG - 4, B = 1 << lgB;
        const int pr = tid & (P - 1), j = tid >> lgP;
        double2* p = buf + ((j << lgP) + pr);
        double2 x[16];
        if (KIND == 0) {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                double2 v = p[(s << lgB) << lgP];
                if (s == 8 && j == 0) v = make_double2(v.x * a.in_last, v.y * a.in_last);
                x[s] = s < 8 ? v : make_double2(-v.x, -v.y);
            }
        } else {
            // Q_k = (conj(q_k) Z_k + q_{k'} Z_{k'}) / 2,  k' = (N-k) mod N:
            // j > 0: k' = (B - j) + (15 - s) B;  j = 0: k' = (16 - s) B mod N
            const int jp = j == 0 ? 0 : B - j;
            const double2* pp = buf + ((jp << lgP) + pr);
            // q at k = j + s B and k' = jp + sp B from q_j, q_jp and the constants
            // (cos, sin)(pi s / 32): 2 table reads instead of 32
            const double2 qj = __ldg(a.tq + j), qjp = __ldg(a.tq + jp);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                double2 zk = p[(s << lgB) << lgP];
                const int sp = j == 0 ? (16 - s) & 15 : 15 - s;
                double2 zp = pp[(sp << lgB) << lgP];
                if (s == 0 && j == 0) {
                    zk = make_double2(zk.x * a.in_last, zk.y * a.in_last);
                    zp = zk;
                }
                const double2 qk = s == 0 ? qj : cmul(qj, rot32(s));
                // j > 0: sp = 15 - s is a compile-time index; j == 0: (16 - s) & 15
                const double2 qp0 = cmul(qjp, rot32((16 - s) & 15)), qp1 = cmul(qjp, rot32(15 - s));
                const double2 qp = j == 0 ? (s == 0 ? qjp : qp0) : qp1;
                const double2 u1 = cadd(cmul(make_double2(qk.x, -qk.y), zk), cmul(qp, zp));
                x[s] = make_double2(0.5 * u1.x, 0.5 * u1.y);
            }
            __syncthreads();  // partners' reads before anyone overwrites
        }
        dft<16>(x);
        p[0] = x[0];
        if (j == 0) {
#pragma unroll
            for (int s = 1; s < 16; ++s) p[(s << lgB) << lgP] = x[s];
        } else {
            double2 w[16];
            twiddle16(a.twp[0] + j, B, w);  // [s-1][j], j < N/16
#pragma unroll
            for (int s = 1; s < 16; ++s) p[(s << lgB) << lgP] = cmul(x[s], w[s]);
        }
    }
    __syncthreads();
    // ---- middle passes ----
    if constexpr (S::np >= 3) {
        constexpr int L2 = LG - 4;
        mid_pass<S::r1, L2, LG, P, NT>(buf, a.twp[1]);
        __syncthreads();
        if constexpr (S::np == 4) {
            constexpr int L3 = L2 - ilog2(S::r1);
            mid_pass<S::r2, L3, LG, P, NT>(buf, a.twp[2]);
            __syncthreads();
        }
    }
    // ---- final radix-4 pass: results to smem in output-row order ----
    // (reads of every group finish before the barrier, writes after it)
    constexpr int Q4 = N / 4;
    auto load_group = [&](int g, int pr, double2* x) {
#pragma unroll
        for (int s = 0; s < 4; ++s) x[s] = buf[(swz(4 * g + s) << lgP) + pr];
        dft4(x[0], x[1], x[2], x[3]);
    };
    if (KIND == 1) {
        // D at k = r + s N/4;  out_j = (-1)^j x_j, x = inverse Makhoul permutation of (Re D | Im D)
        constexpr int per = (P * Q4) / NT;
        double2 x[per][4];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            load_group(item >> lgP, item & (P - 1), x[i]);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), r = group_freq<LG>(item >> lgP);
            // k = r + s N/4 < N/2 <=> s < 2:  rows 2k (s < 2), 2(N-1-k)+1 (s >= 2)
            buf[((2 * r) << lgP) + pr] = x[i][0];
            buf[((2 * (r + Q4)) << lgP) + pr] = x[i][1];
            buf[((2 * (N - 1 - r - 2 * Q4) + 1) << lgP) + pr] = make_double2(-x[i][2].x, -x[i][2].y);
            buf[((2 * (N - 1 - r - 3 * Q4) + 1) << lgP) + pr] = make_double2(-x[i][3].x, -x[i][3].y);
        }
    } else {
        // X_m of the two real columns from C_m and C_{N-m}; out_{N-1-m} = X_m
        constexpr int per = (P * (Q4 / 2)) / NT;
        double2 x[per][4], y[per][4];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), u = item >> lgP;
            load_group(freq_group<LG>(u == 0 ? 0 : u), pr, x[i]);
            load_group(freq_group<LG>(u == 0 ? N / 8 : Q4 - u), pr, y[i]);
        }
        __syncthreads();
        // q_m = (cos, sin)(pi m / 2N) of m = r + s N/4 is q_r rotated by pi s / 8
        // (rot32(4 s)): one table read per group instead of four
        auto emit = [&](int m, int pr, double2 C, double2 D, double2 q) {
            const double va = 0.5 * (q.x * (C.x + D.x) + q.y * (C.y - D.y));
            const double vb = 0.5 * (q.x * (C.y + D.y) - q.y * (C.x - D.x));
            buf[(swz(N - 1 - m) << lgP) + pr] = make_double2(va, vb);
        };
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), u = item >> lgP;
            if (u == 0) {
                // self-partnered groups r = 0 (N-k = (4-s) N/4) and r = N/8 (N-k = N/8 + (3-s) N/4)
                emit(0, pr, x[i][0], x[i][0], rot32(0));
                emit(Q4, pr, x[i][1], x[i][3], rot32(4));
                emit(2 * Q4, pr, x[i][2], x[i][2], rot32(8));
                emit(3 * Q4, pr, x[i][3], x[i][1], rot32(12));
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    emit(N / 8 + s * Q4, pr, y[i][s], y[i][3 - s], rot32(2 + 4 * s));
            } else {
                // k = r + s N/4  <->  N - k = rp + (3 - s) N/4
                const int r = u, rp = Q4 - u;
                const double2 qr = __ldg(a.tq + r), qrp = __ldg(a.tq + rp);
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    emit(r + s * Q4, pr, x[i][s], y[i][3 - s], s == 0 ? qr : cmul(qr, rot32(4 * s)));
                    emit(rp + s * Q4, pr, y[i][s], x[i][3 - s], s == 0 ? qrp : cmul(qrp, rot32(4 * s)));
                }
            }
        }
    }
    __syncthreads();
    // ---- store: coalesced row segments, alpha / out_last / base ----
    if (cok) {
        const long long step = (long long)DR * n;
        double* out = a.out + c0 + (long long)row0 * n + cc;
        const double* basep = a.base ? a.base + c0 + (long long)row0 * n + cc : nullptr;
        const double* sp = sd + ((swz(row0) << lgP) + (cc >> 1)) * 2 + (cc & 1);
        constexpr int sstep = (DR << lgP) * 2;
        // KIND 0 (S, carries the fused u += omega*y): all N/DR (= 32) base values
        // of the thread's column are requested before the first store, so one
        // HBM latency is exposed instead of one per batch of 8 (S 0.50 -> 0.41 ms
        // on c2); S^T keeps batches of 8 (measured slower with 32)
        constexpr int LB = KIND == 0 ? N / DR : 8;
        const double alpha = a.alpha;
#pragma unroll 1
        for (int i0 = 0; i0 < N / DR; i0 += LB) {
            double bv[LB];
            if (basep) {
#pragma unroll
                for (int i = 0; i < LB; ++i) bv[i] = __ldg(basep + (i0 + i) * step);
            }
#pragma unroll
            for (int i = 0; i < LB; ++i) {
                const int row = row0 + (i0 + i) * DR;
                double v = alpha * sp[(i0 + i) * sstep];
                if (row == N - 1) v *= a.out_last;
                out[(i0 + i) * step] = basep ? bv[i] + v : v;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Cluster transform for N = 2^11 .. 2^13 (config 4's time axis; the GLOBAL
// time axis of the time-sharded configs): the N x 8-column tile no longer fits
// one CTA's shared memory (k_dst_reg falls back to 4- and 2-column tiles,
// 32- / 16-byte row segments, one CTA per SM: 1.4 / 1.1 TB/s), so a thread-block
// cluster of CL = N / 1024 CTAs holds it in distributed shared memory, 1024
// positions x 4 pairs (64 KB) per CTA -- the shape of the N = 1024 kernel,
// several CTAs per SM.  The algebra, radix schedule and tables are
// k_dst_reg's.  Who holds what:
//   staging   CTA q stages the inputs of ITS pass-1 butterflies j in
//             [q B/CL, (q+1) B/CL), B = N/16: position s B + j at local s B/CL + jj;
//   pass 1    reads local (S: the Hermitian partner from the CTA that staged
//             it, a DSMEM read), cluster barrier, DFT-16, twiddle, output s of
//             butterfly j to its HOME: position p lives in CTA p / (N/CL)
//             (DSMEM writes), cluster barrier;
//   middle    sub-blocks of length N/16 are whole inside a CTA: local;
//   final     radix-4 groups local; S^T reads the partner group (k <-> N-k)
//             from its home CTA; cluster barrier; results to the home of their
//             OUTPUT ROW (CTA row / (N/CL)); cluster barrier;
//   store     every CTA writes its N/CL consecutive output rows.
// Five cluster barriers per tile; about 2.5 tile volumes cross DSMEM.
// ---------------------------------------------------------------------------
namespace cgx = cooperative_groups;

template <int KIND, int LG, int P, int CL>
__global__ void __launch_bounds__((P << (LG - 4)) / CL, 2) k_dst_cl(DstArgs a) {
    extern __shared__ double2 buf[];
    using S = Sched<LG>;
    constexpr int N = 1 << LG, lgCL = ilog2(CL), lgNL = LG - lgCL, NL = 1 << lgNL;
    constexpr int NT = (P << (LG - 4)) >> lgCL;
    constexpr int W = 2 * P, lgP = ilog2(P), lgW = lgP + 1;
    constexpr int lgB = LG - 4, B = 1 << lgB, lgBL = lgB - lgCL, BL = 1 << lgBL;
    constexpr int Q4 = N / 4, GL = NL / 4;   // radix-4 groups: all / per CTA
    static_assert(CL * (16 / CL) == 16 && BL >= 1, "cluster size divides the radix-16 sub-blocks");
    cgx::cluster_group cluster = cgx::this_cluster();
    const int q = (int)cluster.block_rank();
    const int tid = threadIdx.x, n = a.n;
    const long long c0 = (long long)(blockIdx.x >> lgCL) * W;
    const int ncol = (int)min((long long)W, (long long)n - c0);
    double* sd = reinterpret_cast<double*>(buf);
    auto rbuf = [&](int rank) -> double2* { return cluster.map_shared_rank(buf, rank); };
    constexpr int DR = NT >> lgW;  // local positions / rows per sweep
    const int cc = tid & (W - 1), lrow0 = tid >> lgW;
    const bool cok = cc < ncol;
    // ---- stage: the inputs of this CTA's butterflies (raw values; signs in pass 1) ----
    {
        const double* src0 = a.in + c0 + (cok ? cc : 0);
        double* dst = sd + ((lrow0 << lgP) + (cc >> 1)) * 2 + (cc & 1);
        // lp = lrow0 + i DR with lrow0 < DR <= BL: the sub-block s = lp / BL and the
        // offset inside it are compile-time functions of i, so unrolled the loop
        // is one multiply-add per copy
        static_assert(DR <= BL && BL % DR == 0, "staging sweeps stay inside a sub-block");
        const long long nn = cok ? n : 0;
        const int pbase = q * BL + lrow0;
#pragma unroll
        for (int i = 0; i < NL / DR; ++i) {
            constexpr int per_s = BL / DR;
            const int s_ = i / per_s, off = (i % per_s) * DR;
            const int pos = s_ * B + off + pbase;
            const int row = KIND == 0 ? (s_ < 8 ? 2 * pos : 2 * (N - 1 - pos) + 1) : N - 1 - pos;
            cp_async8(dst + (size_t)i * ((DR << lgP) * 2), src0 + row * nn, cok);
        }
        cp_async_wait_all();
    }
    cluster.sync();
    // ---- pass 1: radix 16 over the whole column, one butterfly per thread ----
    {
        const int pr = tid & (P - 1), jj = tid >> lgP, j = q * BL + jj;
        const double2* p = buf + ((jj << lgP) + pr);   // staging layout: s at + s BL
        double2 x[16];
        if (KIND == 0) {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                double2 v = p[(s << lgBL) << lgP];
                if (s == 8 && j == 0) v = make_double2(v.x * a.in_last, v.y * a.in_last);
                x[s] = s < 8 ? v : make_double2(-v.x, -v.y);
            }
        } else {
            // Q_k = (conj(q_k) Z_k + q_{k'} Z_{k'}) / 2,  k' = (N-k) mod N (k_dst_reg);
            // butterfly jp was staged by CTA jp / BL
            const int jp = j == 0 ? 0 : B - j;
            const double2* pp = rbuf(jp >> lgBL) + (((jp & (BL - 1)) << lgP) + pr);
            const double2 qj = __ldg(a.tq + j), qjp = __ldg(a.tq + jp);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                double2 zk = p[(s << lgBL) << lgP];
                const int sp = j == 0 ? (16 - s) & 15 : 15 - s;
                double2 zp = pp[(sp << lgBL) << lgP];
                if (s == 0 && j == 0) {
                    zk = make_double2(zk.x * a.in_last, zk.y * a.in_last);
                    zp = zk;
                }
                const double2 qk = s == 0 ? qj : cmul(qj, rot32(s));
                const double2 qp0 = cmul(qjp, rot32((16 - s) & 15)), qp1 = cmul(qjp, rot32(15 - s));
                const double2 qp = j == 0 ? (s == 0 ? qjp : qp0) : qp1;
                const double2 u1 = cadd(cmul(make_double2(qk.x, -qk.y), zk), cmul(qp, zp));
                x[s] = make_double2(0.5 * u1.x, 0.5 * u1.y);
            }
        }
        cluster.sync();  // every CTA has read its (and its partners') staged inputs
        dft<16>(x);
        double2 w[16];
        if (j != 0) twiddle16(a.twp[0] + j, B, w);
        // output s -> position s B + j, home CTA s / (16 / CL)
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            double2* hb = rbuf(s >> (4 - lgCL));
            const int lpos = ((s & (16 / CL - 1)) << lgB) + j;
            hb[(lpos << lgP) + pr] = (s == 0 || j == 0) ? x[s] : cmul(x[s], w[s]);
        }
    }
    cluster.sync();
    // ---- middle passes: sub-blocks of length N/16, local ----
    if constexpr (S::np >= 3) {
        constexpr int L2 = LG - 4;
        mid_pass<S::r1, L2, lgNL, P, NT>(buf, a.twp[1]);
        __syncthreads();
        if constexpr (S::np == 4) {
            constexpr int L3 = L2 - ilog2(S::r1);
            mid_pass<S::r2, L3, lgNL, P, NT>(buf, a.twp[2]);
            __syncthreads();
        }
    }
    // S^T reads partner groups from other CTAs: their middle passes must be done
    if constexpr (KIND == 0) cluster.sync();
    // ---- final radix-4 pass ----
    auto load_group = [&](const double2* b, int gl, int pr, double2* x) {
#pragma unroll
        for (int s = 0; s < 4; ++s) x[s] = b[((4 * gl + s) << lgP) + pr];
        dft4(x[0], x[1], x[2], x[3]);
    };
    // result of output row `row` to its home CTA
    auto put = [&](int row, int pr, double2 v) {
        rbuf(row >> lgNL)[((row & (NL - 1)) << lgP) + pr] = v;
    };
    if (KIND == 1) {
        constexpr int per = (P * GL) / NT;
        double2 x[per][4];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            load_group(buf, item >> lgP, item & (P - 1), x[i]);
        }
        cluster.sync();
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), r = group_freq<LG>(q * GL + (item >> lgP));
            put(2 * r, pr, x[i][0]);
            put(2 * (r + Q4), pr, x[i][1]);
            put(2 * (N - 1 - r - 2 * Q4) + 1, pr, make_double2(-x[i][2].x, -x[i][2].y));
            put(2 * (N - 1 - r - 3 * Q4) + 1, pr, make_double2(-x[i][3].x, -x[i][3].y));
        }
    } else {
        // units: this CTA's groups whose frequency base r is below N/8, i.e. whose
        // lowest digit (the last middle pass's) has its top bit clear; the partner
        // group of r is the group of N/4 - r, read from its home CTA
        constexpr int lb = ilog2(sched_r(LG, S::np - 2));
        constexpr int per = (P * (GL / 2)) / NT;
        double2 x[per][4], y[per][4];
        int rr[per];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), v = item >> lgP;
            const int gl = ((v >> (lb - 1)) << lb) | (v & ((1 << (lb - 1)) - 1));
            const int r = group_freq<LG>(q * GL + gl);
            rr[i] = r;
            load_group(buf, gl, pr, x[i]);
            const int gy = freq_group<LG>(r == 0 ? N / 8 : Q4 - r);
            load_group(rbuf(gy / GL), gy % GL, pr, y[i]);
        }
        cluster.sync();
        auto emit = [&](int m, int pr, double2 C, double2 D, double2 qv) {
            const double va = 0.5 * (qv.x * (C.x + D.x) + qv.y * (C.y - D.y));
            const double vb = 0.5 * (qv.x * (C.y + D.y) - qv.y * (C.x - D.x));
            put(N - 1 - m, pr, make_double2(va, vb));
        };
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int item = tid + i * NT;
            const int pr = item & (P - 1), r = rr[i];
            if (r == 0) {
                emit(0, pr, x[i][0], x[i][0], rot32(0));
                emit(Q4, pr, x[i][1], x[i][3], rot32(4));
                emit(2 * Q4, pr, x[i][2], x[i][2], rot32(8));
                emit(3 * Q4, pr, x[i][3], x[i][1], rot32(12));
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    emit(N / 8 + s * Q4, pr, y[i][s], y[i][3 - s], rot32(2 + 4 * s));
            } else {
                const int rp = Q4 - r;
                const double2 qr = __ldg(a.tq + r), qrp = __ldg(a.tq + rp);
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    emit(r + s * Q4, pr, x[i][s], y[i][3 - s], s == 0 ? qr : cmul(qr, rot32(4 * s)));
                    emit(rp + s * Q4, pr, y[i][s], x[i][3 - s], s == 0 ? qrp : cmul(qrp, rot32(4 * s)));
                }
            }
        }
    }
    cluster.sync();
    // ---- store: this CTA's N/CL consecutive output rows ----
    if (cok) {
        const long long step = (long long)DR * n;
        const long long g0 = c0 + (long long)(q * NL + lrow0) * n + cc;
        double* out = a.out + g0;
        const double* basep = a.base ? a.base + g0 : nullptr;
        const double* sp = sd + ((lrow0 << lgP) + (cc >> 1)) * 2 + (cc & 1);
        constexpr int sstep = (DR << lgP) * 2;
        constexpr int LB = KIND == 0 ? NL / DR : 8;
        const double alpha = a.alpha;
#pragma unroll 1
        for (int i0 = 0; i0 < NL / DR; i0 += LB) {
            double bv[LB];
            if (basep) {
#pragma unroll
                for (int i = 0; i < LB; ++i) bv[i] = __ldg(basep + (i0 + i) * step);
            }
#pragma unroll
            for (int i = 0; i < LB; ++i) {
                const int row = q * NL + lrow0 + (i0 + i) * DR;
                double v = alpha * sp[(i0 + i) * sstep];
                if (row == N - 1) v *= a.out_last;
                out[(i0 + i) * step] = basep ? bv[i] + v : v;
            }
        }
    }
}

}  // namespace dstreg

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
    for (auto* p : d.twp) cudaFree(p);
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
        // register-radix kernel (k_dst_reg) for 2^8 <= N <= 2^13
        d.reg_lg = (lg >= 8 && lg <= 13 && !getenv("PINT_DST_OLD")) ? lg : 0;
        if (d.reg_lg) {
            // per-pass twiddle tables W_L^{j s}, stored [s-1][j] (j fastest):
            // pass 1 L = N, R = 16; middle passes L = N/16 (R = r1), N/(16 r1) (R = r2)
            const int np = dstreg::sched_np(lg);
            int L = N, lgL = lg;
            for (int ps = 0; ps + 1 < np; ++ps) {
                const int R = dstreg::sched_r(lg, ps);
                const int B = L / R;
                std::vector<double2> t((size_t)(R - 1) * B);
                for (int sidx = 1; sidx < R; ++sidx)
                    for (int j = 0; j < B; ++j) {
                        const long double ang = -2.0L * PI * (long double)((long long)j * sidx) / L;
                        t[(size_t)(sidx - 1) * B + j] = make_double2((double)cosl(ang), (double)sinl(ang));
                    }
                PINT_CUDA_CHECK(cudaMalloc(&d.twp[ps], t.size() * sizeof(double2)));
                PINT_CUDA_CHECK(cudaMemcpy(d.twp[ps], t.data(), t.size() * sizeof(double2),
                                           cudaMemcpyHostToDevice));
                L = B;
                (void)lgL;
            }
            d.reg_p = dst_reg_pairs(lg);
            if (const char* e = getenv("PINT_DST_P")) {
                const int want = atoi(e);
                if ((lg == 10 && (want == 2 || want == 4)) || (lg == 9 && (want == 4 || want == 8)) ||
                    (lg == 11 && (want == 2 || want == 4)) || (lg == 12 && (want == 1 || want == 2)))
                    d.reg_p = want;
            }
            static bool attr_done = false;
            if (!attr_done) {
#define PINT_REGATTR(LGV, PV)                                                                   \
                PINT_CUDA_CHECK(cudaFuncSetAttribute(dstreg::k_dst_reg<0, LGV, PV>,              \
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                     PV * (16 << LGV)));                          \
                PINT_CUDA_CHECK(cudaFuncSetAttribute(dstreg::k_dst_reg<1, LGV, PV>,              \
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                     PV * (16 << LGV)));
                PINT_REGATTR(8, 16) PINT_REGATTR(9, 8) PINT_REGATTR(9, 4) PINT_REGATTR(10, 4)
                PINT_REGATTR(10, 2) PINT_REGATTR(11, 2) PINT_REGATTR(12, 1) PINT_REGATTR(13, 1)
                PINT_REGATTR(11, 4) PINT_REGATTR(12, 2)
#undef PINT_REGATTR
                attr_done = true;
            }
        }
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

template <int K, int LG, int CL>
static void launch_dst_cl(pint_ctx* c, const DstArgs& a, long long ncols) {
    constexpr int P = 4, W = 2 * P, NT = (P << (LG - 4)) / CL;
    constexpr size_t smem = ((size_t)1 << LG) / CL * P * 16;
    auto kern = dstreg::k_dst_cl<K, LG, P, CL>;
    static bool attr_done = false;
    if (!attr_done) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(((ncols + W - 1) / W) * CL));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PINT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

// N >= 2048: the thread-block-cluster transform (PINT_DST_NOCL: the single-CTA tiles)
static bool dst_cluster_enabled() {
    static const bool on = getenv("PINT_DST_NOCL") == nullptr;
    return on;
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
    for (int q = 0; q < 3; ++q) a.twp[q] = d.twp[q];
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
    if (d.fast && d.reg_lg >= 12 && dst_cluster_enabled()) {
        if (d.reg_lg == 12) {
            if (K == 0) launch_dst_cl<0, 12, 4>(c, a, ncols); else launch_dst_cl<1, 12, 4>(c, a, ncols);
        } else {
            if (K == 0) launch_dst_cl<0, 13, 8>(c, a, ncols); else launch_dst_cl<1, 13, 8>(c, a, ncols);
        }
    } else if (d.fast && d.reg_lg) {
        // N = 2048: S (KIND 1) runs 2.5x faster on 64 KB tiles (2 CTAs per SM) than on
        // 128 KB ones, S^T slightly slower (measured: 1.68 vs 0.95 and 2.00 vs 2.13 TB/s)
        const int P = (d.reg_lg == 11 && K == 1 && d.reg_p == 4 && !getenv("PINT_DST_P")) ? 2 : d.reg_p;
        const dim3 g((unsigned)((ncols + 2 * P - 1) / (2 * P)));
        const size_t smem = (size_t)P * d.N * 16;
        auto launch = [&](auto kern, int nt) { kern<<<g, nt, smem, c->stream>>>(a); };
#define PINT_REGL(LGV, PV)                                                                       \
    if (d.reg_lg == LGV && P == PV) {                                                            \
        if (K == 0) launch(dstreg::k_dst_reg<0, LGV, PV>, dstreg::reg_threads<LGV, PV>());      \
        else launch(dstreg::k_dst_reg<1, LGV, PV>, dstreg::reg_threads<LGV, PV>());             \
    }
        PINT_REGL(8, 16) PINT_REGL(9, 8) PINT_REGL(9, 4) PINT_REGL(10, 4) PINT_REGL(10, 2)
        PINT_REGL(11, 2) PINT_REGL(12, 1) PINT_REGL(13, 1) PINT_REGL(11, 4) PINT_REGL(12, 2)
#undef PINT_REGL
    } else if (d.fast) {
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
