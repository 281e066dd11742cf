// Fused Uzawa residual operators as persistent TMA band kernels.
//
// Reference (solvers.py:224, 227-229; operators.py:78-99):
//   r1_n = (K u - A p - f)_n  = ((M u_n - M u_{n-1}) - s_n (A_n p_n)) - f_n
//   z_n  = (f - K^T p - (K u + K^T u + A u))_n
//        = (f_n - (M p_n - M p_{n+1})) - (((M u_n - M u_{n-1}) + (M u_n - M u_{n+1})) + s_n (A_n u_n))
// (first / last step without the missing neighbour), bit-identical to the
// reference (CSR order, no FMA).
//
// A CTA owns a band of H rows of the plane and a chunk of G consecutive time
// steps; a producer warp streams the (H+2)-row bands of u_q and p_q with 1D
// TMA bulk copies into a two-stage ring while the consumer threads march
// down their column with a 3x3 register window and march forward in time
// carrying M u, M p and A u of the previous planes in registers, so every
// plane of u and p crosses HBM once and f once.  The apply-A_ref kernel of
// the Schur preconditioner (schur.py:72) uses the same machinery.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "band.cuh"
#include "pint_device.cuh"
#include "pint_internal.cuh"

#ifndef PINT_VARIANT
#define PINT_VARIANT exact
#endif

namespace pint {
namespace PINT_VARIANT {  // compiled as pint::exact (-fmad=false) and pint::fast (FMA)

namespace {

constexpr int TB_MAXSTAGE = 4;
constexpr int TB_NT = 256;

enum TShape : int { TS_FULL = 0, TS_SEVEN = 1, TS_FIVE = 2 };

template <int SH>
__device__ __forceinline__ constexpr bool tused(int k) {
    return SH == TS_FULL ? true
         : SH == TS_SEVEN ? (k != 2 && k != 6)
                          : (k == 1 || k == 3 || k == 4 || k == 5 || k == 7);
}

template <int SH>
__device__ __forceinline__ double wsum(const double* c, const double* a, const double* b,
                                       const double* cc) {
    double s = 0.0;
    bool first = true;
#define PINT_T(K, V)                 \
    if (tused<SH>(K)) {              \
        const double t_ = c[K] * (V); \
        s = first ? t_ : s + t_;     \
        first = false;               \
    }
    PINT_T(0, a[0])
    PINT_T(1, a[1])
    PINT_T(2, a[2])
    PINT_T(3, b[0])
    PINT_T(4, b[1])
    PINT_T(5, b[2])
    PINT_T(6, cc[0])
    PINT_T(7, cc[1])
    PINT_T(8, cc[2])
#undef PINT_T
    return s;
}

__device__ __forceinline__ int tb_shift(long long pb, int m, int first, int r_lo) {
    const long long e0 = pb + (long long)r_lo * m;
    return ((r_lo - first) * m - (int)(e0 & 1)) & 1;
}

__device__ __forceinline__ void tb_issue(double* buf, const double* slab, long long pb, int m,
                                         int first, int r_lo, int r_hi, uint64_t* bar) {
    const Span s = span_of(pb + (long long)r_lo * m, pb + (long long)r_hi * m);
    double* dst = buf + tb_shift(pb, m, first, r_lo) + (r_lo - first) * m - s.off;
    bulk_g2s(dst, slab + s.g0, s.bytes, bar);
}

struct TopParams {
    int m, N, G, nchunks, nbands, H, stages;
    int words;   // one halo band (H+2 rows) of u or p
    int wordsf;  // one band (H rows) of f
    int one_a;   // every step uses stencil a0 (the proportional / constant case)
    int qmin, qmax;  // planes addressable through u/p: -1 / N when a neighbour rank's ghost plane is present
    double cmass[9], a0[9];  // by value: kernel-parameter (constant bank) operands
    const double* mass;
    const double* ast;
    const int* asid;
    const double* ascale;
    const double* u;
    const double* p;
    const double* f;
    double* out;
};

// window row loader: values of `row` (plane row gy, staged) at x-1, x, x+1, zero outside
__device__ __forceinline__ void wrow(const double* row, bool in, int x, bool w, bool e,
                                     double* v) {
    v[0] = (in && w) ? row[x - 1] : 0.0;
    v[1] = in ? row[x] : 0.0;
    v[2] = (in && e) ? row[x + 1] : 0.0;
}

// OP 0: r1 (needs u, p);  OP 1: z (needs u, p, look-ahead)
template <int OP, int CPT, int H, int SHM, int SHA, int ONEA>
__global__ void __launch_bounds__(TB_NT + 32, 2) k_band_timeop(TopParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[TB_MAXSTAGE], empty[TB_MAXSTAGE];
    __shared__ double meta[TB_MAXSTAGE][10];  // A_q stencil + scale, producer-written
    const int m = P.m, N = P.N, S = P.stages;
    const long long n = (long long)m * m;
    const int units = P.nbands * P.nchunks;
    const int tid = threadIdx.x;
    // alignment parity of each slab's base (see span_of): offsets relative to 16-B aligned bases
    const int bou = (int)((reinterpret_cast<uintptr_t>(P.u) >> 3) & 1);
    const int bop = (int)((reinterpret_cast<uintptr_t>(P.p) >> 3) & 1);
    const int bof = (int)((reinterpret_cast<uintptr_t>(P.f) >> 3) & 1);
    // unit u -> band j (fast), chunk c
    auto unit = [&](int u, int& y0, int& y1, int& n0, int& n1) {
        const int c = u / P.nbands, j = u - c * P.nbands;
        y0 = j * H;
        y1 = min(m, y0 + H);
        n0 = c * P.G;
        n1 = min(N, n0 + P.G);
    };
    // staged planes of a unit: r1: q in [max(0,n0-1), n1);  z: q in [max(0,n0-1), min(N, n1+1))
    auto qrange = [&](int n0, int n1, int& qs, int& qe) {
        qs = max(P.qmin, n0 - 1);
        qe = OP == 0 ? n1 : min(P.qmax + 1, n1 + 1);
    };
    const int wst = 2 * P.words + P.wordsf;
    auto ustage = [&](int s) { return smem + s * wst; };
    auto pstage = [&](int s) { return smem + s * wst + P.words; };
    auto fstage = [&](int s) { return smem + s * wst + 2 * P.words; };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid >= TB_NT) {  // ---- producer warp ----
        if (tid == TB_NT) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int y0, y1, n0, n1, qs, qe;
                unit(u, y0, y1, n0, n1);
                qrange(n0, n1, qs, qe);
                const int first = y0 - 1, lo = max(0, first), hi = min(m, y1 + 1);
                for (int q = qs; q < qe; ++q, ++k) {
                    const int s = k % S;
                    if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                    const long long pb = q * n;
                    const Span sp = span_of(pb + bou + (long long)lo * m, pb + bou + (long long)hi * m);
                    const Span spp = span_of(pb + bop + (long long)lo * m, pb + bop + (long long)hi * m);
                    const bool need_p = OP == 1 || q >= n0;
                    // f of the output plane: r1 -> q, z -> q-1
                    const int t = OP == 0 ? q : q - 1;
                    const bool need_f = t >= n0 && t < n1;
                    const long long tb = (long long)t * n;
                    const uint32_t fbytes =
                        need_f ? span_of(tb + bof + (long long)y0 * m, tb + bof + (long long)y1 * m).bytes
                               : 0;
                    {
                        const double* a = P.ast + 9 * __ldg(P.asid + q);
#pragma unroll
                        for (int t2 = 0; t2 < 9; ++t2) meta[s][t2] = __ldg(a + t2);
                        meta[s][9] = __ldg(P.ascale + q);
                    }
                    mbar_expect_tx(&full[s], sp.bytes + (need_p ? spp.bytes : 0) + fbytes);
                    tb_issue(ustage(s), P.u - bou, pb + bou, m, first, lo, hi, &full[s]);
                    if (need_p) tb_issue(pstage(s), P.p - bop, pb + bop, m, first, lo, hi, &full[s]);
                    if (need_f) tb_issue(fstage(s), P.f - bof, tb + bof, m, y0, y0, y1, &full[s]);
                }
            }
        }
        return;
    }
    // ---- consumers ----
    const double* cm = P.cmass;
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int y0, y1, n0, n1, qs, qe;
        unit(u, y0, y1, n0, n1);
        qrange(n0, n1, qs, qe);
        const int first = y0 - 1, lo = max(0, first);
        const int nrow = y1 - y0;
        // carries per (column j, row r)
        double mu_prev[CPT][H], mu_cur[CPT][H], mp_cur[CPT][H], au_cur[CPT][H];
        const int qlast = OP == 0 ? qe - 1 : qe;  // z: one extra (virtual) step at q = N
        for (int q = qs; q <= qlast; ++q) {
            const bool staged = q < qe;
            const int s = k % S;
            const long long pb = q * n;
            double ca[9];
            double sc = 0.0;
            // z output plane t = q-1, r1 output plane t = q
            const int t = OP == 0 ? q : q - 1;
            const bool emit = t >= n0 && t < n1;
            if (staged) {
                mbar_wait(&full[s], (k / S) & 1);
                if (!ONEA) {
#pragma unroll
                    for (int t2 = 0; t2 < 9; ++t2) ca[t2] = meta[s][t2];
                }
                sc = meta[s][9];
            }
            const double* us = ustage(s) + tb_shift(pb + bou, m, first, lo);
            const double* ps = pstage(s) + tb_shift(pb + bop, m, first, lo);
            const double* fs = fstage(s) + tb_shift((long long)t * n + bof, m, y0, y0);
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int x = tid + j * TB_NT;
                if (x >= m) continue;
                const bool w = x > 0, e = x < m - 1;
                double ua[3], ub[3], uc[3], pa[3], pbv[3], pc[3];
                if (staged) {
                    wrow(us, first >= 0, x, w, e, ua);
                    wrow(us + m, true, x, w, e, ub);
                    if (OP == 1 || q >= n0) {
                        wrow(ps, first >= 0, x, w, e, pa);
                        wrow(ps + m, true, x, w, e, pbv);
                    }
                }
#pragma unroll
                for (int r = 0; r < H; ++r) {
                    if (r >= nrow) continue;
                    const int gy = y0 + r;
                    double mu = 0.0, mp = 0.0, au = 0.0, ap = 0.0;
                    if (staged) {
                        wrow(us + (r + 2) * m, gy + 1 < m, x, w, e, uc);
                        mu = wsum<SHM>(cm, ua, ub, uc);
                        if (OP == 1) au = sc * wsum<SHA>(ONEA ? P.a0 : ca, ua, ub, uc);
                        if (OP == 1 || q >= n0) {
                            wrow(ps + (r + 2) * m, gy + 1 < m, x, w, e, pc);
                            if (OP == 1) mp = wsum<SHM>(cm, pa, pbv, pc);
                            else ap = sc * wsum<SHA>(ONEA ? P.a0 : ca, pa, pbv, pc);
                        }
                    }
                    double* o = P.out + t * n + (long long)gy * m + x;
                    if (OP == 0) {
                        if (emit) {
                            const double ku = t - 1 >= P.qmin ? mu - mu_prev[j][r] : mu;
                            *o = (ku - ap) - fs[r * m + x];
                        }
                        mu_prev[j][r] = mu;
                    } else {
                        if (emit) {
                            const bool has_next = t + 1 <= P.qmax;
                            const double ktp = has_next ? mp_cur[j][r] - mp : mp_cur[j][r];
                            const double ku =
                                t - 1 >= P.qmin ? mu_cur[j][r] - mu_prev[j][r] : mu_cur[j][r];
                            const double ktu = has_next ? mu_cur[j][r] - mu : mu_cur[j][r];
                            // the virtual step q = N has no stage: f_{N-1} straight from HBM
                            const double fval =
                                staged ? fs[r * m + x] : __ldg(P.f + t * n + (long long)gy * m + x);
                            *o = (fval - ktp) - ((ku + ktu) + au_cur[j][r]);
                        }
                        mu_prev[j][r] = mu_cur[j][r];
                        mu_cur[j][r] = mu;
                        mp_cur[j][r] = mp;
                        au_cur[j][r] = au;
                    }
                    if (staged) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            ua[i] = ub[i];
                            ub[i] = uc[i];
                            pa[i] = pbv[i];
                            pbv[i] = pc[i];
                        }
                    }
                }
            }
            if (staged) {
                consumer_sync<TB_NT>();
                if (tid == 0) mbar_arrive(&empty[s]);
                ++k;
            }
        }
    }
}

// Paired-column form (default): consumer thread t owns columns 2t and 2t+1,
// sharing a 4-column register window of u and p (2 loads per point instead
// of 3) and interleaving two independent CSR-order sums.
template <int OP, int NT, int H, int SHM, int SHA, int ONEA>
__global__ void __launch_bounds__(NT + 32, 2) k_band_timeop2(TopParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[TB_MAXSTAGE], empty[TB_MAXSTAGE];
    __shared__ double meta[TB_MAXSTAGE][10];
    const int m = P.m, N = P.N, S = P.stages;
    const long long n = (long long)m * m;
    const int units = P.nbands * P.nchunks;
    const int tid = threadIdx.x;
    const int bou = (int)((reinterpret_cast<uintptr_t>(P.u) >> 3) & 1);
    const int bop = (int)((reinterpret_cast<uintptr_t>(P.p) >> 3) & 1);
    const int bof = (int)((reinterpret_cast<uintptr_t>(P.f) >> 3) & 1);
    auto unit = [&](int u, int& y0, int& y1, int& n0, int& n1) {
        const int c = u / P.nbands, j = u - c * P.nbands;
        y0 = j * H;
        y1 = min(m, y0 + H);
        n0 = c * P.G;
        n1 = min(N, n0 + P.G);
    };
    auto qrange = [&](int n0, int n1, int& qs, int& qe) {
        qs = max(P.qmin, n0 - 1);
        qe = OP == 0 ? n1 : min(P.qmax + 1, n1 + 1);
    };
    const int wst = 2 * P.words + P.wordsf;
    auto ustage = [&](int s) { return smem + s * wst; };
    auto pstage = [&](int s) { return smem + s * wst + P.words; };
    auto fstage = [&](int s) { return smem + s * wst + 2 * P.words; };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid >= NT) {  // ---- producer warp (as k_band_timeop) ----
        if (tid == NT) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int y0, y1, n0, n1, qs, qe;
                unit(u, y0, y1, n0, n1);
                qrange(n0, n1, qs, qe);
                const int first = y0 - 1, lo = max(0, first), hi = min(m, y1 + 1);
                for (int q = qs; q < qe; ++q, ++k) {
                    const int s = k % S;
                    if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                    const long long pb = q * n;
                    const Span sp = span_of(pb + bou + (long long)lo * m, pb + bou + (long long)hi * m);
                    const Span spp = span_of(pb + bop + (long long)lo * m, pb + bop + (long long)hi * m);
                    const bool need_p = OP == 1 || q >= n0;
                    const int t = OP == 0 ? q : q - 1;
                    const bool need_f = t >= n0 && t < n1;
                    const long long tb = (long long)t * n;
                    const uint32_t fbytes =
                        need_f ? span_of(tb + bof + (long long)y0 * m, tb + bof + (long long)y1 * m).bytes
                               : 0;
                    if (!ONEA) {
                        const double* a = P.ast + 9 * __ldg(P.asid + q);
#pragma unroll
                        for (int t2 = 0; t2 < 9; ++t2) meta[s][t2] = __ldg(a + t2);
                    }
                    meta[s][9] = __ldg(P.ascale + q);
                    mbar_expect_tx(&full[s], sp.bytes + (need_p ? spp.bytes : 0) + fbytes);
                    tb_issue(ustage(s), P.u - bou, pb + bou, m, first, lo, hi, &full[s]);
                    if (need_p) tb_issue(pstage(s), P.p - bop, pb + bop, m, first, lo, hi, &full[s]);
                    if (need_f) tb_issue(fstage(s), P.f - bof, tb + bof, m, y0, y0, y1, &full[s]);
                }
            }
        }
        return;
    }
    const double* cm = P.cmass;
    const int t0c = 2 * tid;            // columns xa = 2t, xb = 2t+1
    const bool act = t0c < m;
    const bool hb = t0c + 1 < m;        // column xb exists
    const bool hl = t0c >= 1;           // column 2t-1 exists
    const bool hr = t0c + 2 < m;        // column 2t+2 exists
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int y0, y1, n0, n1, qs, qe;
        unit(u, y0, y1, n0, n1);
        qrange(n0, n1, qs, qe);
        const int first = y0 - 1, lo = max(0, first);
        const int nrow = y1 - y0;
        // interior band: H rows with both halo rows inside the plane (no row predicates)
        // (r1 is at the HBM roofline: it keeps one row-predicated body, smaller code)
        const bool interior = OP == 1 && nrow == H && y0 > 0 && y1 < m;
        // carried state, zero-initialised: a missing previous plane enters as
        // x - (+0) == x, bit-identical to the reference's one-sided first step
        double mu_prev[2][H], mu_cur[2][H], mp_cur[2][H], au_cur[2][H];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int r = 0; r < H; ++r) {
                mu_prev[c][r] = 0.0;
                mu_cur[c][r] = 0.0;
                mp_cur[c][r] = 0.0;
                au_cur[c][r] = 0.0;
            }
        // one staged plane q; IN: interior band, EM: plane q completes output step t
        // (r1: t = q >= n0; z: t = q-1 >= n0, the first one or two planes only warm up)
        auto step = [&](auto in_tag, auto em_tag, int q) {
            constexpr bool IN = decltype(in_tag)::value;
            constexpr bool EM = decltype(em_tag)::value;
            const int s = k % S;
            const long long pb = q * n;
            const int t = OP == 0 ? q : q - 1;
            double ca[9];
            mbar_wait(&full[s], (k / S) & 1);
            if (!ONEA) {
#pragma unroll
                for (int t2 = 0; t2 < 9; ++t2) ca[t2] = meta[s][t2];
            }
            const double sc = meta[s][9];
            const double* A = ONEA ? P.a0 : ca;
            if (act) {
                const double* us = ustage(s) + tb_shift(pb + bou, m, first, lo) + t0c;
                const double* ps = pstage(s) + tb_shift(pb + bop, m, first, lo) + t0c;
                const double* fs = fstage(s) + tb_shift((long long)t * n + bof, m, y0, y0) + t0c;
                // 4-wide window rows: columns 2t-1, 2t, 2t+1, 2t+2
                auto wr4 = [&](const double* row, bool in, double* v) {
                    v[0] = (in && hl) ? row[-1] : 0.0;
                    v[1] = in ? row[0] : 0.0;
                    v[2] = (in && hb) ? row[1] : 0.0;
                    v[3] = (in && hr) ? row[2] : 0.0;
                };
                constexpr bool NEED_P = OP == 1 || EM;  // r1 reads p of the emitted steps only
                double ua[4], ub[4], uc[4], pa[4], pbv[4], pc[4];
                wr4(us, IN || first >= 0, ua);
                wr4(us + m, true, ub);
                if (NEED_P) {
                    wr4(ps, IN || first >= 0, pa);
                    wr4(ps + m, true, pbv);
                }
#pragma unroll
                for (int r = 0; r < H; ++r) {
                    if (!IN && r >= nrow) continue;
                    const int gy = y0 + r;
                    double mu[2], mp[2] = {0.0, 0.0}, au[2] = {0.0, 0.0}, ap[2] = {0.0, 0.0};
                    wr4(us + (r + 2) * m, IN || gy + 1 < m, uc);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        mu[c] = wsum<SHM>(cm, ua + c, ub + c, uc + c);
                        if (OP == 1) au[c] = sc * wsum<SHA>(A, ua + c, ub + c, uc + c);
                    }
                    if (NEED_P) {
                        wr4(ps + (r + 2) * m, IN || gy + 1 < m, pc);
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            if (OP == 1) mp[c] = wsum<SHM>(cm, pa + c, pbv + c, pc + c);
                            else ap[c] = sc * wsum<SHA>(A, pa + c, pbv + c, pc + c);
                        }
                    }
                    double* o = P.out + t * n + (long long)gy * m + t0c;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const bool ok = c == 0 || hb;
                        if (OP == 0) {
                            if (EM && ok) o[c] = ((mu[c] - mu_prev[c][r]) - ap[c]) - fs[r * m + c];
                            mu_prev[c][r] = mu[c];
                        } else {
                            if (EM && ok) {
                                // a staged plane q = t+1 always exists here (has_next)
                                const double ktp = mp_cur[c][r] - mp[c];
                                const double ku = mu_cur[c][r] - mu_prev[c][r];
                                const double ktu = mu_cur[c][r] - mu[c];
                                o[c] = (fs[r * m + c] - ktp) - ((ku + ktu) + au_cur[c][r]);
                            }
                            mu_prev[c][r] = mu_cur[c][r];
                            mu_cur[c][r] = mu[c];
                            mp_cur[c][r] = mp[c];
                            au_cur[c][r] = au[c];
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        ua[i] = ub[i];
                        ub[i] = uc[i];
                        pa[i] = pbv[i];
                        pbv[i] = pc[i];
                    }
                }
            }
            consumer_sync<NT>();
            if (tid == 0) mbar_arrive(&empty[s]);
            ++k;
        };
        using TT = std::integral_constant<bool, true>;
        using FF = std::integral_constant<bool, false>;
        const int qem = min(qe, OP == 0 ? n0 : n0 + 1);
        int q = qs;
        for (; q < qem; ++q) {
            if (interior) step(TT{}, FF{}, q);
            else step(FF{}, FF{}, q);
        }
        for (; q < qe; ++q) {
            if (interior) step(TT{}, TT{}, q);
            else step(FF{}, TT{}, q);
        }
        if (OP == 1 && act) {
            // last step of the time axis (t = qe-1 = qmax, no plane t+1): K^T has
            // no next-step term
            const int t = qe - 1;
            if (t >= n0 && t < n1 && qe > P.qmax) {
#pragma unroll
                for (int r = 0; r < H; ++r) {
                    if (r >= nrow) continue;
                    const int gy = y0 + r;
                    double* o = P.out + t * n + (long long)gy * m + t0c;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (!(c == 0 || hb)) continue;
                        const double ku = mu_cur[c][r] - mu_prev[c][r];
                        const double fval = __ldg(P.f + t * n + (long long)gy * m + t0c + c);
                        o[c] = (fval - mp_cur[c][r]) - ((ku + mu_cur[c][r]) + au_cur[c][r]);
                    }
                }
            }
        }
    }
}

// out_plane = A stencil (one stencil for all planes) * in_plane, planes [0, count)
struct ApplyParams {
    int m, count, nbands, H, stages, words;
    double cst[9];
    const double* st;
    const double* in;
    double* out;
};

template <int SH, int CPT, int H>
__global__ void __launch_bounds__(TB_NT + 32) k_band_apply(ApplyParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[TB_MAXSTAGE], empty[TB_MAXSTAGE];
    const int m = P.m, S = P.stages;
    const long long n = (long long)m * m;
    const int units = P.nbands * P.count;
    const int tid = threadIdx.x;
    const int boi = (int)((reinterpret_cast<uintptr_t>(P.in) >> 3) & 1);
    auto unit = [&](int u, int& plane, int& y0, int& y1) {
        plane = u / P.nbands;
        const int j = u - plane * P.nbands;
        y0 = j * H;
        y1 = min(m, y0 + H);
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid >= TB_NT) {
        if (tid == TB_NT) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                int plane, y0, y1;
                unit(u, plane, y0, y1);
                const long long pb = plane * n + boi;
                const int first = y0 - 1, lo = max(0, first), hi = min(m, y1 + 1);
                const Span sp = span_of(pb + (long long)lo * m, pb + (long long)hi * m);
                mbar_expect_tx(&full[s], sp.bytes);
                tb_issue(smem + s * P.words, P.in - boi, pb, m, first, lo, hi, &full[s]);
            }
        }
        return;
    }
    const double* ca = P.cst;
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % S;
        int plane, y0, y1;
        unit(u, plane, y0, y1);
        const long long pb = plane * n;
        const int first = y0 - 1, lo = max(0, first);
        const int nrow = y1 - y0;
        mbar_wait(&full[s], (k / S) & 1);
        const double* vs = smem + s * P.words + tb_shift(pb + boi, m, first, lo);
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int x = tid + j * TB_NT;
            if (x >= m) continue;
            const bool w = x > 0, e = x < m - 1;
            double a[3], b[3], c[3];
            wrow(vs, first >= 0, x, w, e, a);
            wrow(vs + m, true, x, w, e, b);
#pragma unroll
            for (int r = 0; r < H; ++r) {
                if (r >= nrow) continue;
                const int gy = y0 + r;
                wrow(vs + (r + 2) * m, gy + 1 < m, x, w, e, c);
                P.out[pb + (long long)gy * m + x] = wsum<SH>(ca, a, b, c);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    a[i] = b[i];
                    b[i] = c[i];
                }
            }
        }
        consumer_sync<TB_NT>();
        if (tid == 0) mbar_arrive(&empty[s]);
    }
}

int sms_count() {
    static int v = 0;
    if (v == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
    }
    return v;
}

int shape_of(const double* st9_host) {
    const double* z = st9_host;
    if (z[0] == 0.0 && z[2] == 0.0 && z[6] == 0.0 && z[8] == 0.0) return TS_FIVE;
    if (z[2] == 0.0 && z[6] == 0.0) return TS_SEVEN;
    return TS_FULL;
}

int grid_for(size_t smem, int units) {
    int per = (int)((227 * 1024) / (smem + 1024));
    per = std::max(1, std::min(per, 4));
    if (const char* e = getenv("PINT_CTAS")) per = std::max(1, std::min(per, atoi(e)));
    return std::max(1, std::min(units, sms_count() * per));
}

template <int OP, int CPT, int H, int SHM, int SHA>
void launch_timeop_cfg(pint_ctx* c, const TopParams& P, size_t smem, int grid) {
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_timeop<OP, CPT, H, SHM, SHA, 0>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_timeop<OP, CPT, H, SHM, SHA, 1>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    if (P.one_a)
        k_band_timeop<OP, CPT, H, SHM, SHA, 1><<<grid, TB_NT + 32, smem, c->stream>>>(P);
    else
        k_band_timeop<OP, CPT, H, SHM, SHA, 0><<<grid, TB_NT + 32, smem, c->stream>>>(P);
}

template <int OP, int NT, int SHM, int SHA>
void launch_timeop2_cfg(pint_ctx* c, const TopParams& P, size_t smem, int units) {
    constexpr int H = 4;
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_timeop2<OP, NT, H, SHM, SHA, 0>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_timeop2<OP, NT, H, SHM, SHA, 1>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    int occ = 0;
    if (P.one_a) {
        PINT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ, k_band_timeop2<OP, NT, H, SHM, SHA, 1>, NT + 32, smem));
    } else {
        PINT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ, k_band_timeop2<OP, NT, H, SHM, SHA, 0>, NT + 32, smem));
    }
    occ = std::max(1, occ);
    if (const char* e = getenv("PINT_CTAS")) occ = std::max(1, std::min(occ, atoi(e)));
    const int grid = std::max(1, std::min(units, sms_count() * occ));
    if (P.one_a)
        k_band_timeop2<OP, NT, H, SHM, SHA, 1><<<grid, NT + 32, smem, c->stream>>>(P);
    else
        k_band_timeop2<OP, NT, H, SHM, SHA, 0><<<grid, NT + 32, smem, c->stream>>>(P);
}

template <int OP, int NT>
void launch_timeop2_shapes(pint_ctx* c, const TopParams& P, size_t smem, int units, int shm,
                           int sha) {
    if (shm == TS_SEVEN && sha == TS_FIVE) launch_timeop2_cfg<OP, NT, TS_SEVEN, TS_FIVE>(c, P, smem, units);
    else if (shm == TS_SEVEN) launch_timeop2_cfg<OP, NT, TS_SEVEN, TS_FULL>(c, P, smem, units);
    else launch_timeop2_cfg<OP, NT, TS_FULL, TS_FULL>(c, P, smem, units);
}

template <int OP, int CPT>
void launch_timeop_shapes(pint_ctx* c, const TopParams& P, size_t smem, int grid, int shm,
                          int sha) {
    constexpr int H = 4;  // z carries 4 planes of state per row: keep it in registers
    if (shm == TS_SEVEN && sha == TS_FIVE) launch_timeop_cfg<OP, CPT, H, TS_SEVEN, TS_FIVE>(c, P, smem, grid);
    else if (shm == TS_SEVEN) launch_timeop_cfg<OP, CPT, H, TS_SEVEN, TS_FULL>(c, P, smem, grid);
    else launch_timeop_cfg<OP, CPT, H, TS_FULL, TS_FULL>(c, P, smem, grid);
}

}  // namespace

bool band_timeop_supported(const pint_ctx* c) { return c->dims == 2 && c->m >= 64 && c->m <= 512; }

void launch_band_timeop(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                        double* out) {
    TopParams P{};
    P.m = c->m;
    P.N = c->N;
    P.H = 4;
    // long time chunks amortise the extra (halo) planes; keep >= 4 units per CTA slot
    P.G = 32;
    {
        const int nb = (P.m + P.H - 1) / P.H;
        while (P.G > 4 && (long long)nb * ((P.N + P.G - 1) / P.G) < 4LL * 2 * sms_count()) P.G /= 2;
    }
    if (const char* e = getenv("PINT_TOP_G")) P.G = std::max(1, atoi(e));
    P.nbands = (P.m + P.H - 1) / P.H;
    P.nchunks = (P.N + P.G - 1) / P.G;
    P.words = band_words(P.H + 2, P.m);
    P.wordsf = band_words(P.H, P.m);
    {
        // deepest ring that keeps two CTAs per SM
        const size_t wst = sizeof(double) * (2 * (size_t)P.words + P.wordsf);
        int st = (int)((110 * 1024) / wst);
        P.stages = std::max(2, std::min(TB_MAXSTAGE, st));
        const char* e = getenv("PINT_STAGES");
        if (e) P.stages = std::max(2, std::min(TB_MAXSTAGE, atoi(e)));
    }
    P.qmin = c->has_prev ? -1 : 0;
    P.qmax = c->has_next ? c->N : c->N - 1;
    P.mass = c->d_mass;
    for (int q = 0; q < 9; ++q) P.cmass[q] = c->h_mass[q];
    P.one_a = c->n_a == 1;
    for (int q = 0; q < 9; ++q) P.a0[q] = c->h_ast[q];
    P.ast = c->d_ast;
    P.asid = c->d_asid;
    P.ascale = c->d_ascale;
    P.u = u;
    P.p = p;
    P.f = f;
    P.out = out;
    const size_t smem = sizeof(double) * (size_t)P.stages * (2 * P.words + P.wordsf);
    const int grid = grid_for(smem, P.nbands * P.nchunks);
    const int shm = shape_of(c->h_mass.data());
    int sha = TS_FIVE;
    for (int s = 0; s < c->n_a; ++s) sha = std::min(sha, shape_of(&c->h_ast[9 * s]));
    ProfScope prof(c, op == OP_R1 ? K_TIMEOP_R1 : K_TIMEOP_Z, 8.0 * 4 * (double)c->N * c->n);
    const bool wide = P.m > 256;
    if (!getenv("PINT_TOP1")) {
        const int units = P.nbands * P.nchunks;
        const int nt = ((P.m + 1) / 2 + 31) / 32 * 32;   // one thread per column pair
        if (op == OP_R1) {
            if (nt <= 64) launch_timeop2_shapes<0, 64>(c, P, smem, units, shm, sha);
            else if (nt <= 128) launch_timeop2_shapes<0, 128>(c, P, smem, units, shm, sha);
            else launch_timeop2_shapes<0, 256>(c, P, smem, units, shm, sha);
        } else {
            if (nt <= 64) launch_timeop2_shapes<1, 64>(c, P, smem, units, shm, sha);
            else if (nt <= 128) launch_timeop2_shapes<1, 128>(c, P, smem, units, shm, sha);
            else launch_timeop2_shapes<1, 256>(c, P, smem, units, shm, sha);
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        return;
    }
    if (op == OP_R1) {
        if (wide) launch_timeop_shapes<0, 2>(c, P, smem, grid, shm, sha);
        else launch_timeop_shapes<0, 1>(c, P, smem, grid, shm, sha);
    } else {
        if (wide) launch_timeop_shapes<1, 2>(c, P, smem, grid, shm, sha);
        else launch_timeop_shapes<1, 1>(c, P, smem, grid, shm, sha);
    }
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_band_apply(pint_ctx* c, const double* st_dev, const double* st_host, const double* in,
                       double* out, int count) {
    ApplyParams P{};
    P.m = c->m;
    P.count = count;
    P.stages = 2;
    constexpr int H = 8;
    P.H = H;
    P.nbands = (P.m + H - 1) / H;
    P.words = band_words(H + 2, P.m);
    P.st = st_dev;
    for (int q = 0; q < 9; ++q) P.cst[q] = st_host[q];
    P.in = in;
    P.out = out;
    const size_t smem = sizeof(double) * (size_t)P.stages * P.words;
    const int grid = grid_for(smem, P.nbands * count);
    const int sh = shape_of(st_host);
    const bool wide = P.m > 256;
    ProfScope prof(c, K_AREF, 16.0 * (double)count * c->n);
#define PINT_AP(SHV, CPTV)                                                                      \
    {                                                                                           \
        static bool attr = false;                                                               \
        if (!attr) {                                                                            \
            PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_apply<SHV, CPTV, H>,                    \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                                 200 * 1024));                                  \
            attr = true;                                                                        \
        }                                                                                       \
        k_band_apply<SHV, CPTV, H><<<grid, TB_NT + 32, smem, c->stream>>>(P);                   \
    }
    if (sh == TS_FIVE) {
        if (wide) PINT_AP(TS_FIVE, 2) else PINT_AP(TS_FIVE, 1)
    } else if (sh == TS_SEVEN) {
        if (wide) PINT_AP(TS_SEVEN, 2) else PINT_AP(TS_SEVEN, 1)
    } else {
        if (wide) PINT_AP(TS_FULL, 2) else PINT_AP(TS_FULL, 1)
    }
#undef PINT_AP
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace PINT_VARIANT
}  // namespace pint
