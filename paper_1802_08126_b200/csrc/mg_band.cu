// Batched multigrid V-cycle, B200 edition.
//
// Reference: MgVCycleSolver._vcycle / apply (spatial.py:148-169), 2D
// hierarchy of build_mg_hierarchy (spatial.py:100-113): one damped-Jacobi
// pre- and post-sweep (dinv = damping/diag, spatial.py:142), restriction P^T
// (unscaled bilinear full weighting), prolongation P = kron(P1, P1)
// (spatial.py:75-84,110), Galerkin coarse stencils (host tables), 1x1 direct
// coarsest solve b/a (SpdFactor, spatial.py:143,149-150).  Every plane of the
// batch (all N time steps for A~, all N DST modes for H~) goes through the
// same launches.
//
// Large levels (m >= 64) stream through persistent band kernels: a CTA owns
// a row band of one plane at a time, the band's inputs arrive by TMA bulk
// copy into a double-buffered shared-memory ring (band.cuh) while the
// previous band is computed, so HBM latency is hidden without occupancy.
//   k_band_pre : x0 = dinv*b, r = b - A x0, b_c = P^T r    (one pass over b)
//   k_band_post: x = x0 + P e, x += dinv*(b - A x), epilogue (one pass)
// Small levels (m <= 63) run in k_mg_tail: one CTA per plane holds every
// remaining level in shared memory and does descend, coarsest solve and
// ascend in one launch (for BASELINE config 1 that is the whole V-cycle).
//
// Bit-exactness: every row sum is evaluated in scipy's CSR column order
// starting from 0, without FMA (-fmad=false); terms whose coefficient is an
// exact zero on every plane (the SE/NW entries of the P1 diagonal split, the
// four diagonal entries of the stiffness) are skipped, which adds +-0 and so
// cannot change a non-zero sum.
#include <type_traits>
#include <algorithm>
#include <cstdlib>

#include "band.cuh"
#include "pint_device.cuh"
#include "pint_internal.cuh"

#ifndef PINT_VARIANT
#define PINT_VARIANT exact
#endif
#ifndef PINT_FAST
#define PINT_FAST 0
#endif

namespace pint {
namespace PINT_VARIANT {  // compiled as pint::exact (-fmad=false) and pint::fast (FMA)

// x / y out of line: a select between v * (1/tau) and v / tau is otherwise
// if-converted and the division evaluated for every point
__device__ __noinline__ double band_div(double x, double y) { return x / y; }

constexpr int BT = 256;       // threads of the band kernels
constexpr int TT = 512;       // threads of the tail kernel

// stencil shapes: which of the 9 CSR positions can be non-zero
enum Shape : int { SH_FULL = 0, SH_SEVEN = 1, SH_FIVE = 2 };

template <int SH>
__device__ __forceinline__ constexpr bool used(int k) {
    return SH == SH_FULL ? true
         : SH == SH_SEVEN ? (k != 2 && k != 6)
                          : (k == 1 || k == 3 || k == 4 || k == 5 || k == 7);
}

// CSR-ordered row sum at column x; rm/r0/rp point at column 0 of rows y-1,
// y, y+1; hs/hn: rows y-1 / y+1 exist; w/e: columns x-1 / x+1 exist.
template <int SH>
__device__ __forceinline__ double row_sum(const double* c, const double* rm, const double* r0,
                                          const double* rp, int x, bool hs, bool hn, bool w,
                                          bool e) {
    double s = 0.0;
    bool first = true;
    auto acc = [&](double t) {
        if (first) {
            s = t;
            first = false;
        } else {
            s = s + t;
        }
    };
    if (used<SH>(0)) acc(c[0] * ((hs && w) ? rm[x - 1] : 0.0));
    if (used<SH>(1)) acc(c[1] * (hs ? rm[x] : 0.0));
    if (used<SH>(2)) acc(c[2] * ((hs && e) ? rm[x + 1] : 0.0));
    if (used<SH>(3)) acc(c[3] * (w ? r0[x - 1] : 0.0));
    if (used<SH>(4)) acc(c[4] * r0[x]);
    if (used<SH>(5)) acc(c[5] * (e ? r0[x + 1] : 0.0));
    if (used<SH>(6)) acc(c[6] * ((hn && w) ? rp[x - 1] : 0.0));
    if (used<SH>(7)) acc(c[7] * (hn ? rp[x] : 0.0));
    if (used<SH>(8)) acc(c[8] * ((hn && e) ? rp[x + 1] : 0.0));
    return s;
}

// logical row pointer of a band buffer whose slot 0 holds plane row `first`,
// filled by a copy of rows [r_lo, r_hi) of plane `pb` (element base of plane)
struct BandView {
    const double* p;  // &row(first)[0]
    __device__ __forceinline__ const double* row(int slot, int m) const { return p + slot * m; }
};

// element shift that makes the bulk-copy destination 16-byte aligned
__device__ __forceinline__ int band_shift(long long pb, int m, int first, int r_lo) {
    const long long e0 = pb + (long long)r_lo * m;
    const int off = (int)(e0 & 1);
    const int slot = (r_lo - first) * m;
    return (slot - off) & 1;
}

// producer: copy rows [r_lo, r_hi) (clipped to [0, rows_total)) of plane
// `plane` into `buf` laid out with slot 0 = plane row `first`
__device__ __forceinline__ void band_issue(double* buf, const double* slab, long long pb, int m,
                                           int first, int r_lo, int r_hi, uint64_t* bar) {
    if (r_hi <= r_lo) return;
    const Span s = span_of(pb + (long long)r_lo * m, pb + (long long)r_hi * m);
    const int sh = band_shift(pb, m, first, r_lo);
    double* dst = buf + sh + (r_lo - first) * m - s.off;
    bulk_g2s(dst, slab + s.g0, s.bytes, bar);
}

__device__ __forceinline__ uint32_t band_bytes(long long pb, int m, int r_lo, int r_hi) {
    if (r_hi <= r_lo) return 0;
    return span_of(pb + (long long)r_lo * m, pb + (long long)r_hi * m).bytes;
}

__device__ __forceinline__ BandView band_view(const double* buf, long long pb, int m, int first,
                                              int r_lo) {
    return BandView{buf + band_shift(pb, m, first, r_lo)};
}

// ============================================================================
// shared helpers for the padded work tiles
// ============================================================================
// Row sum on a zero-padded tile (pitch m+2, zero columns 0 and m+1, zero rows
// outside the plane): no boundary predicates.  rm/r0/rp point at column 0 of
// the padded rows y-1, y, y+1; x is the padded column (1..m).
template <int SH>
__device__ __forceinline__ double row_sum_pad(const double* c, const double* rm,
                                              const double* r0, const double* rp, int x) {
    double s = 0.0;
    bool first = true;
#define PINT_TERM(K, V)                      \
    if (used<SH>(K)) {                       \
        const double t_ = c[K] * (V);        \
        s = first ? t_ : s + t_;             \
        first = false;                       \
    }
    PINT_TERM(0, rm[x - 1])
    PINT_TERM(1, rm[x])
    PINT_TERM(2, rm[x + 1])
    PINT_TERM(3, r0[x - 1])
    PINT_TERM(4, r0[x])
    PINT_TERM(5, r0[x + 1])
    PINT_TERM(6, rp[x - 1])
    PINT_TERM(7, rp[x])
    PINT_TERM(8, rp[x + 1])
#undef PINT_TERM
    return s;
}

// ============================================================================
// pre-smoothing + residual + restriction, level (m -> mc)
// ============================================================================
// Warp-specialised: the last warp of the CTA is the TMA producer (full/empty
// mbarrier ring of P.stages stages), the first NT threads compute.  Each
// consumer thread owns CPT fine columns and marches down the band's rows with
// a 3x3 register window, so a stencil costs 3 shared loads per point and the
// loop structure is fully unrolled (HC compile-time).
constexpr int MAXSTAGE = 4;

struct PreParams {
    int m, mc, B, Hc, nbands, stages;
    int words_b, words_r;  // smem words: stage b, residual rows
    int aref;              // b = A_ref y formed on the fly from y = P.b (k_band_pre2<.., AR = 1>)
    int ppu;               // planes per unit (k_band_pre2 PPU; 1 or 128 / NT)
    double ar[9];          // A_ref stencil (CSR order), by value
    const double* b;
    double* bc;
    const double* tab;  // level table [n_sets][10]
    const int* sid;
};

// CSR-ordered 9-point row sum from a register window (rows a = y-1, b = y, c = y+1;
// columns 0 = x-1, 1 = x, 2 = x+1)
template <int SH>
__device__ __forceinline__ double win_sum(const double* ca, double a0, double a1, double a2,
                                          double b0, double b1, double b2, double c0, double c1,
                                          double c2) {
    double s = 0.0;
    bool first = true;
#define PINT_W(K, V)                  \
    if (used<SH>(K)) {                \
        const double t_ = ca[K] * (V); \
        s = first ? t_ : s + t_;      \
        first = false;                \
    }
    PINT_W(0, a0)
    PINT_W(1, a1)
    PINT_W(2, a2)
    PINT_W(3, b0)
    PINT_W(4, b1)
    PINT_W(5, b2)
    PINT_W(6, c0)
    PINT_W(7, c1)
    PINT_W(8, c2)
#undef PINT_W
    return s;
}

// 5-point A_ref row sum for the fused mode right-hand side b2 = A_ref y1
// (schur.py:72).  Exact arithmetic evaluates scipy's CSR row order
// S, W, C, E, N (the stored zeros SW/NE add +0) with separate multiplies and
// adds, bit-identical to the separate pass (k_band_apply); fast arithmetic
// uses fused multiply-adds (5 fp64 instructions instead of 9).
__device__ __forceinline__ double aref5(const double* ar, double s_, double w_, double c_,
                                        double e_, double n_) {
#if PINT_FAST
    double v = ar[1] * s_;
    v = __fma_rn(ar[3], w_, v);
    v = __fma_rn(ar[4], c_, v);
    v = __fma_rn(ar[5], e_, v);
    return __fma_rn(ar[7], n_, v);
#else
    double v = __dmul_rn(ar[1], s_);
    v = __dadd_rn(v, __dmul_rn(ar[3], w_));
    v = __dadd_rn(v, __dmul_rn(ar[4], c_));
    v = __dadd_rn(v, __dmul_rn(ar[5], e_));
    return __dadd_rn(v, __dmul_rn(ar[7], n_));
#endif
}

template <int SH, int NT, int CPT, int HC>
__global__ void __launch_bounds__(NT + 32) k_band_pre(PreParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[MAXSTAGE], empty[MAXSTAGE];
    __shared__ double meta[MAXSTAGE][PINT_TW];  // per-stage stencil + dinv, written by the producer
    constexpr int RR = 2 * HC + 1;  // residual rows per unit
    const int m = P.m, mc = P.mc, S = P.stages;
    const long long n = (long long)m * m, nc = (long long)mc * mc;
    double* sr = smem + S * P.words_b;  // RR x m
    const int units = P.B * P.nbands;
    const int tid = threadIdx.x;
    // element offsets are taken from a 16-byte aligned virtual base so that the
    // bulk-copy alignment does not depend on where the caller's slab starts
    const int bob = (int)((reinterpret_cast<uintptr_t>(P.b) >> 3) & 1);
    const double* gb = P.b - bob;
    auto unit_rows = [&](int u, int& plane, int& Y0, int& Y1) {
        plane = u / P.nbands;
        const int j = u - plane * P.nbands;
        Y0 = j * HC;
        Y1 = min(mc, Y0 + HC);
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid >= NT) {  // ---- producer warp ----
        if (tid == NT) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                int plane, Y0, Y1;
                unit_rows(u, plane, Y0, Y1);
                const long long pb = plane * n + bob;
                const int first = 2 * Y0 - 1;
                const int lo = max(0, first), hi = min(m, 2 * Y1 + 2);
                const double* tb = P.tab + (size_t)__ldg(P.sid + plane) * PINT_TW;
#pragma unroll
                for (int q = 0; q < PINT_TW; ++q) meta[s][q] = __ldg(tb + q);
                mbar_expect_tx(&full[s], band_bytes(pb, m, lo, hi));  // release: meta visible
                band_issue(smem + s * P.words_b, gb, pb, m, first, lo, hi, &full[s]);
            }
        }
        return;
    }
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % S;
        int plane, Y0, Y1;
        unit_rows(u, plane, Y0, Y1);
        const long long pb = plane * n + bob;
        const int first = 2 * Y0 - 1;
        const int lo = max(0, first);
        const int nr = 2 * (Y1 - Y0) + 1;
        mbar_wait(&full[s], (k / S) & 1);
        double ca[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) ca[q] = meta[s][q];
        const double d = meta[s][9];
        const BandView vb = band_view(smem + s * P.words_b, pb, m, first, lo);
        // residual r = b - A(dinv*b) on fine rows 2*Y0 .. 2*Y1 (slots 1 .. nr)
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int x = tid + j * NT;
            if (x >= m) continue;
            const bool w = x > 0, e = x < m - 1;
            double a0, a1, a2, b0, b1, b2, bb, braw_b;
            auto ld = [&](int slot, double& l, double& c, double& r, double& raw) {
                const int gy = first + slot;
                const bool in = gy >= 0 && gy < m;
                const double* row = vb.row(slot, m);
                raw = in ? row[x] : 0.0;
                l = (in && w) ? d * row[x - 1] : 0.0;
                c = d * raw;
                r = (in && e) ? d * row[x + 1] : 0.0;
            };
            ld(0, a0, a1, a2, bb);
            ld(1, b0, b1, b2, braw_b);
#pragma unroll
            for (int rho = 0; rho < RR; ++rho) {
                if (rho < nr) {
                    double c0, c1, c2, braw_c;
                    ld(rho + 2, c0, c1, c2, braw_c);
                    sr[rho * m + x] =
                        braw_b - win_sum<SH>(ca, a0, a1, a2, b0, b1, b2, c0, c1, c2);
                    a0 = b0; a1 = b1; a2 = b2;
                    b0 = c0; b1 = c1; b2 = c2;
                    braw_b = braw_c;
                }
            }
        }
        consumer_sync<NT>();
        if (tid == 0) mbar_arrive(&empty[s]);  // stage s fully consumed
        // restriction: P^T r, ascending fine index (csc_matvec order)
        const int ncr = Y1 - Y0;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int X = tid + j * NT;
            if (X >= mc) continue;
            const int f = 2 * X;
            double p0 = sr[f], p1 = sr[f + 1], p2 = sr[f + 2];
            double* out = P.bc + plane * nc + (long long)Y0 * mc + X;
#pragma unroll
            for (int r = 0; r < HC; ++r) {
                if (r < ncr) {
                    const double* r1 = sr + (2 * r + 1) * m + f;
                    const double* r2 = r1 + m;
                    const double q0 = r1[0], q1 = r1[1], q2 = r1[2];
                    const double t0 = r2[0], t1 = r2[1], t2 = r2[2];
                    double v = 0.25 * p0;
                    v = v + 0.5 * p1;
                    v = v + 0.25 * p2;
                    v = v + 0.5 * q0;
                    v = v + 1.0 * q1;
                    v = v + 0.5 * q2;
                    v = v + 0.25 * t0;
                    v = v + 0.5 * t1;
                    v = v + 0.25 * t2;
                    out[(long long)r * mc] = v;
                    p0 = t0; p1 = t1; p2 = t2;
                }
            }
        }
        consumer_sync<NT>();
    }
}

// Paired-column form of k_band_pre (default): consumer thread t computes the
// residual of fine columns 2t-1 and 2t from a 4-column register window of
// x0 = dinv*b (one multiply per loaded value instead of three), stores the
// pair as one 16-byte word of the padded residual tile, and then restricts
// coarse column t from padded columns 2t+1 .. 2t+3.
//
// AR = 1 (schur.py:72-73 fused): the right-hand side is b = A_ref y (y = the
// first mode V-cycle's output) and is never stored.  The stage holds y on one
// more halo row per side and every b value of the window is the 5-point
// A_ref row sum (aref5, zero fill as k_band_apply) of a rolling 3-row window
// of y; k_band_post2<AR = 1> forms the identical values.
//
// PPU > 1 (narrow levels, NT <= 64 column pairs): one unit is the same band
// of PPU consecutive planes, consumer warp group pl of the CTA owning plane
// g*PPU + pl, so a stage carries PPU bands and the per-unit barrier and
// mbarrier latency is paid once for PPU planes.
template <int SH, int NT, int HC, int AR = 0, int PPU = 1>
__global__ void __launch_bounds__(NT * PPU + 32, (AR && NT * PPU <= 128) ? 3 : 1) k_band_pre2(PreParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[MAXSTAGE], empty[MAXSTAGE];
    __shared__ double meta[MAXSTAGE][PPU][PINT_TW];
    constexpr int RR = 2 * HC + 1;  // residual rows per unit
    constexpr int NC = NT * PPU;    // consumer threads
    const int m = P.m, mc = P.mc, S = P.stages;
    const int mp = m + 3;           // padded residual pitch (even): fine x at index x+1
    const long long n = (long long)m * m, nc = (long long)mc * mc;
    const int tid = threadIdx.x;
    const int pl = tid < NC ? tid / NT : 0;  // plane of the unit this consumer works on
    double* sr = smem + S * PPU * P.words_b + pl * P.words_r;  // RR x mp
    const int groups = (P.B + PPU - 1) / PPU;
    const int units = groups * P.nbands;
    const int bob = (int)((reinterpret_cast<uintptr_t>(P.b) >> 3) & 1);
    const double* gb = P.b - bob;
    auto stage_b = [&](int s, int q) { return smem + (s * PPU + q) * P.words_b; };
    auto unit_rows = [&](int u, int& g, int& Y0, int& Y1) {
        g = u / P.nbands;
        const int j = u - g * P.nbands;
        Y0 = j * HC;
        Y1 = min(mc, Y0 + HC);
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid >= NC) {  // ---- producer warp (as k_band_pre) ----
        if (tid == NC) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                int g, Y0, Y1;
                unit_rows(u, g, Y0, Y1);
                const int first = 2 * Y0 - 1 - AR;  // AR: y on one more halo row per side
                const int lo = max(0, first), hi = min(m, 2 * Y1 + 2 + AR);
                uint32_t bytes = 0;
                for (int q = 0; q < PPU; ++q) {
                    const int plane = g * PPU + q;
                    if (plane >= P.B) break;
                    const double* tb = P.tab + (size_t)__ldg(P.sid + plane) * PINT_TW;
#pragma unroll
                    for (int w = 0; w < PINT_TW; ++w) meta[s][q][w] = __ldg(tb + w);
                    bytes += band_bytes(plane * n + bob, m, lo, hi);
                }
                mbar_expect_tx(&full[s], bytes);
                for (int q = 0; q < PPU; ++q) {
                    const int plane = g * PPU + q;
                    if (plane >= P.B) break;
                    band_issue(stage_b(s, q), gb, plane * n + bob, m, first, lo, hi, &full[s]);
                }
            }
        }
        return;
    }
    const int t = tid - pl * NT;
    const bool tcol = t <= mc;
    const bool has_a = t >= 1;          // fine column 2t-1 exists
    const bool has_l = t >= 1;          // fine column 2t-2 exists
    const bool has_r = t < mc;          // fine column 2t+1 exists
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % S;
        int g, Y0, Y1;
        unit_rows(u, g, Y0, Y1);
        const int plane = g * PPU + pl;
        const bool pok = PPU == 1 || plane < P.B;
        const bool active = tcol && pok;
        const long long pb = plane * n + bob;
        const int first = 2 * Y0 - 1;
        const int lo = max(0, first);
        const int nr = 2 * (Y1 - Y0) + 1;
        // interior band: HC coarse rows whose fine rows (and the A_ref halo) are
        // all inside the plane, so the row loops carry no boundary predicates
        const bool interior = Y1 - Y0 == HC && Y0 >= 1 && 2 * Y1 + 2 < m;
        auto unit_body = [&](auto in_tag) {
        constexpr bool IN = decltype(in_tag)::value;
        mbar_wait(&full[s], (k / S) & 1);
        double ca[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) ca[q] = meta[s][pl][q];
        const double d = meta[s][pl][9];
        const BandView vb = AR ? band_view(stage_b(s, pl), pb, m, first - 1, max(0, first - 1))
                               : band_view(stage_b(s, pl), pb, m, first, lo);
        if (active) {
            // window columns: 0 = 2t-2, 1 = 2t-1 (xa), 2 = 2t (xb), 3 = 2t+1
            const double* bcol = vb.p + 2 * t;
            // AR: y rows (slot 0 = plane row first-1) at columns 2t-3 .. 2t+2, zero outside
            double ya[6], yb[6], yc[6];
            auto yrow = [&](int ys, double* v) {
                const int gy = first - 1 + ys;
                const bool in = IN || (gy >= 0 && gy < m);
                const double* row = bcol + ys * m;
                v[0] = (in && t >= 2) ? row[-3] : 0.0;
                v[1] = (in && has_l) ? row[-2] : 0.0;
                v[2] = (in && has_a) ? row[-1] : 0.0;
                v[3] = in ? row[0] : 0.0;
                v[4] = (in && has_r) ? row[1] : 0.0;
                v[5] = (in && has_r) ? row[2] : 0.0;
            };
            if (AR) {
                yrow(0, ya);
                yrow(1, yb);
            }
            auto ld = [&](int slot, double& w0, double& w1, double& w2, double& w3, double& ra,
                          double& rb) {
                const int gy = first + slot;
                const bool in = IN || (gy >= 0 && gy < m);
                if (AR) {
                    // b row `slot` from y slots slot .. slot+2 (5-point A_ref, k_band_apply order)
                    yrow(slot + 2, yc);
                    double bq[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        bq[i] = aref5(P.ar, ya[i + 1], yb[i], yb[i + 1], yb[i + 2], yc[i + 1]);
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        ya[i] = yb[i];
                        yb[i] = yc[i];
                    }
                    ra = (in && has_a) ? bq[1] : 0.0;
                    rb = in ? bq[2] : 0.0;
                    w0 = (in && has_l) ? d * bq[0] : 0.0;
                    w1 = d * ra;
                    w2 = d * rb;
                    w3 = (in && has_r) ? d * bq[3] : 0.0;
                    return;
                }
                const double* row = bcol + slot * m;
                ra = (in && has_a) ? row[-1] : 0.0;
                rb = in ? row[0] : 0.0;
                w0 = (in && has_l) ? d * row[-2] : 0.0;
                w1 = d * ra;
                w2 = d * rb;
                w3 = (in && has_r) ? d * row[1] : 0.0;
            };
            double a0, a1, a2, a3, b0, b1, b2, b3, bra, brb, dummy0, dummy1;
            ld(0, a0, a1, a2, a3, dummy0, dummy1);
            ld(1, b0, b1, b2, b3, bra, brb);
            double* out = sr + 2 * t;  // padded columns 2t, 2t+1 = fine 2t-1, 2t
#pragma unroll
            for (int rho = 0; rho < RR; ++rho) {
                if (IN || rho < nr) {
                    double c0, c1, c2, c3, cra, crb;
                    ld(rho + 2, c0, c1, c2, c3, cra, crb);
                    const double ra = has_a ? bra - win_sum<SH>(ca, a0, a1, a2, b0, b1, b2, c0, c1, c2)
                                            : 0.0;
                    const double rb = brb - win_sum<SH>(ca, a1, a2, a3, b1, b2, b3, c1, c2, c3);
                    *reinterpret_cast<double2*>(out + rho * mp) = make_double2(ra, rb);
                    a0 = b0; a1 = b1; a2 = b2; a3 = b3;
                    b0 = c0; b1 = c1; b2 = c2; b3 = c3;
                    bra = cra;
                    brb = crb;
                }
            }
        }
        consumer_sync<NC>();
        if (tid == 0) mbar_arrive(&empty[s]);  // stage s fully consumed
        // restriction: P^T r, ascending fine index (csc_matvec order);
        // coarse X = t reads fine columns 2X .. 2X+2 = padded 2X+1 .. 2X+3
        const int ncr = Y1 - Y0;
        if (t < mc && pok) {
            const double* col = sr + 2 * t;
            auto ld3 = [&](int row, double& v0, double& v1, double& v2) {
                const double* q = col + row * mp;
                v0 = q[1];
                const double2 pr = *reinterpret_cast<const double2*>(q + 2);
                v1 = pr.x;
                v2 = pr.y;
            };
            double p0, p1, p2;
            ld3(0, p0, p1, p2);
            double* outc = P.bc + plane * nc + (long long)Y0 * mc + t;
#pragma unroll
            for (int r = 0; r < HC; ++r) {
                if (IN || r < ncr) {
                    double q0, q1, q2, t0, t1, t2;
                    ld3(2 * r + 1, q0, q1, q2);
                    ld3(2 * r + 2, t0, t1, t2);
                    double v = 0.25 * p0;
                    v = v + 0.5 * p1;
                    v = v + 0.25 * p2;
                    v = v + 0.5 * q0;
                    v = v + 1.0 * q1;
                    v = v + 0.5 * q2;
                    v = v + 0.25 * t0;
                    v = v + 0.5 * t1;
                    v = v + 0.25 * t2;
                    outc[(long long)r * mc] = v;
                    p0 = t0; p1 = t1; p2 = t2;
                }
            }
        }
        consumer_sync<NC>();
        };
        if (interior) unit_body(std::true_type{});
        else unit_body(std::false_type{});
    }
}

// ============================================================================
// prolongation + post-smoothing (+ finest-level epilogue), level (mc -> m)
// ============================================================================
struct PostBandParams {
    int m, mc, B, H, nbands, stages;
    int words_b, words_e, words_q, words_x;  // stage: b, e, pin|aux ; work: padded x
    int aref;                                // b = A_ref y formed on the fly from y = P.b
    int ppu;                                 // planes per unit (k_band_post2 PPU)
    double ar[9];
    const double* b;
    const double* ec;
    const double* tab;
    const int* sid;
    double* out;
    int epi;
    double scale;
    const double* steps;
    const double* rsteps;
    const double* pin;
    const double* aux;
    double* part;
};

template <int SH, int EPI, int NT, int CPT, int H>
__global__ void __launch_bounds__(NT + 32) k_band_post(PostBandParams P) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[MAXSTAGE], empty[MAXSTAGE];
    __shared__ double meta[MAXSTAGE][PINT_TW + 2];  // stencil, dinv, tau, 1/tau|0 (producer-written)
    __shared__ double red[NT / 32];
    const int m = P.m, mc = P.mc, mp = m + 2, S = P.stages;
    const long long n = (long long)m * m, nc = (long long)mc * mc;
    const int wstage = P.words_b + P.words_e + P.words_q;
    double* sx = smem + S * wstage;  // (H+2) x (m+2) zero-padded
    const int units = P.B * P.nbands;
    const int tid = threadIdx.x;
    const double* qsrc0 = EPI == EPI_UZAWA_P ? P.pin : P.aux;
    const int bob = (int)((reinterpret_cast<uintptr_t>(P.b) >> 3) & 1);
    const int boe = (int)((reinterpret_cast<uintptr_t>(P.ec) >> 3) & 1);
    const int boq = (int)((reinterpret_cast<uintptr_t>(qsrc0) >> 3) & 1);
    constexpr bool HAS_Q = EPI == EPI_UZAWA_P || EPI == EPI_SCALE_DOT || EPI == EPI_SCALE_DOTONLY;
    constexpr bool HAS_DOT =
        EPI == EPI_UZAWA_P || EPI == EPI_DOT_TAU || EPI == EPI_SCALE_DOT || EPI == EPI_SCALE_DOTONLY;
    constexpr bool HAS_TAU = EPI == EPI_DIV_TAU || EPI == EPI_UZAWA_P || EPI == EPI_DOT_TAU;
    auto sb = [&](int s) { return smem + s * wstage; };
    auto se = [&](int s) { return smem + s * wstage + P.words_b; };
    auto sq = [&](int s) { return smem + s * wstage + P.words_b + P.words_e; };
    auto unit_rows = [&](int u, int& plane, int& y0, int& y1) {
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
    for (int i = tid; i < P.words_x; i += NT + 32) sx[i] = 0.0;
    __syncthreads();
    if (tid >= NT) {  // ---- producer warp ----
        if (tid == NT) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                int plane, y0, y1;
                unit_rows(u, plane, y0, y1);
                const long long pb = plane * n + bob, pc = plane * nc + boe, pq = plane * n + boq;
                const int fb = y0 - 1, lob = max(0, fb), hib = min(m, y1 + 1);
                const int fe = y0 / 2 - 1, loe = max(0, fe), hie = min(mc, y1 / 2 + 1);
                uint32_t bytes = band_bytes(pb, m, lob, hib) + band_bytes(pc, mc, loe, hie);
                if (HAS_Q) bytes += band_bytes(pq, m, y0, y1);
                const double* tb = P.tab + (size_t)__ldg(P.sid + plane) * PINT_TW;
#pragma unroll
                for (int q = 0; q < PINT_TW; ++q) meta[s][q] = __ldg(tb + q);
                meta[s][PINT_TW] = HAS_TAU ? __ldg(P.steps + plane) : 1.0;
                meta[s][PINT_TW + 1] = HAS_TAU ? __ldg(P.rsteps + plane) : 0.0;
                mbar_expect_tx(&full[s], bytes);
                band_issue(sb(s), P.b - bob, pb, m, fb, lob, hib, &full[s]);
                band_issue(se(s), P.ec - boe, pc, mc, fe, loe, hie, &full[s]);
                if (HAS_Q) band_issue(sq(s), qsrc0 - boq, pq, m, y0, y0, y1, &full[s]);
            }
        }
        return;
    }
    double acc = 0.0;
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % S;
        int plane, y0, y1;
        unit_rows(u, plane, y0, y1);
        const long long pb = plane * n + bob, pc = plane * nc + boe, pq = plane * n + boq;
        const long long po = plane * n;  // output plane (plain stores, no alignment needs)
        const int fb = y0 - 1, lob = max(0, fb);
        const int fe = y0 / 2 - 1, loe = max(0, fe);
        const int nrow = y1 - y0;
        mbar_wait(&full[s], (k / S) & 1);
        double ca[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) ca[q] = meta[s][q];
        const double d = meta[s][9];
        const BandView vb = band_view(sb(s), pb, m, fb, lob);
        const BandView ve = band_view(se(s), pc, mc, fe, loe);
        // x = dinv*b + P e on rows y0-1 .. y1 (tile rows 0 .. nrow+1)
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int x = tid + j * NT;
            if (x >= m) continue;
            const bool xodd = x & 1;
            const int c0 = xodd ? (x - 1) >> 1 : (x >> 1) - 1;  // odd: the one coarse column
            const int c1 = x >> 1;
            const bool h0 = xodd || x >= 2, h1 = !xodd && c1 < mc;
#pragma unroll
            for (int r = 0; r < H + 2; ++r) {
                if (r > nrow + 1) continue;
                const int gy = fb + r;
                double xv = 0.0;
                if (gy >= 0 && gy < m) {
                    const double bv = vb.row(r, m)[x];
                    double pe;
                    if (gy & 1) {
                        const double* ea = ve.row(((gy - 1) >> 1) - fe, mc);
                        if (xodd) {
                            pe = (1.0 * 1.0) * ea[c0];
                        } else {
                            if (h0 && h1) pe = (1.0 * 0.5) * ea[c0] + (1.0 * 0.5) * ea[c1];
                            else pe = h0 ? (1.0 * 0.5) * ea[c0] : (1.0 * 0.5) * ea[c1];
                        }
                    } else {
                        const int ja = (gy >> 1) - 1, jb = gy >> 1;
                        const bool va = ja >= 0, vbb = jb < mc;
                        const double* ea = ve.row(va ? ja - fe : 0, mc);
                        const double* eb = ve.row(vbb ? jb - fe : 0, mc);
                        if (xodd) {
                            const double a = va ? ea[c0] : 0.0, bq = vbb ? eb[c0] : 0.0;
                            pe = (0.5 * 1.0) * a;
                            pe = pe + (0.5 * 1.0) * bq;
                        } else {
                            const double a0 = (va && h0) ? ea[c0] : 0.0;
                            const double a1 = (va && h1) ? ea[c1] : 0.0;
                            const double b0 = (vbb && h0) ? eb[c0] : 0.0;
                            const double b1 = (vbb && h1) ? eb[c1] : 0.0;
                            pe = (0.5 * 0.5) * a0;
                            pe = pe + (0.5 * 0.5) * a1;
                            pe = pe + (0.5 * 0.5) * b0;
                            pe = pe + (0.5 * 0.5) * b1;
                        }
                    }
                    xv = d * bv + pe;
                }
                sx[r * mp + x + 1] = xv;
            }
        }
        consumer_sync<NT>();
        // x += dinv * (b - A x) on rows y0 .. y1-1, epilogue
        const BandView vq = band_view(sq(s), pq, m, y0, y0);
        const double tau = meta[s][PINT_TW];
        const double rtau = meta[s][PINT_TW + 1];  // > 0: tau is a power of two
        auto divtau = [&](double v) { return rtau > 0.0 ? v * rtau : band_div(v, tau); };
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int x = tid + j * NT;
            if (x >= m) continue;
            const double* col = sx + x;  // padded columns x, x+1, x+2 = fine x-1, x, x+1
            double a0 = col[0], a1 = col[1], a2 = col[2];
            double b0 = col[mp], b1 = col[mp + 1], b2 = col[mp + 2];
            double* orow = P.out + po + (long long)y0 * m + x;
#pragma unroll
            for (int r = 0; r < H; ++r) {
                if (r < nrow) {
                    const double* cr = col + (r + 2) * mp;
                    const double c0 = cr[0], c1 = cr[1], c2 = cr[2];
                    const double bv = vb.row(r + 1, m)[x];
                    const double xn =
                        b1 + d * (bv - win_sum<SH>(ca, a0, a1, a2, b0, b1, b2, c0, c1, c2));
                    double* o = orow + (long long)r * m;
                    if (EPI == EPI_PLAIN) {
                        *o = xn;
                    } else if (EPI == EPI_DIV_TAU) {
                        *o = divtau(xn);
                    } else if (EPI == EPI_UZAWA_P) {
                        const double dp = divtau(xn);
                        *o = vq.row(r, m)[x] + dp;
                        acc += bv * dp;
                    } else if (EPI == EPI_DOT_TAU) {
                        acc += bv * divtau(xn);
                    } else if (EPI == EPI_SCALE) {
                        *o = P.scale * xn;
                    } else if (EPI == EPI_SCALE_DOT) {
                        const double wv = P.scale * xn;
                        *o = wv;
                        acc += vq.row(r, m)[x] * wv;
                    } else if (EPI == EPI_SCALE_DOTONLY) {
                        acc += vq.row(r, m)[x] * (P.scale * xn);
                    }
                    a0 = b0; a1 = b1; a2 = b2;
                    b0 = c0; b1 = c1; b2 = c2;
                }
            }
        }
        consumer_sync<NT>();
        if (tid == 0) mbar_arrive(&empty[s]);
    }
    if (HAS_DOT) {
        const double sum = consumer_sum<NT>(acc, red);
        if (tid == 0) P.part[blockIdx.x] = sum;
    }
}

// ----------------------------------------------------------------------------
// Paired-column form of k_band_post (default): consumer thread t owns the fine
// columns xa = 2t-1 (odd) and xb = 2t (even), t = 0..mc, which share their
// coarse columns t-1 and t.  The band's row parity is known at compile time
// (bands start at even rows), so the prolongation is branch-free: absent
// coarse neighbours enter as exact zeros (0 + v == v, v + (+-0) == v), which
// leaves every sum bit-identical to the ascending-coarse-index csr_matvec of P.
// The smoothing window is 3 rows x 4 padded columns in registers, reading one
// 16-byte pair plus two scalars of the padded x tile per row.
// AR = 1: b = A_ref y formed on the fly (see k_band_pre2); the stage holds y
// on rows y0-2 .. y1+1 and the b values of rows y0-1 .. y1 are kept in
// registers between the prolongation and the smoothing sweep.
// PPU > 1: PPU planes per unit, as in k_band_pre2.
template <int SH, int EPI, int NT, int H, int AR = 0, int PPU = 1>
__global__ void __launch_bounds__(NT * PPU + 32) k_band_post2(PostBandParams P) {
    constexpr int NC = NT * PPU;  // consumer threads
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t full[MAXSTAGE], empty[MAXSTAGE];
    __shared__ double meta[MAXSTAGE][PPU][PINT_TW + 2];
    __shared__ double red[NC / 32 > 0 ? NC / 32 : 1];
    static_assert(H % 2 == 0, "bands start at even rows");
    const int m = P.m, mc = P.mc, S = P.stages;
    const int mp = m + 3;  // even pitch: padded column c sits at index c, pairs are 16-byte aligned
    const long long n = (long long)m * m, nc = (long long)mc * mc;
    const int wstage = P.words_b + P.words_e + P.words_q;
    const int tid = threadIdx.x;
    const int pl = tid < NC ? tid / NT : 0;  // plane of the unit this consumer works on
    double* sx = smem + S * PPU * wstage + pl * P.words_x;  // (H+2) x mp, zero-padded columns 0 and m+1
    const int units = (P.B + PPU - 1) / PPU * P.nbands;
    const double* qsrc0 = EPI == EPI_UZAWA_P ? P.pin : P.aux;
    const int bob = (int)((reinterpret_cast<uintptr_t>(P.b) >> 3) & 1);
    const int boe = (int)((reinterpret_cast<uintptr_t>(P.ec) >> 3) & 1);
    const int boq = (int)((reinterpret_cast<uintptr_t>(qsrc0) >> 3) & 1);
    constexpr bool HAS_Q = EPI == EPI_UZAWA_P || EPI == EPI_SCALE_DOT || EPI == EPI_SCALE_DOTONLY;
    constexpr bool HAS_DOT =
        EPI == EPI_UZAWA_P || EPI == EPI_DOT_TAU || EPI == EPI_SCALE_DOT || EPI == EPI_SCALE_DOTONLY;
    constexpr bool HAS_TAU = EPI == EPI_DIV_TAU || EPI == EPI_UZAWA_P || EPI == EPI_DOT_TAU;
    auto sb = [&](int s, int q) { return smem + (s * PPU + q) * wstage; };
    auto se = [&](int s, int q) { return smem + (s * PPU + q) * wstage + P.words_b; };
    auto sq = [&](int s, int q) { return smem + (s * PPU + q) * wstage + P.words_b + P.words_e; };
    auto unit_rows = [&](int u, int& g, int& y0, int& y1) {
        g = u / P.nbands;
        const int j = u - g * P.nbands;
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
    {
        double* sx0 = smem + S * PPU * wstage;
        for (int i = tid; i < PPU * P.words_x; i += NC + 32) sx0[i] = 0.0;
    }
    __syncthreads();
    if (tid >= NC) {  // ---- producer warp (as k_band_post) ----
        if (tid == NC) {
            int k = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait_sleep(&empty[s], ((k / S) - 1) & 1);
                int g, y0, y1;
                unit_rows(u, g, y0, y1);
                const int fb = y0 - 1 - AR, lob = max(0, fb), hib = min(m, y1 + 1 + AR);
                const int fe = y0 / 2 - 1, loe = max(0, fe), hie = min(mc, y1 / 2 + 1);
                uint32_t bytes = 0;
                for (int q = 0; q < PPU; ++q) {
                    const int plane = g * PPU + q;
                    if (plane >= P.B) break;
                    const long long pb = plane * n + bob, pc = plane * nc + boe, pq = plane * n + boq;
                    bytes += band_bytes(pb, m, lob, hib) + band_bytes(pc, mc, loe, hie);
                    if (HAS_Q) bytes += band_bytes(pq, m, y0, y1);
                    const double* tb = P.tab + (size_t)__ldg(P.sid + plane) * PINT_TW;
#pragma unroll
                    for (int w = 0; w < PINT_TW; ++w) meta[s][q][w] = __ldg(tb + w);
                    meta[s][q][PINT_TW] = HAS_TAU ? __ldg(P.steps + plane) : 1.0;
                    meta[s][q][PINT_TW + 1] = HAS_TAU ? __ldg(P.rsteps + plane) : 0.0;
                }
                mbar_expect_tx(&full[s], bytes);
                for (int q = 0; q < PPU; ++q) {
                    const int plane = g * PPU + q;
                    if (plane >= P.B) break;
                    const long long pb = plane * n + bob, pc = plane * nc + boe, pq = plane * n + boq;
                    band_issue(sb(s, q), P.b - bob, pb, m, fb, lob, hib, &full[s]);
                    band_issue(se(s, q), P.ec - boe, pc, mc, fe, loe, hie, &full[s]);
                    if (HAS_Q) band_issue(sq(s, q), qsrc0 - boq, pq, m, y0, y0, y1, &full[s]);
                }
            }
        }
        return;
    }
    const int t = tid - pl * NT;
    double bsa[AR ? H + 2 : 1], bsb[AR ? H + 2 : 1];  // AR: b at xa, xb of tile rows 0 .. H+1
    const bool tcol = t <= mc;
    const bool has_cb = t < mc;            // coarse column t exists
    const int xa = 2 * t - 1, xb = 2 * t;
    double acc = 0.0;
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % S;
        int g, y0, y1;
        unit_rows(u, g, y0, y1);
        const int plane = g * PPU + pl;
        const bool active = tcol && (PPU == 1 || plane < P.B);
        const bool has_a = t >= 1 && active;   // column xa = 2t-1 exists (and coarse column t-1)
        const long long pb = plane * n + bob, pc = plane * nc + boe, pq = plane * n + boq;
        const int fb = y0 - 1, lob = max(0, fb);
        const int fe = y0 / 2 - 1, loe = max(0, fe);
        const int nrow = y1 - y0;
        // interior band: H rows whose prolongation and halo rows are all inside
        // the plane, so the row loops carry no boundary predicates
        const bool interior = nrow == H && y0 >= 2 && y1 <= m - 2;
        auto unit_body = [&](auto in_tag) {
        constexpr bool IN = decltype(in_tag)::value;
        mbar_wait(&full[s], (k / S) & 1);
        double ca[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) ca[q] = meta[s][pl][q];
        const double d = meta[s][pl][9];
        const BandView vb = AR ? band_view(sb(s, pl), pb, m, fb - 1, max(0, fb - 1))
                               : band_view(sb(s, pl), pb, m, fb, lob);
        const BandView ve = band_view(se(s, pl), pc, mc, fe, loe);
        if (active) {
            // x = dinv*b + P e on tile rows 0 .. nrow+1 (fine rows y0-1 .. y1)
            const double* brow = vb.p + xb;       // slot r at brow + r*m (AR: y slot r+1)
            const double* erow = ve.p + (t - 1);  // coarse column t-1 of slot 0
            // AR: y rows at columns 2t-2 .. 2t+1 (y slot 0 = fine row y0-2), zero outside
            double ya[4], yb[4], yc[4];
            auto yrow = [&](int ys, double* v) {
                const int gy = fb - 1 + ys;
                const bool in = IN || (gy >= 0 && gy < m);
                const double* row = brow + ys * m;
                v[0] = (in && has_a) ? row[-2] : 0.0;
                v[1] = (in && has_a) ? row[-1] : 0.0;
                v[2] = in ? row[0] : 0.0;
                v[3] = (in && has_cb) ? row[1] : 0.0;
            };
            if (AR) {
                yrow(0, ya);
                yrow(1, yb);
            }
#pragma unroll
            for (int r = 0; r < H + 2; ++r) {
                if (!IN && r > nrow + 1) continue;
                const int gy = fb + r;
                double xva = 0.0, xvb = 0.0;
                double b2a = 0.0, b2b = 0.0;
                if (AR) {
                    yrow(r + 2, yc);
                    b2a = aref5(P.ar, ya[1], yb[0], yb[1], yb[2], yc[1]);
                    b2b = aref5(P.ar, ya[2], yb[1], yb[2], yb[3], yc[2]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        ya[i] = yb[i];
                        yb[i] = yc[i];
                    }
                    bsa[AR ? r : 0] = b2a;
                    bsb[AR ? r : 0] = b2b;
                }
                if (IN || (gy >= 0 && gy < m)) {
                    const double* bp = brow + r * m;
                    const double bva = has_a ? (AR ? b2a : bp[-1]) : 0.0;
                    const double bvb = AR ? b2b : bp[0];
                    double pa, pbv;
                    if ((r & 1) == 0) {
                        // odd fine row: one coarse row, slot r/2
                        const double* e = erow + (r >> 1) * mc;
                        const double e0 = has_a ? e[0] : 0.0;
                        const double e1 = has_cb ? e[1] : 0.0;
                        pa = (1.0 * 1.0) * e0;
                        pbv = (1.0 * 0.5) * e0;
                        pbv = pbv + (1.0 * 0.5) * e1;
                    } else {
                        // even fine row gy: coarse rows gy/2-1 (slot (r-1)/2) and gy/2 (slot (r+1)/2)
                        const bool va = IN || gy >= 2, vbr = IN || (gy >> 1) < mc;
                        const double* e = erow + ((r - 1) >> 1) * mc;
                        const double a0 = (va && has_a) ? e[0] : 0.0;
                        const double a1 = (va && has_cb) ? e[1] : 0.0;
                        const double b0 = (vbr && has_a) ? e[mc] : 0.0;
                        const double b1 = (vbr && has_cb) ? e[mc + 1] : 0.0;
                        pa = (0.5 * 1.0) * a0;
                        pa = pa + (0.5 * 1.0) * b0;
                        pbv = (0.5 * 0.5) * a0;
                        pbv = pbv + (0.5 * 0.5) * a1;
                        pbv = pbv + (0.5 * 0.5) * b0;
                        pbv = pbv + (0.5 * 0.5) * b1;
                    }
                    xva = has_a ? d * bva + pa : 0.0;
                    xvb = d * bvb + pbv;
                }
                *reinterpret_cast<double2*>(sx + r * mp + 2 * t) = make_double2(xva, xvb);
            }
        }
        consumer_sync<NC>();
        const BandView vq = band_view(sq(s, pl), pq, m, y0, y0);
        const double tau = meta[s][pl][PINT_TW];
        const double rtau = meta[s][pl][PINT_TW + 1];
        auto divtau = [&](double v) { return rtau > 0.0 ? v * rtau : band_div(v, tau); };
        if (active) {
            // x += dinv * (b - A x) on rows y0 .. y1-1; padded columns 2t-1 .. 2t+2
            const double* col = sx + 2 * t;
            auto ldrow = [&](int r, double& c0, double& c1, double& c2, double& c3) {
                const double* q = col + r * mp;
                c0 = t >= 1 ? q[-1] : 0.0;
                const double2 mid = *reinterpret_cast<const double2*>(q);
                c1 = mid.x;
                c2 = mid.y;
                c3 = q[2];
            };
            double a0, a1, a2, a3, b0, b1, b2, b3;
            ldrow(0, a0, a1, a2, a3);
            ldrow(1, b0, b1, b2, b3);
            double* orow = P.out + plane * n + (long long)y0 * m + xb;
            const double* brow = vb.p + m + xb;  // slot r+1
            const double* qrow = vq.p + xb;
#pragma unroll
            for (int r = 0; r < H; ++r) {
                if (IN || r < nrow) {
                    double c0, c1, c2, c3;
                    ldrow(r + 2, c0, c1, c2, c3);
                    const double bvb = AR ? bsb[AR ? r + 1 : 0] : brow[r * m];
                    const double bva = has_a ? (AR ? bsa[AR ? r + 1 : 0] : brow[r * m - 1]) : 0.0;
                    const double xna =
                        b1 + d * (bva - win_sum<SH>(ca, a0, a1, a2, b0, b1, b2, c0, c1, c2));
                    const double xnb =
                        b2 + d * (bvb - win_sum<SH>(ca, a1, a2, a3, b1, b2, b3, c1, c2, c3));
                    double* o = orow + (long long)r * m;
                    auto emit = [&](double xn, double bv, int off, bool ok) {
                        if (!ok) return;
                        if (EPI == EPI_PLAIN) {
                            o[off] = xn;
                        } else if (EPI == EPI_DIV_TAU) {
                            o[off] = divtau(xn);
                        } else if (EPI == EPI_UZAWA_P) {
                            const double dp = divtau(xn);
                            o[off] = qrow[r * m + off] + dp;
                            acc += bv * dp;
                        } else if (EPI == EPI_DOT_TAU) {
                            acc += bv * divtau(xn);
                        } else if (EPI == EPI_SCALE) {
                            o[off] = P.scale * xn;
                        } else if (EPI == EPI_SCALE_DOT) {
                            const double wv = P.scale * xn;
                            o[off] = wv;
                            acc += qrow[r * m + off] * wv;
                        } else if (EPI == EPI_SCALE_DOTONLY) {
                            acc += qrow[r * m + off] * (P.scale * xn);
                        }
                    };
                    emit(xna, bva, -1, has_a);
                    emit(xnb, bvb, 0, true);
                    a0 = b0; a1 = b1; a2 = b2; a3 = b3;
                    b0 = c0; b1 = c1; b2 = c2; b3 = c3;
                }
            }
        }
        consumer_sync<NC>();
        if (tid == 0) mbar_arrive(&empty[s]);
        };
        if (interior) unit_body(std::true_type{});
        else unit_body(std::false_type{});
    }
    if (HAS_DOT) {
        const double sum = consumer_sum<NC>(acc, red);
        if (tid == 0) P.part[blockIdx.x] = sum;
    }
}

// ============================================================================
// tail: levels lt..L-1 of one plane entirely in shared memory
// ============================================================================
struct TailParams {
    int lt, L, B;
    int words_plane;           // smem words per plane group
    int m[12];
    int off_b[12], off_x[12];  // smem word offsets per level
    int off_r;
    const double* tab;         // all levels [L][n_sets][10]
    int n_sets;
    const int* sid;
    const double* b;           // level lt rhs, B planes
    double* out;               // level lt solution (or finest epilogue target)
    int epi;
    double scale;
    const double* steps;
    const double* rsteps;
    const double* pin;
    const double* aux;
    double* part;
};

__device__ __forceinline__ double row_sum_any(const double* c, const double* v, int m, int y,
                                              int x) {
    const bool hs = y > 0, hn = y < m - 1, w = x > 0, e = x < m - 1;
    const double* r0 = v + y * m;
    return row_sum<SH_FULL>(c, r0 - m, r0, r0 + m, x, hs, hn, w, e);
}

// barrier over the GT threads of one plane group (named barrier 1 + group)
template <int GT, int GPB>
__device__ __forceinline__ void group_sync() {
    if constexpr (GT == 32)
        __syncwarp();
    else if constexpr (GPB == 1)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / GT)), "n"(GT) : "memory");
}

// GT threads cooperate on one plane; GPB planes per CTA (GT = 32: one warp
// per plane, no CTA barriers -- the small levels are pure latency otherwise)
template <int GT, int GPB>
__global__ void __launch_bounds__(GT * GPB) k_mg_tail(TailParams P) {
    extern __shared__ __align__(16) double smem_all[];
    const int tid = threadIdx.x % GT;
    const int grp = threadIdx.x / GT;
    double* smem = smem_all + (size_t)grp * P.words_plane;
    auto div_tau = [&](double v, int plane) {
        const double r = __ldg(P.rsteps + plane);
        return r > 0.0 ? v * r : v / __ldg(P.steps + plane);
    };
    double acc = 0.0;
    for (int plane = blockIdx.x * GPB + grp; plane < P.B; plane += gridDim.x * GPB) {
        const int set = __ldg(P.sid + plane);
        const int mt = P.m[P.lt];
        const long long nt = (long long)mt * mt;
        {
            double* B0 = smem + P.off_b[P.lt];
            const double* src = P.b + plane * nt;
            for (int i = tid; i < nt; i += GT) B0[i] = __ldg(src + i);
        }
        group_sync<GT, GPB>();
        // descend
        for (int l = P.lt; l + 1 < P.L; ++l) {
            const int m = P.m[l], mc = P.m[l + 1];
            const double* tb = P.tab + ((size_t)l * P.n_sets + set) * PINT_TW;
            double ca[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) ca[q] = __ldg(tb + q);
            const double d = __ldg(tb + 9);
            double* Bl = smem + P.off_b[l];
            double* Xl = smem + P.off_x[l];
            double* R = smem + P.off_r;
            for (int i = tid; i < m * m; i += GT) Xl[i] = d * Bl[i];
            group_sync<GT, GPB>();
            for (int i = tid; i < m * m; i += GT) {
                const int y = i / m, x = i - y * m;
                R[i] = Bl[i] - row_sum_any(ca, Xl, m, y, x);
            }
            group_sync<GT, GPB>();
            double* Bc = smem + P.off_b[l + 1];
            for (int i = tid; i < mc * mc; i += GT) {
                const int Y = i / mc, X = i - Y * mc;
                const double* r0 = R + (2 * Y) * m + 2 * X;
                const double* r1 = r0 + m;
                const double* r2 = r1 + m;
                double v = 0.25 * r0[0];
                v = v + 0.5 * r0[1];
                v = v + 0.25 * r0[2];
                v = v + 0.5 * r1[0];
                v = v + 1.0 * r1[1];
                v = v + 0.5 * r1[2];
                v = v + 0.25 * r2[0];
                v = v + 0.5 * r2[1];
                v = v + 0.25 * r2[2];
                Bc[i] = v;
            }
            group_sync<GT, GPB>();
        }
        // coarsest 1x1 (or general single point): x = b / a
        {
            const int l = P.L - 1;
            const double a = __ldg(P.tab + ((size_t)l * P.n_sets + set) * PINT_TW + 4);
            double* Bl = smem + P.off_b[l];
            double* Xl = smem + P.off_x[l];
            const int mm = P.m[l] * P.m[l];
            for (int i = tid; i < mm; i += GT) Xl[i] = Bl[i] / a;
            group_sync<GT, GPB>();
        }
        // ascend
        for (int l = P.L - 2; l >= P.lt; --l) {
            const int m = P.m[l], mc = P.m[l + 1];
            const double* tb = P.tab + ((size_t)l * P.n_sets + set) * PINT_TW;
            double ca[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) ca[q] = __ldg(tb + q);
            const double d = __ldg(tb + 9);
            double* Bl = smem + P.off_b[l];
            double* Xl = smem + P.off_x[l];
            const double* Ec = smem + P.off_x[l + 1];
            double* R = smem + P.off_r;
            for (int i = tid; i < m * m; i += GT) {
                const int y = i / m, x = i - y * m;
                int ja, jb, ia, ib;
                double wa, wb, ua, ub;
                if (y & 1) { ja = (y - 1) >> 1; wa = 1.0; jb = -1; wb = 0.0; }
                else { ja = (y >> 1) - 1; wa = 0.5; jb = y >> 1; wb = 0.5; }
                if (x & 1) { ia = (x - 1) >> 1; ua = 1.0; ib = -1; ub = 0.0; }
                else { ia = (x >> 1) - 1; ua = 0.5; ib = x >> 1; ub = 0.5; }
                const bool va = ja >= 0, vb2 = jb >= 0 && jb < mc;
                const bool ha = ia >= 0, hb = ib >= 0 && ib < mc;
                double pe = 0.0;
                bool first = true;
                auto add = [&](bool ok, double w, double e) {
                    if (!ok) return;
                    const double t = w * e;
                    pe = first ? t : pe + t;
                    first = false;
                };
                add(va && ha, wa * ua, va && ha ? Ec[ja * mc + ia] : 0.0);
                add(va && hb, wa * ub, va && hb ? Ec[ja * mc + ib] : 0.0);
                add(vb2 && ha, wb * ua, vb2 && ha ? Ec[jb * mc + ia] : 0.0);
                add(vb2 && hb, wb * ub, vb2 && hb ? Ec[jb * mc + ib] : 0.0);
                Xl[i] = Xl[i] + pe;  // x0 (= dinv*b, kept from the descent) + P e
            }
            group_sync<GT, GPB>();
            const bool top = (l == P.lt);
            const long long gplane = plane * (long long)m * m;
            for (int i = tid; i < m * m; i += GT) {
                const int y = i / m, x = i - y * m;
                const double bv = Bl[i];
                const double xn = Xl[i] + d * (bv - row_sum_any(ca, Xl, m, y, x));
                if (!top) {
                    R[i] = xn;
                    continue;
                }
                const long long gi = gplane + i;
                switch (P.epi) {
                    case EPI_PLAIN: P.out[gi] = xn; break;
                    case EPI_DIV_TAU: P.out[gi] = div_tau(xn, plane); break;
                    case EPI_UZAWA_P: {
                        const double dp = div_tau(xn, plane);
                        P.out[gi] = __ldg(P.pin + gi) + dp;
                        acc += bv * dp;
                        break;
                    }
                    case EPI_DOT_TAU: acc += bv * div_tau(xn, plane); break;
                    case EPI_SCALE: P.out[gi] = P.scale * xn; break;
                    case EPI_SCALE_DOT: {
                        const double w = P.scale * xn;
                        P.out[gi] = w;
                        acc += __ldg(P.aux + gi) * w;
                        break;
                    }
                    case EPI_SCALE_DOTONLY: acc += __ldg(P.aux + gi) * (P.scale * xn); break;
                }
            }
            group_sync<GT, GPB>();
            if (!top) {
                for (int i = tid; i < m * m; i += GT) Xl[i] = R[i];
                group_sync<GT, GPB>();
            }
        }
    }
    if (P.part != nullptr) {
        const double s = block_sum<GT * GPB>(acc);
        if (threadIdx.x == 0) P.part[blockIdx.x] = s;
    }
}

// ============================================================================
// host side
// ============================================================================
static bool epi_has_dot(int epi) {
    return epi == EPI_UZAWA_P || epi == EPI_DOT_TAU || epi == EPI_SCALE_DOT ||
           epi == EPI_SCALE_DOTONLY;
}

static int g_num_sms = 0;
static int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

constexpr int TAIL_MAX_M_DEFAULT = 31;  // m = 63 runs through the band kernels

// shapes of the level tables: a position is skipped only if it is exactly 0
// for every set of the level
void mg_compute_shapes(MgSet& set, const double* tab) {
    set.shape.assign(set.levels, SH_FULL);
    for (int l = 0; l < set.levels; ++l) {
        bool z[9] = {true, true, true, true, true, true, true, true, true};
        for (int s = 0; s < set.n_sets; ++s)
            for (int q = 0; q < 9; ++q)
                if (tab[((size_t)l * set.n_sets + s) * PINT_TW + q] != 0.0) z[q] = false;
        if (z[0] && z[2] && z[6] && z[8])
            set.shape[l] = SH_FIVE;
        else if (z[2] && z[6])
            set.shape[l] = SH_SEVEN;
    }
}

// tuning overrides (diagnostic sweeps only): PINT_STAGES, PINT_BAND, PINT_CTAS
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// largest level handled by the shared-memory tail kernel (PINT_TAIL_MAX_M)
static int tail_max_m() {
    static const int v = env_int("PINT_TAIL_MAX_M", TAIL_MAX_M_DEFAULT);
    return v;
}

// persistent grid: as many CTAs as are co-resident (registers and shared
// memory of this instantiation), never more than `cap`
template <typename K>
static int occupancy_grid(K kernel, int threads, size_t smem, int cap) {
    int occ = 0;
    PINT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    occ = std::max(occ, 1);
    const int lim = env_int("PINT_CTAS", 0);
    if (lim > 0) occ = std::min(occ, lim);
    return std::max(1, std::min(cap, num_sms() * occ));
}

template <int SH, int NT, int CPT, int HC>
static void launch_pre_h(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_pre<SH, NT, CPT, HC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    grid = occupancy_grid(k_band_pre<SH, NT, CPT, HC>, NT + 32, smem, grid);
    k_band_pre<SH, NT, CPT, HC><<<grid, NT + 32, smem, c->stream>>>(P);
}

template <int SH, int NT, int CPT>
static void launch_pre_cfg(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    if (P.Hc == 2)
        launch_pre_h<SH, NT, CPT, 2>(c, P, smem, grid);
    else
        launch_pre_h<SH, NT, CPT, 4>(c, P, smem, grid);
}

// planes per unit of the narrow band levels (k_band_pre2 / k_band_post2, PPU);
// PINT_PPU=1 restores one plane per unit
static int planes_per_unit(int nt) {
    static const int off = getenv("PINT_PPU") ? atoi(getenv("PINT_PPU")) == 1 : 0;
    return (nt <= 64 && !off) ? 128 / nt : 1;
}

template <int SH, int NT, int HC, int AR, int PPU>
static void launch_pre2_ppu(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_pre2<SH, NT, HC, AR, PPU>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    grid = occupancy_grid(k_band_pre2<SH, NT, HC, AR, PPU>, NT * PPU + 32, smem, grid);
    k_band_pre2<SH, NT, HC, AR, PPU><<<grid, NT * PPU + 32, smem, c->stream>>>(P);
}

template <int SH, int NT, int HC, int AR>
static void launch_pre2_ar(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    if constexpr (NT <= 64) {
        if (P.ppu > 1) {
            launch_pre2_ppu<SH, NT, HC, AR, 128 / NT>(c, P, smem, grid);
            return;
        }
    }
    launch_pre2_ppu<SH, NT, HC, AR, 1>(c, P, smem, grid);
}

template <int SH, int NT, int HC>
static void launch_pre2_h(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    if (P.aref) {
        // fused A_ref input: only the mode operators' shapes (mu M + tau A is 7- or 9-point)
        if constexpr (SH != SH_FIVE) launch_pre2_ar<SH, NT, HC, 1>(c, P, smem, grid);
        else pint_throw(PINT_INPUT, "fused A_ref input needs a mode-operator level");
        return;
    }
    launch_pre2_ar<SH, NT, HC, 0>(c, P, smem, grid);
}

template <int SH, int NT>
static void launch_pre2_nt(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    if (P.Hc == 2)
        launch_pre2_h<SH, NT, 2>(c, P, smem, grid);
    else
        launch_pre2_h<SH, NT, 4>(c, P, smem, grid);
}

static int pair_threads(int m) {
    const int mc = (m - 1) / 2;
    return ((mc + 1 + 31) / 32) * 32;
}

static bool use_pre2() {
    static const int v = getenv("PINT_PRE1") ? 0 : 1;
    return v != 0;
}

template <int SH>
static void launch_pre_sh(pint_ctx* c, const PreParams& P, size_t smem, int& grid) {
    if (use_pre2()) {
        switch (pair_threads(P.m)) {
            case 32: launch_pre2_nt<SH, 32>(c, P, smem, grid); return;
            case 64: launch_pre2_nt<SH, 64>(c, P, smem, grid); return;
            case 128: launch_pre2_nt<SH, 128>(c, P, smem, grid); return;
            case 256: launch_pre2_nt<SH, 256>(c, P, smem, grid); return;
            default: pint_throw(PINT_INPUT, "unsupported grid width for the paired pre kernel");
        }
    }
    if (P.m <= 128) launch_pre_cfg<SH, 128, 1>(c, P, smem, grid);
    else if (P.m <= 256) launch_pre_cfg<SH, 256, 1>(c, P, smem, grid);
    else if (P.m <= 512) launch_pre_cfg<SH, 256, 2>(c, P, smem, grid);
    else pint_throw(PINT_INPUT, "grid wider than 511 points is not supported");
}

template <int SH, int EPI, int NT, int CPT, int H>
static void launch_post_h(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_post<SH, EPI, NT, CPT, H>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    grid = occupancy_grid(k_band_post<SH, EPI, NT, CPT, H>, NT + 32, smem, grid);
    k_band_post<SH, EPI, NT, CPT, H><<<grid, NT + 32, smem, c->stream>>>(P);
}

template <int SH, int EPI, int NT, int CPT>
static void launch_post_cfg(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    if (P.H == 4)
        launch_post_h<SH, EPI, NT, CPT, 4>(c, P, smem, grid);
    else
        launch_post_h<SH, EPI, NT, CPT, 8>(c, P, smem, grid);
}

// rows per band (measured, tools/sweep_mg.py: taller bands do not help the
// coarse levels; 4 rows keep two CTAs per SM at m = 511)
static int band_rows(int m) {
    if (const char* e = getenv("PINT_BAND")) return atoi(e) <= 4 ? 4 : 8;
    return m > 300 ? 4 : 8;
}

template <int SH, int EPI, int NT, int H, int AR, int PPU>
static void launch_post2_ppu(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    static bool attr = false;
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(k_band_post2<SH, EPI, NT, H, AR, PPU>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    grid = occupancy_grid(k_band_post2<SH, EPI, NT, H, AR, PPU>, NT * PPU + 32, smem, grid);
    k_band_post2<SH, EPI, NT, H, AR, PPU><<<grid, NT * PPU + 32, smem, c->stream>>>(P);
}

template <int SH, int EPI, int NT, int H, int AR>
static void launch_post2_ar(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    if constexpr (NT <= 64) {
        if (P.ppu > 1) {
            launch_post2_ppu<SH, EPI, NT, H, AR, 128 / NT>(c, P, smem, grid);
            return;
        }
    }
    launch_post2_ppu<SH, EPI, NT, H, AR, 1>(c, P, smem, grid);
}

template <int SH, int EPI, int NT, int H>
static void launch_post2_h(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    if (P.aref) {
        // fused A_ref input: the second mode V-cycle (schur.py:73) epilogues only
        if constexpr (SH != SH_FIVE &&
                      (EPI == EPI_SCALE || EPI == EPI_SCALE_DOT || EPI == EPI_SCALE_DOTONLY))
            launch_post2_ar<SH, EPI, NT, H, 1>(c, P, smem, grid);
        else
            pint_throw(PINT_INPUT, "fused A_ref input needs a mode-operator level");
        return;
    }
    launch_post2_ar<SH, EPI, NT, H, 0>(c, P, smem, grid);
}

// consumer threads of the paired kernel: mc + 1 rounded up to warps
static int post2_threads(int m) {
    const int mc = (m - 1) / 2;
    return ((mc + 1 + 31) / 32) * 32;
}

template <int SH, int EPI, int NT>
static void launch_post2_nt(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    if (P.H == 4)
        launch_post2_h<SH, EPI, NT, 4>(c, P, smem, grid);
    else
        launch_post2_h<SH, EPI, NT, 8>(c, P, smem, grid);
}

template <int SH, int EPI>
static void launch_post2_epi(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    switch (post2_threads(P.m)) {
        case 32: launch_post2_nt<SH, EPI, 32>(c, P, smem, grid); break;
        case 64: launch_post2_nt<SH, EPI, 64>(c, P, smem, grid); break;
        case 128: launch_post2_nt<SH, EPI, 128>(c, P, smem, grid); break;
        case 256: launch_post2_nt<SH, EPI, 256>(c, P, smem, grid); break;
        default: pint_throw(PINT_INPUT, "unsupported grid width for the paired post kernel");
    }
}

static bool use_post2() {
    static const int v = getenv("PINT_POST1") ? 0 : 1;
    return v != 0;
}

template <int SH, int EPI>
static void launch_post_epi(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    if (use_post2()) {
        launch_post2_epi<SH, EPI>(c, P, smem, grid);
        return;
    }
    if (P.m <= 128) launch_post_cfg<SH, EPI, 128, 1>(c, P, smem, grid);
    else if (P.m <= 256) launch_post_cfg<SH, EPI, 256, 1>(c, P, smem, grid);
    else if (P.m <= 512) launch_post_cfg<SH, EPI, 256, 2>(c, P, smem, grid);
    else pint_throw(PINT_INPUT, "grid wider than 511 points is not supported");
}

template <int SH>
static void launch_post_sh(pint_ctx* c, const PostBandParams& P, size_t smem, int& grid) {
    switch (P.epi) {
        case EPI_PLAIN: launch_post_epi<SH, EPI_PLAIN>(c, P, smem, grid); break;
        case EPI_DIV_TAU: launch_post_epi<SH, EPI_DIV_TAU>(c, P, smem, grid); break;
        case EPI_UZAWA_P: launch_post_epi<SH, EPI_UZAWA_P>(c, P, smem, grid); break;
        case EPI_DOT_TAU: launch_post_epi<SH, EPI_DOT_TAU>(c, P, smem, grid); break;
        case EPI_SCALE: launch_post_epi<SH, EPI_SCALE>(c, P, smem, grid); break;
        case EPI_SCALE_DOT: launch_post_epi<SH, EPI_SCALE_DOT>(c, P, smem, grid); break;
        case EPI_SCALE_DOTONLY: launch_post_epi<SH, EPI_SCALE_DOTONLY>(c, P, smem, grid); break;
        default: pint_throw(PINT_INPUT, "unknown epilogue");
    }
}

// Stages of the TMA ring.  Measured on B200 (tools/sweep_mg.py): two stages
// and as many CTAs per SM as fit beat deeper rings, so keep two.
static int pick_stages(int words_stage, int words_work) {
    (void)words_stage;
    (void)words_work;
    return 2;
}


static int blocks_per_sm(size_t smem) {
    const size_t per_sm = 227 * 1024;
    int k = (int)(per_sm / (smem + 1024));
    if (k < 1) k = 1;
    if (k > 4) k = 4;
    const int cap = env_int("PINT_CTAS", 0);
    if (cap > 0 && cap < k) k = cap;
    return k;
}

bool vcycle_aref_fusable(const pint_ctx* c, int which) {
    if (c->dims != 2 || c->field || getenv("PINT_AREF_SEPARATE")) return false;
    if (!use_pre2() || !use_post2()) return false;
    const MgSet& s = c->mg[which];
    if (!s.ready || s.levels < 2 || s.m[0] <= tail_max_m() || s.shape[0] == SH_FIVE) return false;
    if (c->h_aref.size() != 9) return false;
    const double* z = c->h_aref.data();
    return z[0] == 0.0 && z[2] == 0.0 && z[6] == 0.0 && z[8] == 0.0;  // 5-point A_ref
}

void vcycle(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
            double scale, const double* pin, const double* aux, int acc_slot, bool aref_in) {
    if (aref_in && !vcycle_aref_fusable(c, which))
        pint_throw(PINT_INPUT, "fused A_ref V-cycle input is not available for this problem");
    if (c->dims == 3) {
        vcycle3(c, which, count, b, out, epi, scale, pin, aux, acc_slot);
        return;
    }
    if (c->field) {
        vcycle_field(c, which, count, b, out, epi, scale, pin, aux, acc_slot);
        return;
    }
    MgSet& s = c->mg[which];
    if (!s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    const int L = s.levels;
    auto lvl_tab = [&](int l) { return s.tab + (size_t)l * s.n_sets * PINT_TW; };
    int lt = 0;
    while (lt < L && s.m[lt] > tail_max_m()) ++lt;
    const int sms = num_sms();
    const bool dot = epi_has_dot(epi);
    // ---- descend through the band levels ----
    const double* bl = b;
    for (int l = 0; l < lt; ++l) {
        PreParams P{};
        P.m = s.m[l];
        P.mc = s.m[l + 1];
        P.B = count;
        P.Hc = band_rows(P.m) / 2;  // coarse rows per unit
        P.nbands = (P.mc + P.Hc - 1) / P.Hc;
        P.aref = (aref_in && l == 0) ? 1 : 0;
        if (P.aref) {
            for (int q = 0; q < 9; ++q) P.ar[q] = c->h_aref[q];
            P.Hc = env_int("PINT_AR_HC", P.Hc) <= 2 ? 2 : 4;
            P.nbands = (P.mc + P.Hc - 1) / P.Hc;
        }
        P.words_b = band_words(2 * P.Hc + 3 + 2 * P.aref, P.m);
        P.words_r = use_pre2() ? (2 * P.Hc + 1) * (P.m + 3) : ((2 * P.Hc + 1) * P.m + 1) / 2 * 2;
        P.stages = env_int("PINT_STAGES", pick_stages(P.words_b, P.words_r));
        P.ppu = use_pre2() ? planes_per_unit(pair_threads(P.m)) : 1;
        P.b = bl;
        P.bc = c->lev_b[l + 1];
        P.tab = lvl_tab(l);
        P.sid = s.sid;
        const size_t smem = sizeof(double) * P.ppu * (P.stages * P.words_b + P.words_r);
        const int units = (P.B + P.ppu - 1) / P.ppu * P.nbands;
        int grid = std::min(units, sms * (l == 0 ? 8 : env_int("PINT_COARSE_CTAS", 8)));
        ProfScope prof(c, l == 0 ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                       8.0 * count * ((double)P.m * P.m + (double)P.mc * P.mc));
        switch (s.shape[l]) {
            case SH_FULL: launch_pre_sh<SH_FULL>(c, P, smem, grid); break;
            case SH_SEVEN: launch_pre_sh<SH_SEVEN>(c, P, smem, grid); break;
            default: launch_pre_sh<SH_FIVE>(c, P, smem, grid); break;
        }
        PINT_LAUNCHED(c);
        bl = c->lev_b[l + 1];
    }
    PINT_CUDA_CHECK(cudaGetLastError());
    // ---- tail: levels lt..L-1 in shared memory ----
    {
        TailParams T{};
        T.lt = lt;
        T.L = L;
        T.B = count;
        int off = 0;
        int maxm2 = 0;
        for (int l = lt; l < L; ++l) {
            T.m[l] = s.m[l];
            T.off_b[l] = off;
            off += ((s.m[l] * s.m[l] + 1) / 2) * 2;
            T.off_x[l] = off;
            off += ((s.m[l] * s.m[l] + 1) / 2) * 2;
            maxm2 = std::max(maxm2, s.m[l] * s.m[l]);
        }
        T.off_r = off;
        off += maxm2;
        T.tab = s.tab;
        T.n_sets = s.n_sets;
        T.sid = s.sid;
        T.b = bl;
        const bool top = lt == 0;
        T.out = top ? out : c->lev_x[lt];
        T.epi = top ? epi : EPI_PLAIN;
        T.scale = scale;
        T.steps = c->d_steps;
        T.rsteps = c->d_rsteps;
        T.pin = pin;
        T.aux = aux;
        T.words_plane = (off + 1) / 2 * 2;
        int gpb = (int)((200 * 1024) / (sizeof(double) * (size_t)T.words_plane));
        gpb = std::max(1, std::min(8, gpb));
        const bool warp_mode = s.m[lt] <= 31 && gpb >= 1;
        if (!warp_mode) gpb = 1;
        const size_t smem = sizeof(double) * (size_t)T.words_plane * gpb;
        static bool attr = false;
        if (!attr) {
            PINT_CUDA_CHECK(cudaFuncSetAttribute(k_mg_tail<32, 8>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 220 * 1024));
            PINT_CUDA_CHECK(cudaFuncSetAttribute(k_mg_tail<64, 4>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 220 * 1024));
            PINT_CUDA_CHECK(cudaFuncSetAttribute(k_mg_tail<128, 4>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 220 * 1024));
            PINT_CUDA_CHECK(cudaFuncSetAttribute(k_mg_tail<TT, 1>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 220 * 1024));
            attr = true;
        }
        if (smem > 220 * 1024) pint_throw(PINT_INPUT, "multigrid tail does not fit shared memory");
        // plane groups of the warp-mode tail: GT threads per plane, GPB planes per CTA
        // (PINT_TAIL_GT = 32 / 64 / 128 for A/B runs)
        const int tail_gt = warp_mode ? env_int("PINT_TAIL_GT", 64) : TT;
        const int per_cta = !warp_mode ? 1 : tail_gt == 32 ? 8 : 4;
        const int ctas_needed = (count + per_cta - 1) / per_cta;
        const size_t smem_cta = sizeof(double) * (size_t)T.words_plane * per_cta;
        int occ_tail = 1;
        if (warp_mode) occ_tail = std::max(1, (int)((227 * 1024) / (smem_cta + 1024)));
        const int grid = std::min(ctas_needed, sms * (warp_mode ? occ_tail : blocks_per_sm(smem)));
        if (top && dot) {
            ensure_partials(c, grid);
            T.part = c->d_part;
        }
        const double fine = (double)s.m[lt] * s.m[lt];
        ProfScope prof(c, top ? K_MG_POST_FINE : K_MG_TAIL, 8.0 * count * 2.0 * fine);
        if (warp_mode) {
            if (smem_cta > 220 * 1024) pint_throw(PINT_INPUT, "multigrid tail does not fit shared memory");
            if (tail_gt == 128) k_mg_tail<128, 4><<<grid, 512, smem_cta, c->stream>>>(T);
            else if (tail_gt == 64) k_mg_tail<64, 4><<<grid, 256, smem_cta, c->stream>>>(T);
            else k_mg_tail<32, 8><<<grid, 256, smem_cta, c->stream>>>(T);
        } else {
            k_mg_tail<TT, 1><<<grid, TT, smem, c->stream>>>(T);
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        if (top && dot) reduce_partials(c, grid, acc_slot);
    }
    // ---- ascend through the band levels ----
    for (int l = lt - 1; l >= 0; --l) {
        PostBandParams P{};
        P.m = s.m[l];
        P.mc = s.m[l + 1];
        P.B = count;
        P.H = band_rows(P.m);
        P.nbands = (P.m + P.H - 1) / P.H;
        const bool top = l == 0;
        P.epi = top ? epi : EPI_PLAIN;
        const bool has_q = P.epi == EPI_UZAWA_P || P.epi == EPI_SCALE_DOT ||
                           P.epi == EPI_SCALE_DOTONLY;
        P.aref = (aref_in && top) ? 1 : 0;
        if (P.aref)
            for (int q = 0; q < 9; ++q) P.ar[q] = c->h_aref[q];
        P.words_b = band_words(P.H + 2 + 2 * P.aref, P.m);
        P.words_e = band_words(P.H / 2 + 2, P.mc);
        P.words_q = has_q ? band_words(P.H, P.m) : 0;
        P.words_x = (P.H + 2) * (use_post2() ? P.m + 3 : P.m + 2);
        P.stages = env_int("PINT_STAGES", pick_stages(P.words_b + P.words_e + P.words_q, P.words_x));
        P.ppu = use_post2() ? planes_per_unit(post2_threads(P.m)) : 1;
        P.b = top ? b : c->lev_b[l];
        P.ec = c->lev_x[l + 1];
        P.tab = lvl_tab(l);
        P.sid = s.sid;
        P.out = top ? out : c->lev_x[l];
        P.scale = scale;
        P.steps = c->d_steps;
        P.rsteps = c->d_rsteps;
        P.pin = pin;
        P.aux = aux;
        const size_t smem =
            sizeof(double) * P.ppu * (P.stages * (P.words_b + P.words_e + P.words_q) + P.words_x);
        const int units = (P.B + P.ppu - 1) / P.ppu * P.nbands;
        int grid = std::min(units, sms * (l == 0 ? 8 : env_int("PINT_COARSE_CTAS", 8)));
        const bool dl = top && dot;
        if (dl) {
            ensure_partials(c, grid);
            P.part = c->d_part;
        }
        const double fine = (double)P.m * P.m, coarse = (double)P.mc * P.mc;
        double words = fine + coarse;
        if (P.epi != EPI_DOT_TAU && P.epi != EPI_SCALE_DOTONLY) words += fine;
        if (has_q) words += fine;
        {
            ProfScope prof(c, top ? K_MG_POST_FINE : K_MG_POST_COARSE, 8.0 * count * words);
            switch (s.shape[l]) {
                case SH_FULL: launch_post_sh<SH_FULL>(c, P, smem, grid); break;
                case SH_SEVEN: launch_post_sh<SH_SEVEN>(c, P, smem, grid); break;
                default: launch_post_sh<SH_FIVE>(c, P, smem, grid); break;
            }
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        if (dl) reduce_partials(c, grid, acc_slot);
    }
}

}  // namespace PINT_VARIANT
}  // namespace pint
