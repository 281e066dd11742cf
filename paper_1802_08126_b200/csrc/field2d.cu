// Variable-coefficient 2D stiffness: A_n with per-point coefficients
// (BASELINE config 4, -div(a(x,t) grad u)).  EXTENSION:
// the reference accepts any list of stiffness matrices (problems.py:153-165,
// operators.py:92-99 general branch, solvers.py:134-140 one hierarchy per
// distinct A_n); this file is the GPU form of that general branch for
// structured 2D grids whose operators are not translation invariant.
//
// Storage:
//   * fine A_n, compact: [N][3][n] = centre, east, north coefficient of every
//     row; the west / south entries of row i are the east / north entries of
//     rows i-1 / i-m (the reference materialises the lower triangle as a
//     mirror of the upper one, linalg.py:49-59), the SW / NE hypotenuse
//     entries are stored zeros of the P1 diagonal split;
//   * A_ref: one compact field [3][n];
//   * H_k = mu_k M + tau_ref A_ref is never stored on the fine level: its
//     coefficients fl(mu_k m) + fl(tau_ref a) are formed on the fly;
//   * coarse Galerkin operators of every set (step or mode): full 9-point
//     rows [sets][9][m_l^2], computed on the GPU in scipy's SpGEMM
//     accumulation order so they are bit-identical to the reference's
//     (P^T A) P (spatial.py:140).
//
// Every row sum follows CSR column order from 0 without FMA (-fmad=false),
// so results are bit-identical to scipy's csr_matvec on the same matrices.
// Round-1 form: one thread per point, neighbours through L1/L2.
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <type_traits>

#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

namespace {

#ifndef PINT_FG
#define PINT_FG 16
#endif
constexpr int FX = 32, FY = 8, FG = PINT_FG;  // 32x8 tile, FG time planes per CTA (marching ops)
constexpr int FT = 256;

// FM_SA / FM_S9 (separable families, pint_field_separable): the operator of
// set s is sum_r sc[s][r] T_r with R time-independent term tables T_r (compact
// [R][3][n] on the fine level, [R][9][m_l^2] Galerkin rows below), so the
// per-set coefficients are formed in registers from cache-resident tables
// instead of being streamed from [sets][..] slabs.
enum FieldMode : int { FM_A = 0, FM_H = 1, FM_9 = 2, FM_SA = 3, FM_S9 = 4 };
constexpr int FSEP_MAX = PINT_FSEP_MAX;

struct Src {
    const double* f = nullptr;     // FM_A: compact [sets][3][n]; FM_9: [sets][9][n]; FM_S*: term tables
    size_t set_stride = 0;         // doubles between consecutive sets (0: shared by all)
    const double* mass = nullptr;  // FM_H: constant mass stencil [9] (device copy, unused by the kernels)
    double massv[9] = {};          // FM_H: the same stencil by value (kernel-parameter constants: no
                                   // load instructions; ncu showed the fine H~ residual LSU bound at 92 %)
    const double* mu = nullptr;    // FM_H: per-set weight mu_k
    double tau = 0.0;              // FM_H: tau_ref
    const double* sc = nullptr;    // FM_S*: per-set term weights [sets][R]
    int R = 0;                     // FM_S*: number of terms (<= FSEP_MAX)
    size_t term_stride = 0;        // FM_S*: doubles between term tables
};

// term weights of set s in registers
struct SepW {
    double w[FSEP_MAX];
    int R;
    ptrdiff_t ts;
};

__device__ __forceinline__ SepW sep_load(const Src& S, int s) {
    SepW W;
    W.R = S.R;
    W.ts = (ptrdiff_t)S.term_stride;
#pragma unroll
    for (int r = 0; r < FSEP_MAX; ++r) W.w[r] = r < S.R ? __ldg(S.sc + (size_t)s * S.R + r) : 0.0;
    return W;
}

// sum_r w_r T_r[p]
__device__ __forceinline__ double sep_at(const SepW& W, const double* p) {
    double v = W.w[0] * __ldg(p);
#pragma unroll
    for (int r = 1; r < FSEP_MAX; ++r)
        if (r < W.R) v = fma(W.w[r], __ldg(p + r * W.ts), v);
    return v;
}

// coefficient k (CSR position SW,S,SE,W,C,E,NW,N,NE) of row (x, y) of set s;
// only called when that neighbour exists
template <int MODE>
__device__ __forceinline__ double coef(const Src& S, int s, int k, int m, int x, int y) {
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    if (MODE == FM_SA || MODE == FM_S9) {
        const SepW W = sep_load(S, s);
        if (MODE == FM_S9) return sep_at(W, S.f + (size_t)k * n + i);
        switch (k) {
            case 1: return sep_at(W, S.f + 2 * n + i - m);
            case 3: return sep_at(W, S.f + n + i - 1);
            case 4: return sep_at(W, S.f + i);
            case 5: return sep_at(W, S.f + n + i);
            case 7: return sep_at(W, S.f + 2 * n + i);
            default: return 0.0;
        }
    }
    const double* f = S.f + (size_t)s * S.set_stride;
    if (MODE == FM_9) return __ldg(f + (size_t)k * n + i);
    double a;
    switch (k) {
        case 1: a = __ldg(f + 2 * n + i - m); break;  // S = north entry of row i-m
        case 3: a = __ldg(f + n + i - 1); break;      // W = east entry of row i-1
        case 4: a = __ldg(f + i); break;
        case 5: a = __ldg(f + n + i); break;
        case 7: a = __ldg(f + 2 * n + i); break;
        default: a = 0.0;
    }
    if (MODE == FM_A) return a;
    // add_matrices(mu_k, M, 1.0, A_ref.scaled(tau_ref)) entry (schur.py:41-47, linalg.py:118-127)
    return __ldg(S.mu + s) * S.massv[k] + 1.0 * (S.tau * a);
}

template <int MODE>
__device__ __forceinline__ bool structural(int k) {
    // FM_A: only S, W, C, E, N can be non-zero (SW / NE are stored zeros);
    // FM_H: SE / NW are absent from both M and A
    if (MODE == FM_A || MODE == FM_SA) return k == 1 || k == 3 || k == 4 || k == 5 || k == 7;
    if (MODE == FM_H) return k != 2 && k != 6;
    return true;
}

// CSR row sum at (x, y) of plane v (m x m): sum = 0; sum += a_k v_k in column order.
// Same terms, coefficients and order as evaluating coef<MODE>() for k = 0..8
// (structural positions whose neighbour exists), with the row's base
// pointers formed once: ncu of the generic loop showed 220 instructions per
// point, almost all 64-bit index arithmetic.
template <int MODE>
__device__ __forceinline__ double frow(const Src& S, int s, const double* __restrict__ v, int m,
                                      int x, int y) {
    const int i = y * m + x;
    const ptrdiff_t n = (ptrdiff_t)m * m;
    const bool w = x > 0, e = x < m - 1, so = y > 0, no = y < m - 1;
    const double* vi = v + i;
    double r = 0.0;
    if constexpr (MODE == FM_S9 || MODE == FM_SA) {
        const SepW W = sep_load(S, s);
        const double* f = S.f + i;
        if constexpr (MODE == FM_S9) {
            if (so && w) r = r + sep_at(W, f) * __ldg(vi - m - 1);
            if (so) r = r + sep_at(W, f + n) * __ldg(vi - m);
            if (so && e) r = r + sep_at(W, f + 2 * n) * __ldg(vi - m + 1);
            if (w) r = r + sep_at(W, f + 3 * n) * __ldg(vi - 1);
            r = r + sep_at(W, f + 4 * n) * __ldg(vi);
            if (e) r = r + sep_at(W, f + 5 * n) * __ldg(vi + 1);
            if (no && w) r = r + sep_at(W, f + 6 * n) * __ldg(vi + m - 1);
            if (no) r = r + sep_at(W, f + 7 * n) * __ldg(vi + m);
            if (no && e) r = r + sep_at(W, f + 8 * n) * __ldg(vi + m + 1);
        } else {
            if (so) r = r + sep_at(W, f + 2 * n - m) * __ldg(vi - m);
            if (w) r = r + sep_at(W, f + n - 1) * __ldg(vi - 1);
            r = r + sep_at(W, f) * __ldg(vi);
            if (e) r = r + sep_at(W, f + n) * __ldg(vi + 1);
            if (no) r = r + sep_at(W, f + 2 * n) * __ldg(vi + m);
        }
        return r;
    }
    const double* f = S.f + (size_t)s * S.set_stride + i;  // centre entry of this row
    if constexpr (MODE == FM_9) {
        if (so && w) r = r + __ldg(f) * __ldg(vi - m - 1);
        if (so) r = r + __ldg(f + n) * __ldg(vi - m);
        if (so && e) r = r + __ldg(f + 2 * n) * __ldg(vi - m + 1);
        if (w) r = r + __ldg(f + 3 * n) * __ldg(vi - 1);
        r = r + __ldg(f + 4 * n) * __ldg(vi);
        if (e) r = r + __ldg(f + 5 * n) * __ldg(vi + 1);
        if (no && w) r = r + __ldg(f + 6 * n) * __ldg(vi + m - 1);
        if (no) r = r + __ldg(f + 7 * n) * __ldg(vi + m);
        if (no && e) r = r + __ldg(f + 8 * n) * __ldg(vi + m + 1);
        return r;
    } else {
        // compact fields: centre f, east f + n, north f + 2n; S / W are the
        // north / east entries of rows i - m / i - 1
        const double aS = so ? __ldg(f + 2 * n - m) : 0.0;
        const double aW = w ? __ldg(f + n - 1) : 0.0;
        const double aC = __ldg(f);
        const double aE = e ? __ldg(f + n) : 0.0;
        const double aN = no ? __ldg(f + 2 * n) : 0.0;
        if constexpr (MODE == FM_A) {
            if (so) r = r + aS * __ldg(vi - m);
            if (w) r = r + aW * __ldg(vi - 1);
            r = r + aC * __ldg(vi);
            if (e) r = r + aE * __ldg(vi + 1);
            if (no) r = r + aN * __ldg(vi + m);
        } else {
            // mu_k M + tau A_ref entry: add_matrices(mu_k, M, 1.0, A_ref.scaled(tau_ref))
            // (schur.py:41-47, linalg.py:118-127); SW / NE carry mass only
            const double mu = __ldg(S.mu + s), tau = S.tau;
            auto hc = [&](int k, double a) { return mu * S.massv[k] + 1.0 * (tau * a); };
            if (so && w) r = r + hc(0, 0.0) * __ldg(vi - m - 1);
            if (so) r = r + hc(1, aS) * __ldg(vi - m);
            if (w) r = r + hc(3, aW) * __ldg(vi - 1);
            r = r + hc(4, aC) * __ldg(vi);
            if (e) r = r + hc(5, aE) * __ldg(vi + 1);
            if (no) r = r + hc(7, aN) * __ldg(vi + m);
            if (no && e) r = r + hc(8, 0.0) * __ldg(vi + m + 1);
        }
        return r;
    }
}

// ---- assembly ------------------------------------------------------------------
// Compact fields of the P1 stiffness with per-cell weights w[j][i] (both
// triangles of cell (i, j) carry the weight; problems.py:99-138 element loop
// with w_e K_e).  The centre is the sum of six triangle contributions in the
// order scipy's coo -> csr conversion sums the duplicates (sort_indices, then
// left to right; translation invariant, probed by tests/test_field.py); east
// and north are two-term sums (order-free).
__global__ void __launch_bounds__(FT)
    k_f_assemble(int c, const double* __restrict__ w, double* __restrict__ fa) {
    const int m = c - 1;
    const size_t n = (size_t)m * m;
    const long long g = (long long)blockIdx.x * FT + threadIdx.x;
    if (g >= (long long)n) return;
    const int t = blockIdx.y;
    const int g32 = (int)g;
    const int jj = g32 / m, ii = g32 - jj * m;
    const int i = ii + 1, j = jj + 1;
    const double* W = w + (size_t)t * c * c;
    auto cw = [&](int ci, int cj) { return __ldg(W + (size_t)cj * c + ci); };
    double s = cw(i - 1, j - 1) * 0.5;
    s = s + cw(i, j) * 0.5;
    s = s + cw(i, j) * 0.5;
    s = s + cw(i - 1, j) * 1.0;
    s = s + cw(i, j - 1) * 1.0;
    s = s + cw(i - 1, j - 1) * 0.5;
    // entries towards the Dirichlet boundary do not exist: stored as 0
    const double e = ii < m - 1 ? cw(i, j) * -0.5 + cw(i, j - 1) * -0.5 : 0.0;
    const double no = jj < m - 1 ? cw(i, j) * -0.5 + cw(i - 1, j) * -0.5 : 0.0;
    double* F = fa + (size_t)t * 3 * n;
    F[g] = s;
    F[n + g] = e;
    F[2 * n + g] = no;
}

// ---- time-global operators ---------------------------------------------------------
template <int OP, int MODE>
__global__ void __launch_bounds__(FX* FY)
    k_f_timeop(int m, int N, int qmin, int qmax, const double* __restrict__ mass, Src A,
               const double* __restrict__ ascale, const double* __restrict__ u,
               const double* __restrict__ p, const double* __restrict__ f,
               double* __restrict__ out) {
    const int x = blockIdx.x * FX + threadIdx.x;
    const int y = blockIdx.y * FY + threadIdx.y;
    if (x >= m || y >= m) return;
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    const int n0 = blockIdx.z * FG;
    const int n1 = min(N, n0 + FG);
    double cm[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) cm[k] = __ldg(mass + k);
    auto Mv = [&](const double* v, long long t) { return stencil9_global(cm, v + t * (long long)n, m, x, y); };
    auto Av = [&](const double* v, int t) {
        return __ldg(ascale + t) * frow<MODE>(A, t, v + (size_t)t * n, m, x, y);
    };
    if (OP == OP_ABD) {
        for (int t = n0; t < n1; ++t) out[t * n + i] = Av(u, t);
        return;
    }
    if (OP == OP_R1) {
        double mprev = (n0 - 1 >= qmin) ? Mv(u, n0 - 1) : 0.0;
        for (int t = n0; t < n1; ++t) {
            const double mcur = Mv(u, t);
            const double ku = (t - 1 >= qmin) ? mcur - mprev : mcur;
            out[t * n + i] = (ku - Av(p, t)) - __ldg(f + t * n + i);
            mprev = mcur;
        }
        return;
    }
    // OP_Z
    double muprev = (n0 - 1 >= qmin) ? Mv(u, n0 - 1) : 0.0;
    double mucur = Mv(u, n0), mpcur = Mv(p, n0);
    for (int t = n0; t < n1; ++t) {
        const bool hn = t + 1 <= qmax;
        const double munext = hn ? Mv(u, t + 1) : 0.0;
        const double mpnext = hn ? Mv(p, t + 1) : 0.0;
        const double ktp = hn ? mpcur - mpnext : mpcur;
        const double ku = (t - 1 >= qmin) ? mucur - muprev : mucur;
        const double ktu = hn ? mucur - munext : mucur;
        out[t * n + i] = (__ldg(f + t * n + i) - ktp) - ((ku + ktu) + Av(u, t));
        muprev = mucur;
        mucur = munext;
        mpcur = mpnext;
    }
}

// out_t = A_set(t) in_t over `count` planes
template <int MODE>
__global__ void __launch_bounds__(FX* FY)
    k_f_apply(int m, int count, Src A, const double* __restrict__ in, double* __restrict__ out) {
    const int x = blockIdx.x * FX + threadIdx.x;
    const int y = blockIdx.y * FY + threadIdx.y;
    if (x >= m || y >= m) return;
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    const int n0 = blockIdx.z * FG;
    const int n1 = min(count, n0 + FG);
    for (int t = n0; t < n1; ++t) out[t * n + i] = frow<MODE>(A, t, in + (size_t)t * n, m, x, y);
}

// ---- multigrid -----------------------------------------------------------------------
// x / y out of line, so a select with v * (1/tau) is not if-converted into an
// unconditional division
__device__ __noinline__ double fdiv_rn(double x, double y) { return x / y; }

// The V-cycle kernels below run one thread per point of a 64 x 4 tile of a
// plane (blockIdx.z = plane): no index divisions, 32-bit offsets inside the
// plane (ncu of the linear-index form: 100-220 instructions per point, almost
// all index arithmetic; the prolongation issue bound at 82 %).
constexpr int GX = 64, GY = 4;

// x0 = dinv * b with dinv = damping / diag  (spatial.py:142, 153)
template <int MODE>
__global__ void __launch_bounds__(FT)
    k_f_x0(int m, Src A, double damping, const double* __restrict__ b, double* __restrict__ x0) {
    const int x = blockIdx.x * GX + threadIdx.x, y = blockIdx.y * GY + threadIdx.y;
    if (x >= m || y >= m) return;
    const int t = blockIdx.z;
    const size_t gi = (size_t)t * m * m + (y * m + x);
    const double d = damping / coef<MODE>(A, t, 4, m, x, y);
    x0[gi] = d * __ldg(b + gi);
}

// b_c = P^T (b - A x0): the nine fine residuals of each coarse point, summed
// over ascending fine index with weights (1/4, 1/2, 1) (spatial.py:156)
// (round-1 form, kept for A/B: PINT_FIELD_RR)
template <int MODE>
__global__ void __launch_bounds__(FT)
    k_f_rr(int m, int mc, Src A, const double* __restrict__ b, const double* __restrict__ x0,
           double* __restrict__ bc) {
    const int X = blockIdx.x * GX + threadIdx.x, Y = blockIdx.y * GY + threadIdx.y;
    if (X >= mc || Y >= mc) return;
    const int t = blockIdx.z;
    const size_t n = (size_t)m * m, nc = (size_t)mc * mc;
    const double* bp = b + (size_t)t * n;
    const double* xp = x0 + (size_t)t * n;
    const double wt[3] = {0.5, 1.0, 0.5};
    double v = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int fy = 2 * Y + a, fx = 2 * X + q;
            const double r = __ldg(bp + fy * m + fx) - frow<MODE>(A, t, xp, m, fx, fy);
            const double term = (wt[a] * wt[q]) * r;
            v = (a == 0 && q == 0) ? term : v + term;
        }
    bc[t * nc + (Y * mc + X)] = v;
}

// r = b - A x0, one thread per FINE point (k_f_rr evaluates every fine
// residual once per coarse point it feeds: 2.25 times on average)
template <int MODE>
__global__ void __launch_bounds__(FT)
    k_f_resid(int m, Src A, const double* __restrict__ b, const double* __restrict__ x0,
              double* __restrict__ r) {
    const int x = blockIdx.x * GX + threadIdx.x, y = blockIdx.y * GY + threadIdx.y;
    if (x >= m || y >= m) return;
    const int t = blockIdx.z;
    const size_t pb = (size_t)t * m * m;
    const int i = y * m + x;
    r[pb + i] = __ldg(b + pb + i) - frow<MODE>(A, t, x0 + pb, m, x, y);
}

// b_c = P^T r from stored residuals: same nine terms, order and weights as k_f_rr
__global__ void __launch_bounds__(FT)
    k_f_restrict(int m, int mc, const double* __restrict__ r, double* __restrict__ bc) {
    const int X = blockIdx.x * GX + threadIdx.x, Y = blockIdx.y * GY + threadIdx.y;
    if (X >= mc || Y >= mc) return;
    const int t = blockIdx.z;
    const double* rp = r + (size_t)t * m * m + (2 * Y) * m + 2 * X;
    const double wt[3] = {0.5, 1.0, 0.5};
    double v = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double term = (wt[a] * wt[q]) * __ldg(rp + a * m + q);
            v = (a == 0 && q == 0) ? term : v + term;
        }
    bc[(size_t)t * mc * mc + (Y * mc + X)] = v;
}

// x = x0 + P e (csr_matvec of P, ascending coarse index); on the last
// level above the 1x1 coarsest grid e = b_c / a_c (spatial.py:149-150, 157).
// Per axis an odd coordinate has one term (weight 1), an even one the two
// neighbours (weight 1/2 each, those inside the coarse grid).
template <bool DIRECT, int MODE>
__global__ void __launch_bounds__(FT)
    k_f_prolong(int m, int mc, Src Ac, const double* __restrict__ ec, double* __restrict__ x) {
    // DIRECT is a template parameter: a runtime flag lets the compiler
    // evaluate e / 1.0 speculatively for every term
    const int xx = blockIdx.x * GX + threadIdx.x, y = blockIdx.y * GY + threadIdx.y;
    if (xx >= m || y >= m) return;
    const int t = blockIdx.z;
    const int nc = mc * mc;
    const double ac = DIRECT ? coef<MODE>(Ac, t, 4, mc, 0, 0) : 1.0;  // DIRECT: mc == 1
    const bool yo = y & 1, xo = xx & 1;
    const int ja = (y - 1) >> 1, ia = (xx - 1) >> 1;      // first term of each axis
    const bool va = ja >= 0, vb = !yo && ja + 1 < mc;      // rows ja, ja + 1
    const bool ha = ia >= 0, hb = !xo && ia + 1 < mc;      // columns ia, ia + 1
    // every existing term carries the weight wy * wx (1, 1/2 or 1/4)
    const double w = (yo ? 1.0 : 0.5) * (xo ? 1.0 : 0.5);
    const double* ep = ec + (size_t)t * nc + (ja * mc + ia);
    double pe = 0.0;
    bool first = true;
    auto add = [&](bool ok, int off) {
        if (!ok) return;
        double e = __ldg(ep + off);
        if (DIRECT) e = e / ac;
        const double term = w * e;
        pe = first ? term : pe + term;
        first = false;
    };
    add(va && ha, 0);
    add(va && hb, 1);
    add(vb && ha, mc);
    add(vb && hb, mc + 1);
    double* xp = x + (size_t)t * m * m + (y * m + xx);
    *xp = *xp + pe;
}

struct FSmooth {
    int m;
    const double* b;
    const double* x;
    double* out;
    int epi;
    double damping, scale;
    const double* steps;
    const double* rsteps;
    const double* pin;
    const double* aux;
    double* part;
};

// x += dinv (b - A x)  (spatial.py:159-160) and the finest-level epilogues
template <int MODE>
__global__ void __launch_bounds__(FT) k_f_smooth(Src A, FSmooth P) {
    const int m = P.m;
    const int x = blockIdx.x * GX + threadIdx.x, y = blockIdx.y * GY + threadIdx.y;
    const int t = blockIdx.z;
    double acc = 0.0;
    if (x < m && y < m) {
        const size_t n = (size_t)m * m;
        const size_t gi = (size_t)t * n + (y * m + x);
        const double d = P.damping / coef<MODE>(A, t, 4, m, x, y);
        const double bv = __ldg(P.b + gi);
        const double xn = __ldg(P.x + gi) + d * (bv - frow<MODE>(A, t, P.x + (size_t)t * n, m, x, y));
        const double rtau = __ldg(P.rsteps + t);
        auto divtau = [&](double v) { return rtau > 0.0 ? v * rtau : fdiv_rn(v, __ldg(P.steps + t)); };
        switch (P.epi) {
            case EPI_PLAIN: P.out[gi] = xn; break;
            case EPI_DIV_TAU: P.out[gi] = divtau(xn); break;
            case EPI_UZAWA_P: {
                const double dp = divtau(xn);
                P.out[gi] = __ldg(P.pin + gi) + dp;
                acc = bv * dp;
                break;
            }
            case EPI_DOT_TAU: acc = bv * divtau(xn); break;
            case EPI_SCALE: P.out[gi] = P.scale * xn; break;
            case EPI_SCALE_DOT: {
                const double w = P.scale * xn;
                P.out[gi] = w;
                acc = __ldg(P.aux + gi) * w;
                break;
            }
            case EPI_SCALE_DOTONLY: acc = __ldg(P.aux + gi) * (P.scale * xn); break;
        }
    }
    if (P.part) {
        const double s = block_sum<FT>(acc);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            P.part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
    }
}

// Galerkin coarse rows C = (P^T A) P of one set, in scipy's SpGEMM order
// (spatial.py:140 via csc/csr matmat):
//   B[I,k] = sum over fine l ascending of A[l,k] P[l,I]      (0 + ...)
//   C[I,J] = sum over fine k ascending of P[k,J] B[I,k]      (0 + ...)
template <int MODE>
__global__ void __launch_bounds__(FT)
    k_f_galerkin(int m, int mc, Src A, double* __restrict__ out) {
    const size_t nc = (size_t)mc * mc;
    const long long g = (long long)blockIdx.x * FT + threadIdx.x;
    if (g >= (long long)nc) return;
    const int s = blockIdx.y;
    const int g32 = (int)g;
    const int Y = g32 / mc, X = g32 - Y * mc;
    const double wt[3] = {0.5, 1.0, 0.5};
    // fine box (2X-1 .. 2X+3) x (2Y-1 .. 2Y+3)
    double B[5][5];
#pragma unroll
    for (int by = 0; by < 5; ++by)
#pragma unroll
        for (int bx = 0; bx < 5; ++bx) B[by][bx] = 0.0;
    // l = (2Y+a, 2X+q) ascending; contributes to k in its 3x3 neighbourhood.
    // For each k the l's arrive in ascending order, as in the reference.
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int ly = 2 * Y + a, lx = 2 * X + q;
            const double pl = wt[a] * wt[q];
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const int k = (dy + 1) * 3 + (dx + 1);
                    if (!structural<MODE>(k)) continue;
                    const int ky = ly + dy, kx = lx + dx;
                    if (ky < 0 || ky >= m || kx < 0 || kx >= m) continue;
                    const double alk = coef<MODE>(A, s, k, m, lx, ly);
                    B[a + dy + 1][q + dx + 1] = B[a + dy + 1][q + dx + 1] + alk * pl;
                }
        }
    double* o = out + (size_t)s * 9 * nc;
#pragma unroll
    for (int jy = -1; jy <= 1; ++jy)
#pragma unroll
        for (int jx = -1; jx <= 1; ++jx) {
            const int J = (jy + 1) * 3 + (jx + 1);
            double cv = 0.0;
            if (Y + jy >= 0 && Y + jy < mc && X + jx >= 0 && X + jx < mc) {
                // k = (2(Y+jy)+ry, 2(X+jx)+rx), ascending; box index = 2j + r + 1
#pragma unroll
                for (int ry = 0; ry < 3; ++ry)
#pragma unroll
                    for (int rx = 0; rx < 3; ++rx) {
                        const int by = 2 * jy + ry + 1, bx = 2 * jx + rx + 1;
                        if (by < 0 || by > 4 || bx < 0 || bx > 4) continue;
                        cv = cv + (wt[ry] * wt[rx]) * B[by][bx];
                    }
            }
            o[(size_t)J * nc + g] = cv;
        }
}

dim3 tile_grid(int m, int planes) {
    return dim3((m + FX - 1) / FX, (m + FY - 1) / FY, (planes + FG - 1) / FG);
}

dim3 grid2(int m, int planes) {  // 64 x 4 tiles of an m x m plane, one plane per z
    return dim3((m + GX - 1) / GX, (m + GY - 1) / GY, planes);
}

dim3 pt_grid(size_t pts, int planes) {
    return dim3((unsigned)((pts + FT - 1) / FT), (unsigned)planes);
}

bool epi_dot(int epi) {
    return epi == EPI_UZAWA_P || epi == EPI_DOT_TAU || epi == EPI_SCALE_DOT ||
           epi == EPI_SCALE_DOTONLY;
}

Src fine_src(pint_ctx* c, int which) {
    Src S;
    if (which == PINT_MG_ATILDE && c->fsep_R) {
        S.f = c->d_fsep;
        S.sc = c->d_fsc;
        S.R = c->fsep_R;
        S.term_stride = 3 * (size_t)c->n;
    } else if (which == PINT_MG_ATILDE) {
        S.f = c->d_fa;
        S.set_stride = 3 * (size_t)c->n;
    } else {
        S.f = c->d_fref;
        S.set_stride = 0;
        S.mass = c->d_mass;
        for (int k = 0; k < 9; ++k) S.massv[k] = c->h_mass[k];
        S.mu = c->fmg[which].d_mu;
        S.tau = c->tau_ref;
    }
    return S;
}

Src coarse_src(const FieldMg& F, int l) {
    Src S;
    S.f = F.f9[l];
    if (F.sep) {  // R term tables [R][9][m_l^2], weights [sets][R]
        S.sc = F.d_sc;
        S.R = F.sep;
        S.term_stride = 9 * (size_t)F.m[l] * F.m[l];
    } else {
        S.set_stride = 9 * (size_t)F.m[l] * F.m[l];
    }
    return S;
}

}  // namespace

void field_assemble(pint_ctx* c, int step0, int count, const double* w_dev, double* dst) {
    const int cells = c->m + 1;
    if (!dst) dst = c->d_fa;
    k_f_assemble<<<pt_grid((size_t)c->n, count), FT, 0, c->stream>>>(
        cells, w_dev, dst + (size_t)step0 * 3 * c->n);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_timeop_field(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                         double* out) {
    if (op == OP_K || op == OP_KT) pint_throw(PINT_INPUT, "K / K^T have no stiffness part");
    static const int kid[] = {K_TIMEOP_K, K_TIMEOP_KT, K_TIMEOP_ABD, K_TIMEOP_R1, K_TIMEOP_Z};
    static const int passes[] = {2, 2, 5, 7, 7};   // + 3 compact coefficient fields
    ProfScope prof(c, kid[op], 8.0 * passes[op] * (double)c->N * c->n);
    const Src A = fine_src(c, PINT_MG_ATILDE);
    const dim3 g = tile_grid(c->m, c->N), b(FX, FY);
    const int qmin = c->has_prev ? -1 : 0, qmax = c->has_next ? c->N : c->N - 1;
    auto run = [&](auto mode_tag) {
        constexpr int MODE = decltype(mode_tag)::value;
        switch (op) {
            case OP_ABD:
                k_f_timeop<OP_ABD, MODE><<<g, b, 0, c->stream>>>(c->m, c->N, qmin, qmax, c->d_mass, A,
                                                                 c->d_ascale, u, p, f, out);
                break;
            case OP_R1:
                k_f_timeop<OP_R1, MODE><<<g, b, 0, c->stream>>>(c->m, c->N, qmin, qmax, c->d_mass, A,
                                                                c->d_ascale, u, p, f, out);
                break;
            case OP_Z:
                k_f_timeop<OP_Z, MODE><<<g, b, 0, c->stream>>>(c->m, c->N, qmin, qmax, c->d_mass, A,
                                                               c->d_ascale, u, p, f, out);
                break;
            default: pint_throw(PINT_INPUT, "unknown time operator");
        }
    };
    if (c->fsep_R) run(std::integral_constant<int, FM_SA>{});
    else run(std::integral_constant<int, FM_A>{});
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_aref_field(pint_ctx* c, const double* in, double* out, int count) {
    if (!c->fref_ready) pint_throw(PINT_INPUT, "A_ref coefficient field not set");
    ProfScope prof(c, K_AREF, 16.0 * (double)count * c->n);
    Src A;
    A.f = c->d_fref;
    A.set_stride = 0;
    k_f_apply<FM_A><<<tile_grid(c->m, count), dim3(FX, FY), 0, c->stream>>>(c->m, count, A, in, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

// out[3][n] = sum_r sc[step][r] T_r: the compact field of one step of a
// separable family (A_ref = A_step, pint_field_aref)
__global__ void __launch_bounds__(FT)
    k_f_sep_combine(size_t cnt, Src S, int step, double* __restrict__ out) {
    const size_t g = (size_t)blockIdx.x * FT + threadIdx.x;
    if (g >= cnt) return;
    out[g] = sep_at(sep_load(S, step), S.f + g);
}

void field_sep_step(pint_ctx* c, int step, double* out) {
    const Src S = fine_src(c, PINT_MG_ATILDE);
    const size_t cnt = 3 * (size_t)c->n;
    k_f_sep_combine<<<(unsigned)((cnt + FT - 1) / FT), FT, 0, c->stream>>>(cnt, S, step, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void field_galerkin(pint_ctx* c, int which) {
    FieldMg& F = c->fmg[which];
    for (int l = 0; l + 1 < F.levels; ++l) {
        const int m = F.m[l], mc = F.m[l + 1];
        const size_t nc = (size_t)mc * mc;
        if (F.sep) {
            // Galerkin rows of every TERM (the product is linear in the operator)
            if (l == 0 && which == PINT_MG_ATILDE) {
                Src S;  // the R term fields as R plain compact sets
                S.f = c->d_fsep;
                S.set_stride = 3 * (size_t)c->n;
                k_f_galerkin<FM_A><<<pt_grid(nc, F.sep), FT, 0, c->stream>>>(m, mc, S, F.f9[1]);
            } else if (l == 0) {
                // H_k = mu_k M + tau_ref A_ref: term 0 = M (mu = 1, tau = 0), term 1 = A_ref
                Src S;
                S.f = c->d_fref;
                S.mass = c->d_mass;
                for (int k = 0; k < 9; ++k) S.massv[k] = c->h_mass[k];
                S.mu = c->d_unit;  // {1.0, 0.0}
                S.tau = 0.0;
                k_f_galerkin<FM_H><<<pt_grid(nc, 1), FT, 0, c->stream>>>(m, mc, S, F.f9[1]);
                S.mu = c->d_unit + 1;
                S.tau = 1.0;
                k_f_galerkin<FM_H><<<pt_grid(nc, 1), FT, 0, c->stream>>>(m, mc, S, F.f9[1] + 9 * nc);
            } else {
                Src S;
                S.f = F.f9[l];
                S.set_stride = 9 * (size_t)m * m;
                k_f_galerkin<FM_9><<<pt_grid(nc, F.sep), FT, 0, c->stream>>>(m, mc, S, F.f9[l + 1]);
            }
            PINT_LAUNCHED(c);
            PINT_CUDA_CHECK(cudaGetLastError());
            continue;
        }
        const dim3 g = pt_grid(nc, c->N);
        if (l == 0) {
            const Src S = fine_src(c, which);
            if (which == PINT_MG_ATILDE)
                k_f_galerkin<FM_A><<<g, FT, 0, c->stream>>>(m, mc, S, F.f9[1]);
            else
                k_f_galerkin<FM_H><<<g, FT, 0, c->stream>>>(m, mc, S, F.f9[1]);
        } else {
            k_f_galerkin<FM_9><<<g, FT, 0, c->stream>>>(m, mc, coarse_src(F, l), F.f9[l + 1]);
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
    }
}

namespace {

template <int MODE>
void pre_level(pint_ctx* c, const Src& S, int m, int mc, int count, double damping,
               const double* b, double* x0, double* bc, bool fine, double* rwork) {
    ProfScope prof(c, fine ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                   8.0 * count * (3.0 * m * m + (double)mc * mc));
    k_f_x0<MODE><<<grid2(m, count), dim3(GX, GY), 0, c->stream>>>(m, S, damping, b, x0);
    static const bool fused_rr = getenv("PINT_FIELD_RR") != nullptr;  // round-1 form (A/B)
    if (fused_rr || !rwork) {
        k_f_rr<MODE><<<grid2(mc, count), dim3(GX, GY), 0, c->stream>>>(m, mc, S, b, x0, bc);
        c->launches += 2;
        return;
    }
    k_f_resid<MODE><<<grid2(m, count), dim3(GX, GY), 0, c->stream>>>(m, S, b, x0, rwork);
    k_f_restrict<<<grid2(mc, count), dim3(GX, GY), 0, c->stream>>>(m, mc, rwork, bc);
    c->launches += 3;
}

template <int MODE>
void post_level(pint_ctx* c, const Src& S, const FieldMg& F, int l, int count, const double* b,
                double* x, double* out, int epi, double scale, const double* pin,
                const double* aux, int acc_slot) {
    const int m = F.m[l], mc = F.m[l + 1];
    const bool top = l == 0;
    const bool direct = l + 1 == F.levels - 1;
    const double* ec = direct ? c->lev_b[l + 1] : c->lev_x[l + 1];
    ProfScope prof(c, top ? K_MG_POST_FINE : K_MG_POST_COARSE,
                   8.0 * count * (4.0 * m * m + (double)mc * mc));
    const Src Ac = coarse_src(F, l + 1);
    if (direct && F.sep)
        k_f_prolong<true, FM_S9><<<grid2(m, count), dim3(GX, GY), 0, c->stream>>>(m, mc, Ac, ec, x);
    else if (direct)
        k_f_prolong<true, FM_9><<<grid2(m, count), dim3(GX, GY), 0, c->stream>>>(m, mc, Ac, ec, x);
    else
        k_f_prolong<false, FM_9><<<grid2(m, count), dim3(GX, GY), 0, c->stream>>>(m, mc, Ac, ec, x);
    FSmooth P{};
    P.m = m;
    P.b = b;
    P.x = x;
    P.out = out;
    P.epi = top ? epi : EPI_PLAIN;
    P.damping = F.damping;
    P.scale = scale;
    P.steps = c->d_steps;
    P.rsteps = c->d_rsteps;
    P.pin = pin;
    P.aux = aux;
    const dim3 g = grid2(m, count);
    const size_t nblk = (size_t)g.x * g.y * g.z;
    const bool dot = top && epi_dot(epi);
    if (dot) {
        ensure_partials(c, nblk);
        P.part = c->d_part;
    }
    k_f_smooth<MODE><<<g, dim3(GX, GY), 0, c->stream>>>(S, P);
    c->launches += 2;
    if (dot) reduce_partials(c, (int)nblk, acc_slot);
}

}  // namespace

void vcycle_field(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
                  double scale, const double* pin, const double* aux, int acc_slot) {
    FieldMg& F = c->fmg[which];
    if (!F.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    const int L = F.levels;
    const Src S0 = fine_src(c, which);
    // descend: x0 = dinv b kept per level (the prolongation adds to it)
    const double* bl = b;
    // residual work planes: the fine level borrows the 3D path's slab-sized
    // scratch, level l >= 1 its own (not yet written) solution buffer lev_x[l]
    {
        const size_t need = (size_t)count * c->n;
        if (c->t3_cap < need) {
            if (c->d_t3a) cudaFree(c->d_t3a);
            if (c->d_t3b) cudaFree(c->d_t3b);
            c->d_t3b = nullptr;
            PINT_CUDA_CHECK(cudaMalloc(&c->d_t3a, need * sizeof(double) + 16));
            PINT_CUDA_CHECK(cudaMalloc(&c->d_t3b, 16));
            c->t3_cap = need;
        }
    }
    for (int l = 0; l + 1 < L; ++l) {
        const int m = F.m[l], mc = F.m[l + 1];
        double* x0 = l == 0 ? c->d_ft : c->lev_t[l];
        double* rw = l == 0 ? c->d_t3a : c->lev_x[l];
        if (l == 0) {
            if (which == PINT_MG_ATILDE && F.sep)
                pre_level<FM_SA>(c, S0, m, mc, count, F.damping, bl, x0, c->lev_b[1], true, rw);
            else if (which == PINT_MG_ATILDE)
                pre_level<FM_A>(c, S0, m, mc, count, F.damping, bl, x0, c->lev_b[1], true, rw);
            else
                pre_level<FM_H>(c, S0, m, mc, count, F.damping, bl, x0, c->lev_b[1], true, rw);
        } else if (F.sep) {
            pre_level<FM_S9>(c, coarse_src(F, l), m, mc, count, F.damping, bl, x0, c->lev_b[l + 1],
                             false, rw);
        } else {
            pre_level<FM_9>(c, coarse_src(F, l), m, mc, count, F.damping, bl, x0, c->lev_b[l + 1],
                            false, rw);
        }
        bl = c->lev_b[l + 1];
    }
    PINT_CUDA_CHECK(cudaGetLastError());
    for (int l = L - 2; l >= 0; --l) {
        double* x = l == 0 ? c->d_ft : c->lev_t[l];
        if (l == 0) {
            if (which == PINT_MG_ATILDE && F.sep)
                post_level<FM_SA>(c, S0, F, 0, count, b, x, out, epi, scale, pin, aux, acc_slot);
            else if (which == PINT_MG_ATILDE)
                post_level<FM_A>(c, S0, F, 0, count, b, x, out, epi, scale, pin, aux, acc_slot);
            else
                post_level<FM_H>(c, S0, F, 0, count, b, x, out, epi, scale, pin, aux, acc_slot);
        } else if (F.sep) {
            post_level<FM_S9>(c, coarse_src(F, l), F, l, count, c->lev_b[l], x, c->lev_x[l],
                              EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        } else {
            post_level<FM_9>(c, coarse_src(F, l), F, l, count, c->lev_b[l], x, c->lev_x[l],
                             EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        }
    }
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
