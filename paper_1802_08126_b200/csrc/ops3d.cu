// 3D (unit cube, P1 on the Kuhn 6-tetrahedron split) versions of the
// time-global operators and the batched multigrid V-cycle: the EXTENSION that
// BASELINE configs 3 and 5 need (the reference assembles 1D/2D only,
// problems.py:78-138, spatial.py:100-113; oracle/pint_oracle.py:p1_3d).
//
// Operators are 27-point stencils in CSR column order (dz, dy, dx
// lexicographic from (-1,-1,-1)); the M (15-point) and A (7-point) patterns
// are zeros in the other positions, which add +-0 and cannot change a sum.
// Row sums follow CSR order from 0 without FMA (-fmad=false), restriction
// sums over ascending fine index, prolongation over ascending coarse index,
// so results are bit-identical to the oracle's scipy products.
//
// Three generations live here: the generic K / K^T / A_bd applies (k3_timeop,
// thread per point); the z-marching register-window kernels (kz_*: r1, z and,
// for grids the band kernels are not built for, the V-cycle phases); and the
// TMA band kernels of mg3_band_kernels.inc (kc3_*: fused V-cycle, stencil
// applies, shared-memory tail), which carry the c3 / c5 hot path.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "band.cuh"
#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

namespace {

constexpr int T3 = 256;
constexpr int G3 = 4;  // time planes per CTA in the marching operators

__device__ __forceinline__ double st27(const double* __restrict__ c, const double* __restrict__ v,
                                       int m, int x, int y, int z) {
    double s = 0.0;
    int k = 0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
        const bool iz = (unsigned)(z + dz) < (unsigned)m;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            const bool iy = iz && (unsigned)(y + dy) < (unsigned)m;
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx, ++k) {
                const bool in = iy && (unsigned)(x + dx) < (unsigned)m;
                const double val = in ? __ldg(v + ((long long)(z + dz) * m + (y + dy)) * m + (x + dx))
                                      : 0.0;
                const double t = __ldg(c + k) * val;
                s = (k == 0) ? t : s + t;
            }
        }
    }
    return s;
}

// same with every neighbour scaled by d first (x0 = dinv*b evaluated in place)
__device__ __forceinline__ double st27_scaled(const double* __restrict__ c, double d,
                                              const double* __restrict__ v, int m, int x, int y,
                                              int z) {
    double s = 0.0;
    int k = 0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
        const bool iz = (unsigned)(z + dz) < (unsigned)m;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            const bool iy = iz && (unsigned)(y + dy) < (unsigned)m;
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx, ++k) {
                const bool in = iy && (unsigned)(x + dx) < (unsigned)m;
                const double val =
                    in ? d * __ldg(v + ((long long)(z + dz) * m + (y + dy)) * m + (x + dx)) : 0.0;
                const double t = __ldg(c + k) * val;
                s = (k == 0) ? t : s + t;
            }
        }
    }
    return s;
}

struct Pt {
    int x, y, z;
    long long i;
    bool ok;
};

__device__ __forceinline__ Pt point3(int m) {
    Pt p;
    const long long g = (long long)blockIdx.x * T3 + threadIdx.x;
    const long long n = (long long)m * m * m;
    p.ok = g < n;
    p.i = g;
    const int mm = m * m;
    p.z = (int)(g / mm);
    const int r = (int)(g - (long long)p.z * mm);
    p.y = r / m;
    p.x = r - p.y * m;
    return p;
}

template <int OP>
__global__ void __launch_bounds__(T3)
    k3_timeop(int m, int N, int qmin, int qmax, const double* __restrict__ mass,
              const double* __restrict__ ast, const int* __restrict__ asid,
              const double* __restrict__ ascale, const double* __restrict__ u,
              const double* __restrict__ p, const double* __restrict__ f,
              double* __restrict__ out) {
    const Pt q = point3(m);
    if (!q.ok) return;
    const long long n = (long long)m * m * m;
    const int n0 = blockIdx.y * G3, n1 = min(N, n0 + G3);
    auto M = [&](const double* v, int t) { return st27(mass, v + (long long)t * n, m, q.x, q.y, q.z); };
    auto A = [&](const double* v, int t) {
        return __ldg(ascale + t) * st27(ast + 27 * __ldg(asid + t), v + (long long)t * n, m, q.x, q.y, q.z);
    };
    if (OP == OP_ABD) {
        for (int t = n0; t < n1; ++t) out[t * n + q.i] = A(u, t);
        return;
    }
    if (OP == OP_K || OP == OP_R1) {
        double mprev = (n0 - 1 >= qmin) ? M(u, n0 - 1) : 0.0;
        for (int t = n0; t < n1; ++t) {
            const double mcur = M(u, t);
            const double ku = (t - 1 >= qmin) ? mcur - mprev : mcur;
            if (OP == OP_K)
                out[t * n + q.i] = ku;
            else
                out[t * n + q.i] = (ku - A(p, t)) - __ldg(f + t * n + q.i);
            mprev = mcur;
        }
        return;
    }
    if (OP == OP_KT) {
        double mcur = M(u, n0);
        for (int t = n0; t < n1; ++t) {
            const double mnext = (t + 1 <= qmax) ? M(u, t + 1) : 0.0;
            out[t * n + q.i] = (t + 1 <= qmax) ? mcur - mnext : mcur;
            mcur = mnext;
        }
        return;
    }
    // OP_Z
    double muprev = (n0 - 1 >= qmin) ? M(u, n0 - 1) : 0.0;
    double mucur = M(u, n0), mpcur = M(p, n0);
    for (int t = n0; t < n1; ++t) {
        const bool hn = t + 1 <= qmax;
        const double munext = hn ? M(u, t + 1) : 0.0;
        const double mpnext = hn ? M(p, t + 1) : 0.0;
        const double ktp = hn ? mpcur - mpnext : mpcur;
        const double ku = (t - 1 >= qmin) ? mucur - muprev : mucur;
        const double ktu = hn ? mucur - munext : mucur;
        out[t * n + q.i] = (__ldg(f + t * n + q.i) - ktp) - ((ku + ktu) + A(u, t));
        muprev = mucur;
        mucur = munext;
        mpcur = mpnext;
    }
}

__global__ void __launch_bounds__(T3)
    k3_fold(int m, const double* __restrict__ steps, const double* __restrict__ mass,
            const double* __restrict__ load, const double* __restrict__ u0,
            double* __restrict__ f) {
    const Pt q = point3(m);
    if (!q.ok) return;
    const long long n = (long long)m * m * m;
    const int t = blockIdx.y;
    double v = __ldg(steps + t) * __ldg(load + t * n + q.i);
    if (t == 0) v = v + st27(mass, u0, m, q.x, q.y, q.z);
    f[t * n + q.i] = v;
}

// ---- multigrid ---------------------------------------------------------------
struct Smooth3 {
    int m;
    const double* tab;
    const int* sid;
    const double* b;
    const double* x;
    double* out;
    int epi;
    double scale;
    const double* steps;
    const double* rsteps;
    const double* pin;
    const double* aux;
    double* part;
};

// ---------------------------------------------------------------------------
// z-marching stencil engine (round-1 rewrite of the thread-per-point form).
// A thread owns one (x, y) column of a 32 x 8 tile and a chunk of ZC
// consecutive z; it keeps a 3-slice register window of the (dy, dx)
// positions its stencil pattern touches, so every input value is loaded once
// per thread instead of once per stencil term (7 loads per point for the
// 15-point mass, 5 for the 7-point stiffness, 9 for Galerkin 27-point
// operators).  Coefficients of the plane's operator are per-CTA registers.
// The row sum runs over the pattern in CSR order (dz, dy, dx lexicographic)
// with no FMA (-fmad=false); positions outside the pattern are exact zeros
// in every table (checked on the host), so skipping them changes no value.
// ---------------------------------------------------------------------------
constexpr int ZX = 32, ZY = 8, ZC = 8;

// x / y out of line: a select between v * (1/tau) and v / tau would otherwise
// be if-converted and the (slow-path-prone) division evaluated for every point
__device__ __noinline__ double div_rn(double x, double y) { return x / y; }

// stencil patterns: bit k = (dz+1)*9 + (dy+1)*3 + (dx+1)
constexpr uint32_t PAT_A7 = (1u << 4) | (1u << 10) | (1u << 12) | (1u << 13) | (1u << 14) |
                            (1u << 16) | (1u << 22);
// P1 mass on the Kuhn split: 0, +-x, +-y, +-z, +-(1,1,0), +-(0,1,1), +-(1,0,1), +-(1,1,1)
constexpr uint32_t PAT_M15 = PAT_A7 | (1u << 0) | (1u << 26) | (1u << 9) | (1u << 17) |
                             (1u << 1) | (1u << 25) | (1u << 3) | (1u << 23);
constexpr uint32_t PAT_F27 = (1u << 27) - 1;

__host__ __device__ constexpr bool pat_has(uint32_t pat, int k) { return (pat >> k) & 1u; }
// (dy, dx) position q = (dy+1)*3 + (dx+1) needed in any z role
__host__ __device__ constexpr bool pat_need(uint32_t pat, int q) {
    return pat_has(pat, q) || pat_has(pat, 9 + q) || pat_has(pat, 18 + q);
}

uint32_t pattern_of(const double* st, int count) {
    uint32_t mask = 0;
    for (int s = 0; s < count; ++s)
        for (int k = 0; k < 27; ++k)
            if (st[(size_t)s * 27 + k] != 0.0) mask |= 1u << k;
    return mask;
}
// smallest compiled pattern containing mask
uint32_t pattern_pick(uint32_t mask) {
    if ((mask & ~PAT_A7) == 0) return PAT_A7;
    if ((mask & ~PAT_M15) == 0) return PAT_M15;
    return PAT_F27;
}

struct ZTile {
    int x, y, z0, zn;  // column and z range [z0, z0 + zn)
    bool ok;
};

// blockIdx.x enumerates (tile, z chunk) of a plane; blockIdx.y the plane
__device__ __forceinline__ ZTile ztile(int m) {
    const int tx = (m + ZX - 1) / ZX, ty = (m + ZY - 1) / ZY;
    int b = blockIdx.x;
    const int xt = b % tx;
    b /= tx;
    const int yt = b % ty;
    const int zc = b / ty;
    ZTile t;
    t.x = xt * ZX + (int)threadIdx.x;
    t.y = yt * ZY + (int)threadIdx.y;
    t.z0 = zc * ZC;
    t.zn = min(ZC, m - t.z0);
    t.ok = t.x < m && t.y < m;
    return t;
}
inline dim3 zgrid(int m, int planes) {
    const int tx = (m + ZX - 1) / ZX, ty = (m + ZY - 1) / ZY, tz = (m + ZC - 1) / ZC;
    return dim3((unsigned)(tx * ty * tz), (unsigned)planes);
}

// per-thread neighbourhood of a column: in-domain flags of x-1, x+1, y-1, y+1
struct ZNbr {
    bool xl, xr, yl, yr;
};
__device__ __forceinline__ ZNbr znbr(int m, int x, int y) {
    ZNbr b;
    b.xl = x > 0;
    b.xr = x + 1 < m;
    b.yl = y > 0;
    b.yr = y + 1 < m;
    return b;
}
__device__ __forceinline__ bool znbr_in(const ZNbr& b, int q) {
    const int dy = q / 3 - 1, dx = q % 3 - 1;
    return (dy < 0 ? b.yl : dy > 0 ? b.yr : true) && (dx < 0 ? b.xl : dx > 0 ? b.xr : true);
}

// the needed (dy, dx) values of the slice whose column element is v[i]
// (zero outside the domain or when !zin), times d when SCALED.  32-bit
// element indices into one plane: a row is one base address, the x
// neighbours are immediate offsets of it.
template <uint32_t PAT, bool SCALED>
__device__ __forceinline__ void zslice(double* w, const double* __restrict__ v, int i, int m,
                                       bool zin, const ZNbr& nb, double d) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        const double* r = v + (i + dy * m);
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const int q = (dy + 1) * 3 + (dx + 1);
            if (!pat_need(PAT, q)) continue;
            const bool in = zin && znbr_in(nb, q);
            const double val = in ? __ldg(r + dx) : 0.0;
            w[q] = SCALED ? (in ? d * val : 0.0) : val;
        }
    }
}

// row sum over the pattern in CSR order; c[k] coefficient registers
template <uint32_t PAT>
__device__ __forceinline__ double zsum(const double* c, const double (&w)[3][9]) {
    double s = 0.0;
    bool first = true;
#pragma unroll
    for (int k = 0; k < 27; ++k) {
        if (!pat_has(PAT, k)) continue;
        const double t = c[k] * w[k / 9][k % 9];
        s = first ? t : s + t;
        first = false;
    }
    return s;
}

template <uint32_t PAT>
__device__ __forceinline__ void zcoef(double* c, const double* __restrict__ tb) {
#pragma unroll
    for (int k = 0; k < 27; ++k) c[k] = pat_has(PAT, k) ? __ldg(tb + k) : 0.0;
}

// march z over the chunk: f(z, li, sum, centre value) for every point of the
// column, li = its element index inside the plane
template <uint32_t PAT, bool SCALED, typename F>
__device__ __forceinline__ void zmarch(const ZTile& t, int m, const double* __restrict__ v,
                                       const double* c, double d, F&& f) {
    const ZNbr nb = znbr(m, t.x, t.y);
    const int S = m * m;
    int i = (t.z0 - 1) * S + t.y * m + t.x;  // may be negative for z0 = 0 (not loaded)
    double w[3][9];
    zslice<PAT, SCALED>(w[0], v, i, m, t.z0 >= 1, nb, d);
    zslice<PAT, SCALED>(w[1], v, i + S, m, true, nb, d);
    i += 2 * S;
    // no early exit: slices past the chunk end load as zeros and their results
    // are dropped, so the unrolled loop has no data-dependent branch
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
        zslice<PAT, SCALED>(w[2], v, i, m, t.z0 + k + 1 < m, nb, d);
        if (k < t.zn) f(t.z0 + k, i - S, zsum<PAT>(c, w), w[1][4]);
        i += S;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            w[0][q] = w[1][q];
            w[1][q] = w[2][q];
        }
    }
}

// zmarch with one-point-ahead prefetch: the window slice of z+2 and the
// point values pre(li, valid) of the next point are loaded before the
// current point is computed, so every thread keeps two iterations of loads
// in flight (the smoother / residual kernels are latency bound otherwise).
// post(li, sum, centre, pv) consumes the point values pre returned.
template <uint32_t PAT, bool SCALED, typename Pre, typename Post>
__device__ __forceinline__ void zmarch_pf(const ZTile& t, int m, const double* __restrict__ v,
                                          const double* c, double d, Pre&& pre, Post&& post) {
    const ZNbr nb = znbr(m, t.x, t.y);
    const int S = m * m;
    const int i0 = t.z0 * S + t.y * m + t.x;  // element index of the chunk's first point
    double w[3][9];
    zslice<PAT, SCALED>(w[0], v, i0 - S, m, t.z0 >= 1, nb, d);
    zslice<PAT, SCALED>(w[1], v, i0, m, true, nb, d);
    zslice<PAT, SCALED>(w[2], v, i0 + S, m, t.z0 + 1 < m, nb, d);
    auto pv = pre(i0, true);
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
        double wn[9];
        decltype(pv) pn = pv;
        if (k + 1 < ZC) {
            zslice<PAT, SCALED>(wn, v, i0 + (k + 2) * S, m, t.z0 + k + 2 < m, nb, d);
            pn = pre(i0 + (k + 1) * S, k + 1 < t.zn);
        }
        if (k < t.zn) post(i0 + k * S, zsum<PAT>(c, w), w[1][4], pv);
        if (k + 1 < ZC) {
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                w[0][q] = w[1][q];
                w[1][q] = w[2][q];
                w[2][q] = wn[q];
            }
            pv = pn;
        }
    }
}

// out[t] = scale_t * S_t in[t] for planes t in [t0, t0 + gridDim.y) (t0 may be -1:
// ghost planes); table row per plane: tab + 27 * (sid ? sid[t] : 0)
template <uint32_t PAT>
__global__ void __launch_bounds__(ZX * ZY)
    kz_apply(int m, int t0, const double* __restrict__ tab, int tstride,
             const int* __restrict__ sid, const double* __restrict__ scale,
             const double* __restrict__ in, double* __restrict__ out) {
    const ZTile t = ztile(m);
    if (!t.ok) return;
    const long long n = (long long)m * m * m;
    const int pl = t0 + (int)blockIdx.y;
    const double* tb = tab + (size_t)tstride * (sid ? __ldg(sid + pl) : 0);
    double c[27];
    zcoef<PAT>(c, tb);
    const double sc = scale ? __ldg(scale + pl) : 1.0;
    const double* v = in + pl * n;
    double* o = out + pl * n;
    // 7-point operators (A_ref y1): window slices requested one point ahead
    // (zmarch_pf), 0.59 -> 0.53 ms on c3; the 15-point mass is slower that way
    // (78 registers: r1 1.51 -> 1.58 ms, z 1.74 -> 1.82 ms)
    if constexpr (PAT != PAT_A7) {
        zmarch<PAT, false>(t, m, v, c, 1.0, [&](int, int li, double s, double) {
            o[li] = scale ? sc * s : s;
        });
    } else {
        zmarch_pf<PAT, false>(
            t, m, v, c, 1.0, [&](int, bool) { return 0; },
            [&](int li, double s, double, int) { o[li] = scale ? sc * s : s; });
    }
}

// r1 = ((Mu_t - Mu_{t-1}) - s_t A p_t) - f_t   (OP_R1 of k3_timeop, Mu precomputed)
template <uint32_t PAT>
__global__ void __launch_bounds__(ZX * ZY)
    kz_r1(int m, int qmin, const double* __restrict__ ast, const int* __restrict__ asid,
          const double* __restrict__ ascale, const double* __restrict__ mu,
          const double* __restrict__ p, const double* __restrict__ f, double* __restrict__ out) {
    const ZTile t = ztile(m);
    if (!t.ok) return;
    const long long n = (long long)m * m * m;
    const int pl = (int)blockIdx.y;
    double c[27];
    zcoef<PAT>(c, ast + 27 * __ldg(asid + pl));
    const double sc = __ldg(ascale + pl);
    const long long col = (long long)t.y * m + t.x;
    const bool hp = pl - 1 >= qmin;
    const double* mup = mu + pl * n;
    const double* fp = f + pl * n;
    zmarch_pf<PAT, false>(
        t, m, p + pl * n, c, 1.0,
        [&](int li, bool ok) {
            double3 r;
            r.x = ok ? __ldg(mup + li) : 0.0;
            r.y = ok && hp ? __ldg(mup + li - n) : 0.0;
            r.z = ok ? __ldg(fp + li) : 0.0;
            return r;
        },
        [&](int li, double s, double, double3 pv) {
            const double ku = hp ? pv.x - pv.y : pv.x;
            out[pl * n + li] = (ku - sc * s) - pv.z;
        });
}

// z = (f - K^T p) - ((K u + K^T u) + s_t A u_t)   (OP_Z of k3_timeop, Mu/Mp precomputed)
template <uint32_t PAT>
__global__ void __launch_bounds__(ZX * ZY)
    kz_z(int m, int qmin, int qmax, const double* __restrict__ ast, const int* __restrict__ asid,
         const double* __restrict__ ascale, const double* __restrict__ mu,
         const double* __restrict__ mp, const double* __restrict__ u, const double* __restrict__ f,
         double* __restrict__ out) {
    const ZTile t = ztile(m);
    if (!t.ok) return;
    const long long n = (long long)m * m * m;
    const int pl = (int)blockIdx.y;
    double c[27];
    zcoef<PAT>(c, ast + 27 * __ldg(asid + pl));
    const double sc = __ldg(ascale + pl);
    const long long col = (long long)t.y * m + t.x;
    const bool hp = pl - 1 >= qmin, hn = pl + 1 <= qmax;
    // the six point operands of the next z are requested one point ahead
    // (zmarch_pf), like kz_r1: the kernel is latency bound otherwise
    struct Pv {
        double mp, mpn, mu, mup, mun, f;
    };
    zmarch_pf<PAT, false>(
        t, m, u + pl * n, c, 1.0,
        [&](int li, bool ok) {
            const long long gi = pl * n + li;
            Pv r;
            r.mp = ok ? __ldg(mp + gi) : 0.0;
            r.mu = ok ? __ldg(mu + gi) : 0.0;
            r.mpn = ok && hn ? __ldg(mp + gi + n) : 0.0;
            r.mun = ok && hn ? __ldg(mu + gi + n) : 0.0;
            r.mup = ok && hp ? __ldg(mu + gi - n) : 0.0;
            r.f = ok ? __ldg(f + gi) : 0.0;
            return r;
        },
        [&](int li, double s, double, Pv pv) {
            const double ktp = hn ? pv.mp - pv.mpn : pv.mp;
            const double ku = hp ? pv.mu - pv.mup : pv.mu;
            const double ktu = hn ? pv.mu - pv.mun : pv.mu;
            out[pl * n + li] = (pv.f - ktp) - ((ku + ktu) + sc * s);
        });
}

// r = b - S(dinv * b)   (spatial.py:153,156)
template <uint32_t PAT>
__global__ void __launch_bounds__(ZX * ZY)
    kz_residual(int m, const double* __restrict__ tab, const int* __restrict__ sid,
                const double* __restrict__ b, double* __restrict__ r) {
    const ZTile t = ztile(m);
    if (!t.ok) return;
    const long long n = (long long)m * m * m;
    const int pl = (int)blockIdx.y;
    const double* tb = tab + (size_t)__ldg(sid + pl) * 28;
    double c[27];
    zcoef<PAT>(c, tb);
    const double d = __ldg(tb + 27);
    const double* bp = b + pl * n;
    const long long col = (long long)t.y * m + t.x;
    zmarch<PAT, true>(t, m, bp, c, d, [&](int, int li, double s, double) {
        r[pl * n + li] = __ldg(bp + li) - s;
    });
}

// x += dinv*(b - S x) (spatial.py:159-160) + the finest-level epilogues
template <uint32_t PAT>
__global__ void __launch_bounds__(ZX * ZY, 3) kz_smooth(Smooth3 a) {
    const ZTile t = ztile(a.m);
    const int m = a.m;
    const long long n = (long long)m * m * m;
    const int pl = (int)blockIdx.y;
    double acc = 0.0;
    // the plane's stencil in shared memory (broadcast reads) instead of 2 x 15..27
    // registers: the smoother is latency bound, registers buy resident warps
    __shared__ double cs[27];
    {
        const double* tb = a.tab + (size_t)__ldg(a.sid + pl) * 28;
        const int q = threadIdx.y * ZX + threadIdx.x;
        if (q < 27) cs[q] = pat_has(PAT, q) ? __ldg(tb + q) : 0.0;
        __syncthreads();
    }
    if (t.ok) {
        const double* tb = a.tab + (size_t)__ldg(a.sid + pl) * 28;
        const double* c = cs;
        const double d = __ldg(tb + 27);
        const long long col = (long long)t.y * m + t.x;
        const double* xp = a.x + pl * n;
        const double rtau = __ldg(a.rsteps + pl), tau = __ldg(a.steps + pl);
        auto divtau = [&](double v) { return rtau > 0.0 ? v * rtau : div_rn(v, tau); };
        const double* bpl = a.b + pl * n;
        const double* epl = a.epi == EPI_UZAWA_P ? a.pin + pl * n
                            : (a.epi == EPI_SCALE_DOT || a.epi == EPI_SCALE_DOTONLY) ? a.aux + pl * n
                                                                                      : nullptr;
        auto pre = [&](int li, bool ok) {
            double2 r;
            r.x = ok ? __ldg(bpl + li) : 0.0;
            r.y = ok && epl ? __ldg(epl + li) : 0.0;
            return r;
        };
        auto post = [&](int li, double s, double xv, double2 pv) {
            const long long gi = pl * n + li;
            const double bv = pv.x;
            const double xn = xv + d * (bv - s);
            switch (a.epi) {
                case EPI_PLAIN: a.out[gi] = xn; break;
                case EPI_DIV_TAU: a.out[gi] = divtau(xn); break;
                case EPI_UZAWA_P: {
                    const double dp = divtau(xn);
                    a.out[gi] = pv.y + dp;
                    acc = acc + bv * dp;
                    break;
                }
                case EPI_DOT_TAU: acc = acc + bv * divtau(xn); break;
                case EPI_SCALE: a.out[gi] = a.scale * xn; break;
                case EPI_SCALE_DOT: {
                    const double w = a.scale * xn;
                    a.out[gi] = w;
                    acc = acc + pv.y * w;
                    break;
                }
                case EPI_SCALE_DOTONLY: acc = acc + pv.y * (a.scale * xn); break;
            }
        };
        if constexpr (PAT == PAT_F27) {
            // coarse levels: no prefetch (register budget of the 27-point window)
            zmarch<PAT, false>(t, m, xp, c, 1.0, [&](int, int li, double s, double xv) {
                post(li, s, xv, pre(li, true));
            });
        } else {
            zmarch_pf<PAT, false>(t, m, xp, c, 1.0, pre, post);
        }
    }
    if (a.part) {
        const double s = block_sum<ZX * ZY>(acc);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.part[(long long)blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

// x = dinv*b + P e  (csr_matvec of the trilinear P over ascending coarse
// index, spatial.py:149-150,157; e = b_c / a_c on a 1x1x1 coarsest grid).
// z-marching: the (y, x) interpolation terms of a column are fixed, and each
// coarse plane's <= 4 values serve the three fine planes 2k, 2k+1, 2k+2.
template <bool DIRECT>
__global__ void __launch_bounds__(ZX * ZY)
    kz_prolong(int m, int mc, const double* __restrict__ tab, const double* __restrict__ tabc,
               const int* __restrict__ sid, const double* __restrict__ b,
               const double* __restrict__ ec, double* __restrict__ x) {
    constexpr bool direct = DIRECT;
    const ZTile t = ztile(m);
    if (!t.ok) return;
    const long long n = (long long)m * m * m, nc = (long long)mc * mc * mc;
    const int pl = (int)blockIdx.y;
    const int set = __ldg(sid + pl);
    const double d = __ldg(tab + (size_t)set * 28 + 27);
    const double ac = direct ? __ldg(tabc + (size_t)set * 28 + 13) : 1.0;
    // interpolation terms of one coordinate f: odd -> coarse (f-1)/2, weight 1;
    // even -> f/2-1 (if >= 0) then f/2 (if < mc), weights 1/2 (pro_terms order)
    auto terms = [&](int f, int& j0, int& j1, double& w, bool& h0, bool& h1) {
        if (f & 1) {
            j0 = (f - 1) >> 1;
            j1 = j0;
            w = 1.0;
            h0 = true;
            h1 = false;
        } else {
            j0 = (f >> 1) - 1;
            j1 = f >> 1;
            w = 0.5;
            h0 = j0 >= 0;
            h1 = j1 < mc;
        }
    };
    int y0, y1, x0, x1;
    double wyv, wxv;
    bool hy0, hy1, hx0, hx1;
    terms(t.y, y0, y1, wyv, hy0, hy1);
    terms(t.x, x0, x1, wxv, hx0, hx1);
    const double* ep = ec + pl * nc;
    // coarse plane k at the column's (y, x) combinations (zero outside)
    auto load = [&](int k, double (&g)[2][2]) {
        const bool kin = k >= 0 && k < mc;
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const bool in = kin && (bb ? hy1 : hy0) && (cc ? hx1 : hx0);
                double e = in ? __ldg(ep + ((long long)k * mc + (bb ? y1 : y0)) * mc + (cc ? x1 : x0))
                              : 0.0;
                if (direct) e = e / ac;
                g[bb][cc] = e;
            }
    };
    auto accum = [&](double wz, const double (&g)[2][2], double& pe, bool& first) {
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                if (!(bb ? hy1 : hy0) || !(cc ? hx1 : hx0)) continue;
                const double tterm = ((wz * wyv) * wxv) * g[bb][cc];
                pe = first ? tterm : pe + tterm;
                first = false;
            }
    };
    const long long col = (long long)t.y * m + t.x;
    const int k0 = t.z0 >> 1;  // z0 is even
    // the chunk's ZC values of b are requested up front (one exposed latency)
    double bv[ZC];
    {
        const double* bp = b + pl * n + (long long)t.z0 * m * m + col;
#pragma unroll
        for (int i = 0; i < ZC; ++i) bv[i] = i < t.zn ? __ldg(bp + (long long)i * m * m) : 0.0;
    }
    double gp[2][2], gc[2][2];
    load(k0 - 1, gp);
    load(k0, gc);
#pragma unroll
    for (int i = 0; i < ZC; i += 2) {
        if (i >= t.zn) break;
        const int k = k0 + i / 2;
        {   // even fine plane z = 2k: coarse k-1 (if any) then k (if any), weights 1/2
            double pe = 0.0;
            bool first = true;
            if (k - 1 >= 0) accum(0.5, gp, pe, first);
            if (k < mc) accum(0.5, gc, pe, first);
            const long long gi = pl * n + (long long)(2 * k) * m * m + col;
            x[gi] = d * bv[i] + pe;
        }
        if (i + 1 < t.zn) {  // odd fine plane 2k+1: coarse k, weight 1
            double pe = 0.0;
            bool first = true;
            accum(1.0, gc, pe, first);
            const long long gi = pl * n + (long long)(2 * k + 1) * m * m + col;
            x[gi] = d * bv[i + 1] + pe;
        }
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) gp[bb][cc] = gc[bb][cc];
        load(k + 1, gc);
    }
}

// b_c = P^T r: for coarse (Z, Y, X) the 27 fine nodes (2Z+a, 2Y+bb, 2X+cc) in
// ascending fine index, weights (wa*wb)*wc with w = (0.5, 1, 0.5) (kron of
// spatial.py:75-84, same order as the oracle).  z-marching over coarse Z:
// fine plane 2Z+2 is plane 2(Z+1) of the next coarse point.
__global__ void __launch_bounds__(ZX * ZY)
    kz_restrict(int m, int mc, const double* __restrict__ r, double* __restrict__ bc) {
    const ZTile t = ztile(mc);
    if (!t.ok) return;
    const long long n = (long long)m * m * m, nc = (long long)mc * mc * mc;
    const int pl = (int)blockIdx.y;
    const double* rp = r + pl * n;
    const double w[3] = {0.5, 1.0, 0.5};
    auto load = [&](int fz, double (&g)[9]) {
#pragma unroll
        for (int q = 0; q < 9; ++q)
            g[q] = __ldg(rp + ((long long)fz * m + (2 * t.y + q / 3)) * m + (2 * t.x + q % 3));
    };
    double g0[9], g1[9], g2[9];
    load(2 * t.z0, g0);
    const long long col = (long long)t.y * mc + t.x;
#pragma unroll
    for (int i = 0; i < ZC; ++i) {
        if (i >= t.zn) break;
        const int Z = t.z0 + i;
        load(2 * Z + 1, g1);
        load(2 * Z + 2, g2);
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 27; ++k) {
            const int a = k / 9, q = k % 9;
            const double v = a == 0 ? g0[q] : a == 1 ? g1[q] : g2[q];
            const double tterm = ((w[a] * w[q / 3]) * w[q % 3]) * v;
            s = k == 0 ? tterm : s + tterm;
        }
        bc[pl * nc + (long long)Z * mc * mc + col] = s;
#pragma unroll
        for (int q = 0; q < 9; ++q) g0[q] = g2[q];
    }
}

constexpr size_t smem_cap3 = 220 * 1024;
#include "mg3_band_kernels.inc"

// run f(std::integral_constant<uint32_t, PAT>) for the smallest compiled pattern covering mask
template <typename F>
void zdispatch(uint32_t mask, F&& f) {
    switch (pattern_pick(mask)) {
        case PAT_A7: f(std::integral_constant<uint32_t, PAT_A7>{}); break;
        case PAT_M15: f(std::integral_constant<uint32_t, PAT_M15>{}); break;
        default: f(std::integral_constant<uint32_t, PAT_F27>{}); break;
    }
}

dim3 grid3(int m, int planes) {
    const long long n = (long long)m * m * m;
    return dim3((unsigned)((n + T3 - 1) / T3), (unsigned)planes);
}

bool epi_dot(int epi) {
    return epi == EPI_UZAWA_P || epi == EPI_DOT_TAU || epi == EPI_SCALE_DOT ||
           epi == EPI_SCALE_DOTONLY;
}

}  // namespace

// M applied to every plane of [qmin, qmax] of src into dst (same plane indexing)
// dst_t = S src_t for planes t0 .. t0 + count - 1 with one shared stencil: the TMA
// band kernel on the 63^3 grid, the z-marching kernel elsewhere (and PINT_3D_OLD)
static void apply_shared3(pint_ctx* c, uint32_t pattern, const double* st, int t0, int count,
                          const double* src, double* dst) {
    static const bool old_path = getenv("PINT_3D_OLD") != nullptr;
    static const int zc = getenv("PINT_3D_APPLY_ZC") ? atoi(getenv("PINT_3D_APPLY_ZC")) : 32;
    if (c->m == A3_M && !old_path) {
        Apply3 P{};
        P.tab = st;
        P.in = src;
        P.out = dst;
        P.t0 = t0;
        P.zc = std::max(1, std::min(zc, A3_M));
        const dim3 g((unsigned)(A3_NRB * ((A3_M + P.zc - 1) / P.zc)), (unsigned)count);
        const size_t smem = sizeof(double) * (size_t)(A3_NS + 1) * A3_SW;
        zdispatch(pattern, [&](auto PT) {
            auto kern = kc3_apply<decltype(PT)::value>;
            static bool attr = false;  // one per pattern instantiation
            if (!attr) {
                PINT_CUDA_CHECK(cudaFuncSetAttribute(
                    kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap3));
                attr = true;
            }
            kern<<<g, C3T, smem, c->stream>>>(P);
        });
        return;
    }
    zdispatch(pattern, [&](auto P) {
        kz_apply<decltype(P)::value><<<zgrid(c->m, count), dim3(ZX, ZY), 0, c->stream>>>(
            c->m, t0, st, 0, nullptr, nullptr, src, dst);
    });
}

static void mass_planes3(pint_ctx* c, const double* src, double* dst, int qmin, int qmax) {
    apply_shared3(c, pattern_of(c->h_mass.data(), 1), c->d_mass, qmin, qmax - qmin + 1, src, dst);
    PINT_LAUNCHED(c);
}

static double* mass_buffer3(pint_ctx* c, double*& buf) {
    // planes -1 .. N (ghost planes of a time partition); returns plane 0
    if (!buf) {
        PINT_CUDA_CHECK(cudaMalloc(&buf, (size_t)(c->N + 2) * c->n * sizeof(double) + 16));
        c->mu3_src = nullptr;
    }
    return buf + c->n;
}

void launch_timeop3(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                    double* out) {
    const dim3 g((unsigned)(((long long)c->n + T3 - 1) / T3), (unsigned)((c->N + G3 - 1) / G3));
    const int qmin = c->has_prev ? -1 : 0, qmax = c->has_next ? c->N : c->N - 1;
    if (op == OP_R1 || op == OP_Z) {
        // z-marching path: M u (and M p) of every plane first, then one fused
        // pass with the stiffness stencil (same arithmetic as k3_timeop)
        const uint32_t pa = pattern_of(c->h_ast.data(), c->n_a);
        double* mu = mass_buffer3(c, c->d_mu3);
        const int kid = op == OP_R1 ? K_TIMEOP_R1 : K_TIMEOP_Z;
        ProfScope prof(c, kid, 8.0 * (op == OP_R1 ? 6 : 9) * (double)c->N * c->n);
        if (op == OP_R1 || !(c->mu3_trust && c->mu3_src == u)) {
            mass_planes3(c, u, mu, qmin, qmax);
            c->mu3_src = u;
        }
        if (op == OP_R1) {
            zdispatch(pa, [&](auto P) {
                kz_r1<decltype(P)::value><<<zgrid(c->m, c->N), dim3(ZX, ZY), 0, c->stream>>>(
                    c->m, qmin, c->d_ast, c->d_asid, c->d_ascale, mu, p, f, out);
            });
        } else {
            double* mp = mass_buffer3(c, c->d_mp3);
            mass_planes3(c, p, mp, 0, qmax);
            zdispatch(pa, [&](auto P) {
                kz_z<decltype(P)::value><<<zgrid(c->m, c->N), dim3(ZX, ZY), 0, c->stream>>>(
                    c->m, qmin, qmax, c->d_ast, c->d_asid, c->d_ascale, mu, mp, u, f, out);
            });
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        return;
    }
    static const int passes[] = {2, 2, 2, 4, 4};
    static const int kid[] = {K_TIMEOP_K, K_TIMEOP_KT, K_TIMEOP_ABD, K_TIMEOP_R1, K_TIMEOP_Z};
    ProfScope prof(c, kid[op], 8.0 * passes[op] * (double)c->N * c->n);
#define PINT_OP3(OPV)                                                                          \
    case OPV:                                                                                  \
        k3_timeop<OPV><<<g, T3, 0, c->stream>>>(c->m, c->N, qmin, qmax, c->d_mass, c->d_ast, \
                                                c->d_asid, c->d_ascale, u, p, f, out);       \
        break;
    switch (op) {
        PINT_OP3(OP_K)
        PINT_OP3(OP_KT)
        PINT_OP3(OP_ABD)
        PINT_OP3(OP_R1)
        PINT_OP3(OP_Z)
        default: pint_throw(PINT_INPUT, "unknown time operator");
    }
#undef PINT_OP3
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_apply3(pint_ctx* c, const double* st, const double* in, double* out, int count) {
    ProfScope prof(c, K_AREF, 16.0 * (double)count * c->n);
    const uint32_t pm = st == c->d_aref ? pattern_of(c->h_aref.data(), 1) : PAT_F27;
    apply_shared3(c, pm, st, 0, count, in, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_fold3(pint_ctx* c, const double* load, const double* u0, double* f) {
    ProfScope prof(c, K_FOLD, 16.0 * (double)c->N * c->n);
    k3_fold<<<grid3(c->m, c->N), T3, 0, c->stream>>>(c->m, c->d_steps, c->d_mass, load, u0, f);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

// fused band V-cycle (kc3_pre / kc3_post): 2 launches per level
static int band3_lp(int m) {  // log2(m + 1) for the level sizes the band kernels are built for
    for (int lp = 2; lp <= 6; ++lp)
        if (m == (1 << lp) - 1) return lp;
    return 0;
}
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e && *e ? atoi(e) : dflt;
}

template <auto Kern>
static void launch_c3(dim3 g, size_t smem, cudaStream_t st, const Band3& P) {
    static bool attr = false;  // one per kernel (Kern is a template value)
    if (!attr) {
        PINT_CUDA_CHECK(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_cap3));
        attr = true;
    }
    Kern<<<g, C3T, smem, st>>>(P);
}

// levels below 63^3 run the 27-point code whatever their pattern (zeros in the table)
template <bool PRE>
static void dispatch_c3(uint32_t shape, int lp, int units_z, int count, bool has_q,
                        cudaStream_t st, const Band3& P, dim3* grid_out) {
    auto go = [&](auto PT, auto LPV) {
        constexpr uint32_t PAT = decltype(PT)::value;
        constexpr int LP = decltype(LPV)::value;
        using G = C3Geom<LP>;
        const dim3 g((unsigned)((PRE ? G::NRB_PRE : G::NRB) * units_z), (unsigned)count);
        if (grid_out) *grid_out = g;
        if constexpr (PRE)
            launch_c3<kc3_pre<PAT, LP>>(g, G::smem_pre(), st, P);
        else
            launch_c3<kc3_post<PAT, LP>>(g, G::smem_post(has_q), st, P);
    };
    using F27 = std::integral_constant<uint32_t, PAT_F27>;
    switch (lp) {
        case 6: zdispatch(shape, [&](auto PT) { go(PT, std::integral_constant<int, 6>{}); }); break;
        case 5: go(F27{}, std::integral_constant<int, 5>{}); break;
        case 4: go(F27{}, std::integral_constant<int, 4>{}); break;
        case 3: go(F27{}, std::integral_constant<int, 3>{}); break;
        case 2: go(F27{}, std::integral_constant<int, 2>{}); break;
        default: pint_throw(PINT_INPUT, "3D band kernels: unsupported level size");
    }
}

static void vcycle3_band(pint_ctx* c, MgSet& s, int count, const double* b, double* out, int epi,
                         double scale, const double* pin, const double* aux, int acc_slot) {
    const int L = s.levels;
    auto tab = [&](int l) { return s.tab + (size_t)l * s.n_sets * 28; };
    // z chunks per unit (A/B on c3, profiles/r2_c3_zc_sweep.txt): 32 fine slices
    // (post) and 16 coarse slices (pre) halve the last-wave tail of whole columns
    static const int zc_post = env_int("PINT_3D_POST_ZC", 32), zc_pre = env_int("PINT_3D_PRE_ZC", 16);
    // levels lt .. L-1 (m <= 15, below the finest) run in the shared-memory tail
    static const bool no_tail = getenv("PINT_3D_NO_TAIL") != nullptr;
    int lt = 1;
    while (lt < L && s.m[lt] > T3_MAXM) ++lt;
    const bool tail = !no_tail && lt <= L - 2 && L - lt <= T3_MAXLEV;
    const int ldown = tail ? lt : L - 1;  // band kernels serve levels 0 .. ldown - 1
    const double* bl = b;
    for (int l = 0; l < ldown; ++l) {
        const int m = s.m[l], mc = s.m[l + 1];
        Band3 P{};
        P.tab = tab(l);
        P.sid = s.sid;
        P.b = bl;
        P.out = c->lev_b[l + 1];
        P.zc = zc_pre > 0 ? std::min(zc_pre, mc) : mc;
        ProfScope prof(c, l == 0 ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                       8.0 * count * ((double)m * m * m + (double)mc * mc * mc));
        dispatch_c3<true>(s.shape3[l], band3_lp(m), (mc + P.zc - 1) / P.zc, count, false,
                          c->stream, P, nullptr);
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        bl = c->lev_b[l + 1];
    }
    if (tail) {
        Tail3 T{};
        T.nlev = L - lt;
        size_t words = 0;
        for (int j = 0; j < T.nlev; ++j) {
            T.m[j] = s.m[lt + j];
            T.tab[j] = tab(lt + j);
            const size_t n3 = (size_t)T.m[j] * T.m[j] * T.m[j];
            words += 2 * ((n3 + 1) & ~(size_t)1);
        }
        words += (size_t)T.m[0] * T.m[0] * T.m[0] + 2;
        T.sid = s.sid;
        T.b = c->lev_b[lt];
        T.x = c->lev_x[lt];
        static bool attr = false;
        if (!attr) {
            PINT_CUDA_CHECK(cudaFuncSetAttribute(kc3_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem_cap3));
            attr = true;
        }
        ProfScope prof(c, K_MG_TAIL, 16.0 * count * (double)T.m[0] * T.m[0] * T.m[0]);
        kc3_tail<<<count, C3T, words * sizeof(double), c->stream>>>(T);
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
    }
    for (int l = ldown - 1; l >= 0; --l) {
        const bool top = l == 0;
        const bool direct = l + 1 == L - 1;
        const int m = s.m[l], mc = s.m[l + 1];
        Band3 P{};
        P.tab = tab(l);
        P.tabc = direct ? tab(l + 1) : nullptr;
        P.sid = s.sid;
        P.b = top ? b : c->lev_b[l];
        P.ec = direct ? c->lev_b[l + 1] : c->lev_x[l + 1];
        P.out = top ? out : c->lev_x[l];
        P.epi = top ? epi : EPI_PLAIN;
        P.scale = scale;
        P.steps = c->d_steps;
        P.rsteps = c->d_rsteps;
        P.pin = pin;
        P.aux = aux;
        P.zc = zc_post > 0 ? std::min(zc_post, m) : m;
        const int nzb = (m + P.zc - 1) / P.zc;
        const bool has_q = P.epi == EPI_UZAWA_P || P.epi == EPI_SCALE_DOT ||
                           P.epi == EPI_SCALE_DOTONLY;
        const int lp = band3_lp(m);
        const int nrb = lp == 6 ? C3Geom<6>::NRB : lp == 5 ? C3Geom<5>::NRB : 1;
        const bool dot = top && epi_dot(epi);
        if (dot) {
            ensure_partials(c, (size_t)nrb * nzb * count);
            P.part = c->d_part;
        }
        const double fine = (double)m * m * m, coarse = (double)mc * mc * mc;
        double words = fine + coarse;
        if (P.epi != EPI_DOT_TAU && P.epi != EPI_SCALE_DOTONLY) words += fine;
        if (has_q) words += fine;
        dim3 g;
        {
            ProfScope prof(c, top ? K_MG_POST_FINE : K_MG_POST_COARSE, 8.0 * count * words);
            dispatch_c3<false>(s.shape3[l], lp, nzb, count, has_q, c->stream, P, &g);
        }
        PINT_LAUNCHED(c);
        PINT_CUDA_CHECK(cudaGetLastError());
        if (dot) reduce_partials(c, (int)(g.x * g.y), acc_slot);
    }
}

void vcycle3(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
             double scale, const double* pin, const double* aux, int acc_slot) {
    MgSet& s = c->mg[which];
    if (!s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    const int L = s.levels;
    auto tab = [&](int l) { return s.tab + (size_t)l * s.n_sets * 28; };
    const size_t need = (size_t)count * c->n;
    if (c->t3_cap < need) {
        if (c->d_t3a) cudaFree(c->d_t3a);
        if (c->d_t3b) cudaFree(c->d_t3b);
        PINT_CUDA_CHECK(cudaMalloc(&c->d_t3a, need * sizeof(double) + 16));
        PINT_CUDA_CHECK(cudaMalloc(&c->d_t3b, need * sizeof(double) + 16));
        c->t3_cap = need;
    }
    // fused band kernels for the level shapes of the BASELINE meshes (m = 2^k - 1 <= 63)
    static const bool old_path = getenv("PINT_3D_OLD") != nullptr;
    bool band_ok = !old_path;
    for (int l = 0; l + 1 < L; ++l) band_ok = band_ok && band3_lp(s.m[l]) != 0;
    if (band_ok) {
        vcycle3_band(c, s, count, b, out, epi, scale, pin, aux, acc_slot);
        return;
    }
    const double* bl = b;
    for (int l = 0; l + 1 < L; ++l) {
        const int m = s.m[l], mc = s.m[l + 1];
        {
            ProfScope prof(c, l == 0 ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                           8.0 * count * ((double)m * m * m + (double)mc * mc * mc));
            zdispatch(s.shape3[l], [&](auto P) {
                kz_residual<decltype(P)::value><<<zgrid(m, count), dim3(ZX, ZY), 0, c->stream>>>(
                    m, tab(l), s.sid, bl, c->d_t3a);
            });
            kz_restrict<<<zgrid(mc, count), dim3(ZX, ZY), 0, c->stream>>>(m, mc, c->d_t3a,
                                                                           c->lev_b[l + 1]);
        }
        c->launches += 2;
        bl = c->lev_b[l + 1];
    }
    PINT_CUDA_CHECK(cudaGetLastError());
    for (int l = L - 2; l >= 0; --l) {
        const int m = s.m[l], mc = s.m[l + 1];
        const bool top = l == 0;
        const bool direct = l + 1 == L - 1;
        const double* bcur = top ? b : c->lev_b[l];
        const double* ec = direct ? c->lev_b[l + 1] : c->lev_x[l + 1];
        {
            ProfScope prof(c, top ? K_MG_POST_FINE : K_MG_POST_COARSE,
                           8.0 * count * (3.0 * m * m * m + (double)mc * mc * mc));
            if (direct)
                kz_prolong<true><<<zgrid(m, count), dim3(ZX, ZY), 0, c->stream>>>(
                    m, mc, tab(l), tab(l + 1), s.sid, bcur, ec, c->d_t3b);
            else
                kz_prolong<false><<<zgrid(m, count), dim3(ZX, ZY), 0, c->stream>>>(
                    m, mc, tab(l), tab(l + 1), s.sid, bcur, ec, c->d_t3b);
            Smooth3 a{};
            a.m = m;
            a.tab = tab(l);
            a.sid = s.sid;
            a.b = bcur;
            a.x = c->d_t3b;
            a.out = top ? out : c->lev_x[l];
            a.epi = top ? epi : EPI_PLAIN;
            a.scale = scale;
            a.steps = c->d_steps;
            a.rsteps = c->d_rsteps;
            a.pin = pin;
            a.aux = aux;
            const dim3 g = zgrid(m, count);
            const bool dot = top && epi_dot(epi);
            if (dot) {
                ensure_partials(c, (size_t)g.x * g.y);
                a.part = c->d_part;
            }
            zdispatch(s.shape3[l], [&](auto P) {
                kz_smooth<decltype(P)::value><<<g, dim3(ZX, ZY), 0, c->stream>>>(a);
            });
            if (dot) reduce_partials(c, (int)(g.x * g.y), acc_slot);
        }
        c->launches += 2;
    }
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
