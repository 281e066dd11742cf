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
// Round-1 form: thread per point, neighbours through L1/L2 (no TMA bands),
// one launch per level and phase over every plane of the batch.
#include <algorithm>

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
    k3_apply(int m, const double* __restrict__ st, const double* __restrict__ in,
             double* __restrict__ out) {
    const Pt q = point3(m);
    if (!q.ok) return;
    const long long n = (long long)m * m * m;
    const long long t = blockIdx.y;
    out[t * n + q.i] = st27(st, in + t * n, m, q.x, q.y, q.z);
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
// r = b - A (dinv*b)   (spatial.py:153,156: x = dinv*b; r = b - A x)
__global__ void __launch_bounds__(T3)
    k3_residual(int m, const double* __restrict__ tab, const int* __restrict__ sid,
                const double* __restrict__ b, double* __restrict__ r) {
    const Pt q = point3(m);
    if (!q.ok) return;
    const long long n = (long long)m * m * m;
    const long long t = blockIdx.y;
    const double* tb = tab + (size_t)__ldg(sid + t) * 28;
    const double d = __ldg(tb + 27);
    const double* bp = b + t * n;
    r[t * n + q.i] = __ldg(bp + q.i) - st27_scaled(tb, d, bp, m, q.x, q.y, q.z);
}

// b_c = P^T r: ascending fine index (z, y, x) over the 27 fine nodes of the
// coarse node, weights (wz*wy)*wx with w = 0.5, 1, 0.5  (kron of spatial.py:75-84)
__global__ void __launch_bounds__(T3)
    k3_restrict(int m, int mc, const double* __restrict__ r, double* __restrict__ bc) {
    const Pt q = point3(mc);
    if (!q.ok) return;
    const long long n = (long long)m * m * m, nc = (long long)mc * mc * mc;
    const long long t = blockIdx.y;
    const double* rp = r + t * n;
    const double w[3] = {0.5, 1.0, 0.5};
    double s = 0.0;
    int k = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc, ++k) {
                const long long fi = ((long long)(2 * q.z + a) * m + (2 * q.y + bb)) * m + (2 * q.x + cc);
                const double tterm = ((w[a] * w[bb]) * w[cc]) * __ldg(rp + fi);
                s = (k == 0) ? tterm : s + tterm;
            }
    bc[t * nc + q.i] = s;
}

__device__ __forceinline__ void pro_terms(int f, int mc, int* j, double* w, int& cnt) {
    if (f & 1) {
        j[0] = (f - 1) >> 1;
        w[0] = 1.0;
        cnt = 1;
    } else {
        cnt = 0;
        if ((f >> 1) - 1 >= 0) {
            j[cnt] = (f >> 1) - 1;
            w[cnt] = 0.5;
            ++cnt;
        }
        if ((f >> 1) < mc) {
            j[cnt] = f >> 1;
            w[cnt] = 0.5;
            ++cnt;
        }
    }
}

// x = dinv*b + P e (csr_matvec of P over ascending coarse index); e = b_c / a_c
// on the 1x1x1 coarsest grid (spatial.py:149-150, 157)
__global__ void __launch_bounds__(T3)
    k3_prolong(int m, int mc, const double* __restrict__ tab, const double* __restrict__ tabc,
               const int* __restrict__ sid, int direct, const double* __restrict__ b,
               const double* __restrict__ ec, double* __restrict__ x) {
    const Pt q = point3(m);
    if (!q.ok) return;
    const long long n = (long long)m * m * m, nc = (long long)mc * mc * mc;
    const long long t = blockIdx.y;
    const int set = __ldg(sid + t);
    const double d = __ldg(tab + (size_t)set * 28 + 27);
    const double ac = direct ? __ldg(tabc + (size_t)set * 28 + 13) : 1.0;
    int jz[2], jy[2], jx[2], nz, ny, nx;
    double wz[2], wy[2], wx[2];
    pro_terms(q.z, mc, jz, wz, nz);
    pro_terms(q.y, mc, jy, wy, ny);
    pro_terms(q.x, mc, jx, wx, nx);
    const double* ep = ec + t * nc;
    double pe = 0.0;
    bool first = true;
    for (int a = 0; a < nz; ++a)
        for (int bb = 0; bb < ny; ++bb)
            for (int cc = 0; cc < nx; ++cc) {
                double e = __ldg(ep + ((long long)jz[a] * mc + jy[bb]) * mc + jx[cc]);
                if (direct) e = e / ac;
                const double tterm = ((wz[a] * wy[bb]) * wx[cc]) * e;
                pe = first ? tterm : pe + tterm;
                first = false;
            }
    x[t * n + q.i] = d * __ldg(b + t * n + q.i) + pe;
}

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

// x += dinv*(b - A x) (spatial.py:159-160) + the finest-level epilogues
__global__ void __launch_bounds__(T3) k3_smooth(Smooth3 a) {
    const Pt q = point3(a.m);
    const long long n = (long long)a.m * a.m * a.m;
    const long long t = blockIdx.y;
    double acc = 0.0;
    if (q.ok) {
        const double* tb = a.tab + (size_t)__ldg(a.sid + t) * 28;
        const double d = __ldg(tb + 27);
        const long long gi = t * n + q.i;
        const double bv = __ldg(a.b + gi);
        const double xv = __ldg(a.x + gi);
        const double xn = xv + d * (bv - st27(tb, a.x + t * n, a.m, q.x, q.y, q.z));
        auto divtau = [&](double v) {
            const double r = __ldg(a.rsteps + t);
            return r > 0.0 ? v * r : v / __ldg(a.steps + t);
        };
        switch (a.epi) {
            case EPI_PLAIN: a.out[gi] = xn; break;
            case EPI_DIV_TAU: a.out[gi] = divtau(xn); break;
            case EPI_UZAWA_P: {
                const double dp = divtau(xn);
                a.out[gi] = __ldg(a.pin + gi) + dp;
                acc = bv * dp;
                break;
            }
            case EPI_DOT_TAU: acc = bv * divtau(xn); break;
            case EPI_SCALE: a.out[gi] = a.scale * xn; break;
            case EPI_SCALE_DOT: {
                const double w = a.scale * xn;
                a.out[gi] = w;
                acc = __ldg(a.aux + gi) * w;
                break;
            }
            case EPI_SCALE_DOTONLY: acc = __ldg(a.aux + gi) * (a.scale * xn); break;
        }
    }
    if (a.part) {
        const double s = block_sum<T3>(acc);
        if (threadIdx.x == 0) a.part[(long long)blockIdx.y * gridDim.x + blockIdx.x] = s;
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

void launch_timeop3(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                    double* out) {
    const dim3 g((unsigned)(((long long)c->n + T3 - 1) / T3), (unsigned)((c->N + G3 - 1) / G3));
    const int qmin = c->has_prev ? -1 : 0, qmax = c->has_next ? c->N : c->N - 1;
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
    k3_apply<<<grid3(c->m, count), T3, 0, c->stream>>>(c->m, st, in, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_fold3(pint_ctx* c, const double* load, const double* u0, double* f) {
    ProfScope prof(c, K_FOLD, 16.0 * (double)c->N * c->n);
    k3_fold<<<grid3(c->m, c->N), T3, 0, c->stream>>>(c->m, c->d_steps, c->d_mass, load, u0, f);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
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
    const double* bl = b;
    for (int l = 0; l + 1 < L; ++l) {
        const int m = s.m[l], mc = s.m[l + 1];
        {
            ProfScope prof(c, l == 0 ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                           8.0 * count * ((double)m * m * m + (double)mc * mc * mc));
            k3_residual<<<grid3(m, count), T3, 0, c->stream>>>(m, tab(l), s.sid, bl, c->d_t3a);
            k3_restrict<<<grid3(mc, count), T3, 0, c->stream>>>(m, mc, c->d_t3a, c->lev_b[l + 1]);
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
            k3_prolong<<<grid3(m, count), T3, 0, c->stream>>>(m, mc, tab(l), tab(l + 1), s.sid,
                                                              direct ? 1 : 0, bcur, ec, c->d_t3b);
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
            const dim3 g = grid3(m, count);
            const bool dot = top && epi_dot(epi);
            if (dot) {
                ensure_partials(c, (size_t)g.x * g.y);
                a.part = c->d_part;
            }
            k3_smooth<<<g, T3, 0, c->stream>>>(a);
            if (dot) reduce_partials(c, (int)(g.x * g.y), acc_slot);
        }
        c->launches += 2;
    }
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
