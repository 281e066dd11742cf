// Time-global stencil operators K, K^T, A-block and the fused Uzawa residuals.
//
// Reference: TimeGlobalSystem.apply_K / apply_Kt / apply_Abd
// (operators.py:78-99), fold_rhs (operators.py:22-26) and the two residual
// expressions of uzawa_solve (solvers.py:224, 227-229):
//   r1 = (K u - A p) - f
//   z  = (f - K^T p) - ((K u + K^T u) + A u)
// evaluated with the reference's association order so results are
// bit-identical to the numpy/scipy reference.
//
// One thread per spatial point; each CTA marches through G consecutive time
// planes, carrying the mass-stencil products M u_{n-1}, M u_n, M u_{n+1}
// (and M p_n, M p_{n+1}) in registers so every input plane is read from HBM
// once (the neighbouring-plane halo is a register carry, not a re-read).
#include <algorithm>
#include <cstdlib>

#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

constexpr int TX = 32, TY = 8, GT = 8;  // 32x8 spatial tile, 8 planes per CTA

template <int OP>
__global__ void __launch_bounds__(TX* TY)
    k_timeop(int m, int N, int qmin, int qmax, const double* __restrict__ mass,
             const double* __restrict__ ast,
             const int* __restrict__ asid, const double* __restrict__ ascale,
             const double* __restrict__ u, const double* __restrict__ p,
             const double* __restrict__ f, double* __restrict__ out) {
    const int x = blockIdx.x * TX + threadIdx.x;
    const int y = blockIdx.y * TY + threadIdx.y;
    if (x >= m || y >= m) return;
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    const int n0 = blockIdx.z * GT;
    const int n1 = min(N, n0 + GT);
    double cm[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) cm[k] = __ldg(mass + k);

    if (OP == OP_ABD) {
        for (int t = n0; t < n1; ++t) {
            const double* a = ast + 9 * __ldg(asid + t);
            double ca[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) ca[k] = __ldg(a + k);
            out[t * n + i] = __ldg(ascale + t) * stencil9_global(ca, u + t * n, m, x, y);
        }
        return;
    }
    if (OP == OP_K || OP == OP_R1) {
        // planes [qmin, qmax] are addressable (qmin = -1 / qmax = N: ghost planes of the
        // neighbouring ranks when the time axis is partitioned)
        double mprev = (n0 - 1 >= qmin)
                           ? stencil9_global(cm, u + (long long)(n0 - 1) * (long long)n, m, x, y)
                           : 0.0;
        for (int t = n0; t < n1; ++t) {
            const double mcur = stencil9_global(cm, u + t * n, m, x, y);
            const double ku = (t - 1 >= qmin) ? mcur - mprev : mcur;
            if (OP == OP_K) {
                out[t * n + i] = ku;
            } else {
                const double* a = ast + 9 * __ldg(asid + t);
                double ca[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) ca[k] = __ldg(a + k);
                const double ap = __ldg(ascale + t) * stencil9_global(ca, p + t * n, m, x, y);
                out[t * n + i] = (ku - ap) - __ldg(f + t * n + i);
            }
            mprev = mcur;
        }
        return;
    }
    if (OP == OP_KT) {
        double mcur = stencil9_global(cm, u + n0 * n, m, x, y);
        for (int t = n0; t < n1; ++t) {
            const double mnext = (t + 1 <= qmax) ? stencil9_global(cm, u + (t + 1) * n, m, x, y) : 0.0;
            out[t * n + i] = (t + 1 <= qmax) ? mcur - mnext : mcur;
            mcur = mnext;
        }
        return;
    }
    if (OP == OP_Z) {
        double muprev = (n0 - 1 >= qmin)
                            ? stencil9_global(cm, u + (long long)(n0 - 1) * (long long)n, m, x, y)
                            : 0.0;
        double mucur = stencil9_global(cm, u + n0 * n, m, x, y);
        double mpcur = stencil9_global(cm, p + n0 * n, m, x, y);
        for (int t = n0; t < n1; ++t) {
            const bool has_next = t + 1 <= qmax;
            const double munext = has_next ? stencil9_global(cm, u + (t + 1) * n, m, x, y) : 0.0;
            const double mpnext = has_next ? stencil9_global(cm, p + (t + 1) * n, m, x, y) : 0.0;
            const double ktp = has_next ? mpcur - mpnext : mpcur;
            const double ku = (t - 1 >= qmin) ? mucur - muprev : mucur;
            const double ktu = has_next ? mucur - munext : mucur;
            const double* a = ast + 9 * __ldg(asid + t);
            double ca[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) ca[k] = __ldg(a + k);
            const double au = __ldg(ascale + t) * stencil9_global(ca, u + t * n, m, x, y);
            out[t * n + i] = (__ldg(f + t * n + i) - ktp) - ((ku + ktu) + au);
            muprev = mucur;
            mucur = munext;
            mpcur = mpnext;
        }
        return;
    }
}

// out_plane = A_ref in_plane (schur.py:72), count planes
__global__ void __launch_bounds__(TX* TY)
    k_aref(int m, int count, const double* __restrict__ aref, const double* __restrict__ in,
           double* __restrict__ out) {
    const int x = blockIdx.x * TX + threadIdx.x;
    const int y = blockIdx.y * TY + threadIdx.y;
    if (x >= m || y >= m) return;
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    double ca[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) ca[k] = __ldg(aref + k);
    const int n0 = blockIdx.z * GT;
    const int n1 = min(count, n0 + GT);
    for (int t = n0; t < n1; ++t) out[t * n + i] = stencil9_global(ca, in + t * n, m, x, y);
}

// fold_rhs (operators.py:22-26): f_n = tau_n * load_n; f_0 += M u_init
__global__ void __launch_bounds__(TX* TY)
    k_fold_rhs(int m, int N, const double* __restrict__ steps, const double* __restrict__ mass,
               const double* __restrict__ load, const double* __restrict__ u_init,
               double* __restrict__ f) {
    const int x = blockIdx.x * TX + threadIdx.x;
    const int y = blockIdx.y * TY + threadIdx.y;
    if (x >= m || y >= m) return;
    const size_t n = (size_t)m * m;
    const size_t i = (size_t)y * m + x;
    const int n0 = blockIdx.z * GT;
    const int n1 = min(N, n0 + GT);
    for (int t = n0; t < n1; ++t) {
        double v = __ldg(steps + t) * __ldg(load + t * n + i);
        if (t == 0) {
            double cm[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) cm[k] = __ldg(mass + k);
            v = v + stencil9_global(cm, u_init, m, x, y);
        }
        f[t * n + i] = v;
    }
}

// u = u + omega * y   (solvers.py:231, time-partitioned driver)
__global__ void __launch_bounds__(256) k_axpy(double* __restrict__ u, const double* __restrict__ y,
                                              double omega, long long count) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < count; i += (long long)gridDim.x * 256)
        u[i] = u[i] + omega * y[i];
}

// out = ((x0 + a1 x1) + a2 x2) * sc, absent terms skipped: the exact
// operation sequence of numpy's  v - a*w1 - b*w2  /  s*y  /  x + phi*w
// (no FMA in this file), used by the MINRES driver (solvers.py:267-327)
__global__ void __launch_bounds__(256)
    k_lincomb(double* __restrict__ out, const double* __restrict__ x0, double a1,
              const double* __restrict__ x1, double a2, const double* __restrict__ x2, double sc,
              int use_sc, long long count) {
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < count;
         i += (long long)gridDim.x * 256) {
        double v = x0[i];
        if (x1) v = v + a1 * x1[i];
        if (x2) v = v + a2 * x2[i];
        out[i] = use_sc ? v * sc : v;
    }
}

// per-CTA partial sums of a.b (grid-stride, fixed grid: deterministic)
__global__ void __launch_bounds__(256)
    k_dot_partials(const double* __restrict__ a, const double* __restrict__ b, long long count,
                   double* __restrict__ part) {
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < count;
         i += (long long)gridDim.x * 256)
        s += a[i] * b[i];
    s = block_sum<256>(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void launch_lincomb(pint_ctx* c, double* out, const double* x0, double a1, const double* x1,
                    double a2, const double* x2, double sc, bool use_sc, long long count) {
    const long long blocks = std::min<long long>((count + 255) / 256, 148LL * 16);
    k_lincomb<<<(unsigned)std::max<long long>(blocks, 1), 256, 0, c->stream>>>(
        out, x0, a1, x1, a2, x2, sc, use_sc ? 1 : 0, count);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_dot(pint_ctx* c, const double* a, const double* b, long long count, int slot) {
    constexpr int kParts = 148 * 8;
    ensure_partials(c, kParts);
    k_dot_partials<<<kParts, 256, 0, c->stream>>>(a, b, count, c->d_part);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
    reduce_partials(c, kParts, slot);
}

void launch_axpy(pint_ctx* c, double* u, const double* y, double omega, long long count) {
    const long long blocks = std::min<long long>((count + 255) / 256, 148LL * 16);
    k_axpy<<<(unsigned)std::max<long long>(blocks, 1), 256, 0, c->stream>>>(u, y, omega, count);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

// Deterministic final reduction of per-CTA partial sums into d_acc[slot].
__global__ void __launch_bounds__(1024) k_reduce_partials(const double* __restrict__ part,
                                                          int nparts, double* __restrict__ acc,
                                                          int slot) {
    double s = 0.0;
    for (int k = threadIdx.x; k < nparts; k += 1024) s += part[k];
    s = block_sum<1024>(s);
    if (threadIdx.x == 0) acc[slot] = s;
}

static dim3 plane_grid(int m, int planes) {
    return dim3((m + TX - 1) / TX, (m + TY - 1) / TY, (planes + GT - 1) / GT);
}

void launch_timeop(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                   double* out) {
    if (c->dims == 3) {
        launch_timeop3(c, op, u, p, f, out);
        return;
    }
    if (c->field && (op == OP_ABD || op == OP_R1 || op == OP_Z)) {
        launch_timeop_field(c, op, u, p, f, out);
        return;
    }
    if ((op == OP_R1 || op == OP_Z) && band_timeop_supported(c) && !getenv("PINT_NO_BAND_TIMEOP")) {
        launch_band_timeop(c, op, u, p, f, out);
        return;
    }
    const dim3 g = plane_grid(c->m, c->N), b(TX, TY);
    static const int kid[] = {K_TIMEOP_K, K_TIMEOP_KT, K_TIMEOP_ABD, K_TIMEOP_R1, K_TIMEOP_Z};
    static const int passes[] = {2, 2, 2, 4, 4};
    if (op < 0 || op > OP_Z) pint_throw(PINT_INPUT, "unknown time operator");
    ProfScope prof(c, kid[op], 8.0 * passes[op] * (double)c->N * c->n);
    switch (op) {
#define PINT_OP(OPV)                                                                         \
    case OPV:                                                                                \
        k_timeop<OPV><<<g, b, 0, c->stream>>>(c->m, c->N, c->has_prev ? -1 : 0,             \
                                              c->has_next ? c->N : c->N - 1, c->d_mass,     \
                                              c->d_ast, c->d_asid, c->d_ascale, u, p, f, out); \
        break;
        PINT_OP(OP_K)
        PINT_OP(OP_KT)
        PINT_OP(OP_ABD)
        PINT_OP(OP_R1)
        PINT_OP(OP_Z)
#undef PINT_OP
        default:
            pint_throw(PINT_INPUT, "unknown time operator");
    }
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_aref(pint_ctx* c, const double* in, double* out, int count) {
    if (c->dims == 3) {
        launch_apply3(c, c->d_aref, in, out, count);
        return;
    }
    if (c->field) {
        launch_aref_field(c, in, out, count);
        return;
    }
    if (band_timeop_supported(c)) {
        launch_band_apply(c, c->d_aref, c->h_aref.data(), in, out, count);
        return;
    }
    ProfScope prof(c, K_AREF, 16.0 * (double)count * c->n);
    k_aref<<<plane_grid(c->m, count), dim3(TX, TY), 0, c->stream>>>(c->m, count, c->d_aref, in,
                                                                     out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void launch_fold_rhs(pint_ctx* c, const double* load, const double* u_init, double* f) {
    if (c->dims == 3) {
        launch_fold3(c, load, u_init, f);
        return;
    }
    ProfScope prof(c, K_FOLD, 16.0 * (double)c->N * c->n);
    k_fold_rhs<<<plane_grid(c->m, c->N), dim3(TX, TY), 0, c->stream>>>(
        c->m, c->N, c->d_steps, c->d_mass, load, u_init, f);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

void ensure_partials(pint_ctx* c, size_t nparts) {
    if (nparts <= c->part_cap) return;
    if (c->d_part) cudaFree(c->d_part);
    PINT_CUDA_CHECK(cudaMalloc(&c->d_part, nparts * sizeof(double)));
    c->part_cap = nparts;
}

void reduce_partials(pint_ctx* c, int nparts, int slot) {
    ProfScope prof(c, K_REDUCE, 8.0 * nparts);
    k_reduce_partials<<<1, 1024, 0, c->stream>>>(c->d_part, nparts, c->d_acc, slot);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
