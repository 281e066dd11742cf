// General V-cycle options: cycles > 1 and smooth_steps > 1
// (spatial.py:148-169; MgVCycleSolver(cycles=, smooth_steps=),
// BlockDiagSolver / SchurPreconditioner pass them through).
//
// No BASELINE config uses them (all run V(1,1), one cycle), so the tuned band
// kernels implement exactly that case.  This module serves every other
// setting from thread-per-point kernels, one launch per sweep, for the
// translation-invariant 2D and 3D operators:
//
//   _vcycle(l, b):  x = dinv b;  (smooth - 1) x  x += dinv (b - A x)
//                   x = x + P vcycle(l + 1, P^T (b - A x))
//                   smooth x  x += dinv (b - A x)                 (spatial.py:148-161)
//   apply(b):       x = vcycle(0, b);  (cycles - 1) x  x += vcycle(0, b - A x)   (:163-169)
//
// Row sums run in CSR column order from 0 without FMA, restriction over
// ascending fine index, prolongation over ascending coarse index, exactly as
// the tuned kernels and the oracle, so the result is bit-identical to the
// reference's scipy products (tests/test_gpu_mg_options.py).  The finest-level
// epilogues of the fused kernels (1/tau, p update, scaling, the two dot
// products) are one more pass here.
#include <algorithm>
#include <vector>

#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

namespace {

constexpr int GT = 256;

template <int D>
__device__ __forceinline__ long long cube(int m) {
    return D == 2 ? (long long)m * m : (long long)m * m * m;
}

// row sum of the plane's stencil at point i of plane v (CSR order, exact zeros
// and out-of-domain neighbours skipped: they add +-0)
template <int D>
__device__ __forceinline__ double row_sum(const double* __restrict__ c, const double* __restrict__ v,
                                          int m, long long i) {
    const int xi = (int)(i % m);
    const int yi = (int)((i / m) % m);
    const int zi = D == 3 ? (int)(i / ((long long)m * m)) : 0;
    double r = 0.0;
    int k = 0;
    for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx, ++k) {
                const int X = xi + dx, Y = yi + dy, Z = zi + dz;
                const double cv = __ldg(c + k);
                if (cv == 0.0) continue;
                if (X < 0 || X >= m || Y < 0 || Y >= m || Z < 0 || Z >= m) continue;
                r = r + cv * __ldg(v + ((long long)Z * m + Y) * m + X);
            }
    return r;
}

// mode 0: out = dinv b;  1: out = x + dinv (b - A x);  2: out = b - A x
template <int D>
__global__ void __launch_bounds__(GT)
    k_g_sweep(int m, long long planes, const double* __restrict__ tab, int tw,
              const int* __restrict__ sid, const double* __restrict__ b,
              const double* __restrict__ x, double* __restrict__ out, int mode) {
    const long long n = cube<D>(m), total = planes * n;
    constexpr int S = D == 2 ? 9 : 27;
    for (long long g = (long long)blockIdx.x * GT + threadIdx.x; g < total;
         g += (long long)gridDim.x * GT) {
        const long long pl = g / n, i = g - pl * n;
        const double* c = tab + (size_t)__ldg(sid + pl) * tw;
        const double bv = __ldg(b + g);
        if (mode == 0) {
            out[g] = __ldg(c + S) * bv;
            continue;
        }
        const double ax = row_sum<D>(c, x + pl * n, m, i);
        out[g] = mode == 2 ? bv - ax : __ldg(x + g) + __ldg(c + S) * (bv - ax);
    }
}

// b_c = P^T r: the 3^D fine nodes of each coarse node in ascending fine index,
// weights (w w) w with w = (1/2, 1, 1/2)  (spatial.py:75-84, 156)
template <int D>
__global__ void __launch_bounds__(GT)
    k_g_restrict(int m, int mc, long long planes, const double* __restrict__ r,
                 double* __restrict__ bc) {
    const long long n = cube<D>(m), nc = cube<D>(mc), total = planes * nc;
    const double w[3] = {0.5, 1.0, 0.5};
    for (long long g = (long long)blockIdx.x * GT + threadIdx.x; g < total;
         g += (long long)gridDim.x * GT) {
        const long long pl = g / nc, i = g - pl * nc;
        const int X = (int)(i % mc), Y = (int)((i / mc) % mc);
        const int Z = D == 3 ? (int)(i / ((long long)mc * mc)) : 0;
        const double* rp = r + pl * n;
        double v = 0.0;
        bool first = true;
        for (int a = 0; a < (D == 3 ? 3 : 1); ++a)
            for (int bb = 0; bb < 3; ++bb)
                for (int cc = 0; cc < 3; ++cc) {
                    const long long fi =
                        ((long long)(D == 3 ? 2 * Z + a : 0) * m + (2 * Y + bb)) * m + (2 * X + cc);
                    const double wt = D == 3 ? (w[a] * w[bb]) * w[cc] : w[bb] * w[cc];
                    const double t = wt * __ldg(rp + fi);
                    v = first ? t : v + t;
                    first = false;
                }
        bc[g] = v;
    }
}

// x = x + P e over ascending coarse index (spatial.py:157); direct: e = b_c / a_c
// on the one-point coarsest grid (spatial.py:149-150)
template <int D>
__global__ void __launch_bounds__(GT)
    k_g_prolong_add(int m, int mc, long long planes, const double* __restrict__ tabc, int tw,
                    const int* __restrict__ sid, bool direct, const double* __restrict__ ec,
                    double* __restrict__ x) {
    const long long n = cube<D>(m), nc = cube<D>(mc), total = planes * n;
    constexpr int S = D == 2 ? 9 : 27;
    for (long long g = (long long)blockIdx.x * GT + threadIdx.x; g < total;
         g += (long long)gridDim.x * GT) {
        const long long pl = g / n, i = g - pl * n;
        const int f[3] = {(int)(i % m), (int)((i / m) % m),
                          D == 3 ? (int)(i / ((long long)m * m)) : 1};
        // per axis: odd f -> coarse (f-1)/2, weight 1; even -> f/2-1 then f/2, weights 1/2
        int j0[3], j1[3];
        double wv[3];
        bool h0[3], h1[3];
        for (int a = 0; a < 3; ++a) {
            if (f[a] & 1) {
                j0[a] = j1[a] = (f[a] - 1) >> 1;
                wv[a] = 1.0;
                h0[a] = true;
                h1[a] = false;
            } else {
                j0[a] = (f[a] >> 1) - 1;
                j1[a] = f[a] >> 1;
                wv[a] = 0.5;
                h0[a] = j0[a] >= 0;
                h1[a] = j1[a] < mc;
            }
        }
        if (D == 2) {  // no z axis: a single unit term
            j0[2] = j1[2] = 0;
            wv[2] = 1.0;
            h0[2] = true;
            h1[2] = false;
        }
        const double ac = direct ? __ldg(tabc + (size_t)__ldg(sid + pl) * tw + S / 2) : 1.0;
        const double* ep = ec + pl * nc;
        double pe = 0.0;
        bool first = true;
        for (int a = 0; a < 2; ++a) {
            if (!(a ? h1[2] : h0[2])) continue;
            for (int bb = 0; bb < 2; ++bb) {
                if (!(bb ? h1[1] : h0[1])) continue;
                for (int cc = 0; cc < 2; ++cc) {
                    if (!(cc ? h1[0] : h0[0])) continue;
                    const long long ci = ((long long)(a ? j1[2] : j0[2]) * mc + (bb ? j1[1] : j0[1])) * mc +
                                         (cc ? j1[0] : j0[0]);
                    double e = __ldg(ep + ci);
                    if (direct) e = e / ac;
                    const double wt = D == 3 ? (wv[2] * wv[1]) * wv[0] : wv[1] * wv[0];
                    const double t = wt * e;
                    pe = first ? t : pe + t;
                    first = false;
                }
            }
        }
        x[g] = x[g] + pe;
    }
}

__global__ void __launch_bounds__(GT)
    k_g_add(long long total, double* __restrict__ x, const double* __restrict__ t) {
    for (long long g = (long long)blockIdx.x * GT + threadIdx.x; g < total;
         g += (long long)gridDim.x * GT)
        x[g] = x[g] + t[g];
}

__device__ __noinline__ double gdiv_rn(double x, double y) { return x / y; }

// finest-level epilogue of the fused kernels as a pass of its own
__global__ void __launch_bounds__(GT)
    k_g_epilogue(long long n, long long planes, int epi, double scale,
                 const double* __restrict__ steps, const double* __restrict__ rsteps,
                 const double* __restrict__ x, const double* __restrict__ b,
                 const double* __restrict__ pin, const double* __restrict__ aux,
                 double* __restrict__ out, double* __restrict__ part) {
    const long long total = planes * n;
    double acc = 0.0;
    for (long long g = (long long)blockIdx.x * GT + threadIdx.x; g < total;
         g += (long long)gridDim.x * GT) {
        const long long pl = g / n;
        const double xn = x[g];
        const double rtau = __ldg(rsteps + pl);
        auto divtau = [&](double v) { return rtau > 0.0 ? v * rtau : gdiv_rn(v, __ldg(steps + pl)); };
        switch (epi) {
            case EPI_PLAIN: out[g] = xn; break;
            case EPI_DIV_TAU: out[g] = divtau(xn); break;
            case EPI_UZAWA_P: {
                const double dp = divtau(xn);
                out[g] = __ldg(pin + g) + dp;
                acc = acc + __ldg(b + g) * dp;
                break;
            }
            case EPI_DOT_TAU: acc = acc + __ldg(b + g) * divtau(xn); break;
            case EPI_SCALE: out[g] = scale * xn; break;
            case EPI_SCALE_DOT: {
                const double w = scale * xn;
                out[g] = w;
                acc = acc + __ldg(aux + g) * w;
                break;
            }
            default: acc = acc + __ldg(aux + g) * (scale * xn); break;
        }
    }
    if (part) {
        const double s = block_sum<GT>(acc);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

int grid_of(long long total) {
    return (int)std::min<long long>((total + GT - 1) / GT, 148LL * 16);
}

double* gen_buf(pint_ctx* c, int slot, size_t count) {
    if (c->gen_scratch.size() <= (size_t)slot) {
        c->gen_scratch.resize(slot + 1, nullptr);
        c->gen_cap.resize(slot + 1, 0);
    }
    if (c->gen_cap[slot] < count) {
        if (c->gen_scratch[slot]) cudaFree(c->gen_scratch[slot]);
        PINT_CUDA_CHECK(cudaMalloc(&c->gen_scratch[slot], count * sizeof(double) + 16));
        c->gen_cap[slot] = count;
    }
    return c->gen_scratch[slot];
}

template <int D>
void cycle_generic(pint_ctx* c, MgSet& s, int count, const double* b, double* x0) {
    const int L = s.levels, tw = D == 2 ? PINT_TW : 28;
    const int smooth = s.smooth;
    auto tab = [&](int l) { return s.tab + (size_t)l * s.n_sets * tw; };
    auto npts = [&](int l) { return (long long)count * (D == 2 ? (long long)s.m[l] * s.m[l]
                                                                : (long long)s.m[l] * s.m[l] * s.m[l]); };
    if (s.m[L - 1] != 1) pint_throw(PINT_INPUT, "generic V-cycle needs a one-point coarsest grid");
    // per level: slot 3l = x, 3l+1 = ping-pong partner, 3l+2 = residual / level rhs
    std::vector<double*> xs(L, nullptr), bs(L, nullptr);
    std::vector<const double*> rhs(L, nullptr);
    rhs[0] = b;
    auto sweep = [&](int l, const double* bb, const double* xin, double* out, int mode) {
        k_g_sweep<D><<<grid_of(npts(l)), GT, 0, c->stream>>>(s.m[l], count, tab(l), tw, s.sid, bb,
                                                             xin, out, mode);
        PINT_LAUNCHED(c);
    };
    for (int l = 0; l + 1 < L; ++l) {
        double* xa = l == 0 ? x0 : gen_buf(c, 3 * l, npts(l));
        double* xb = gen_buf(c, 3 * l + 1, npts(l));
        double* rl = gen_buf(c, 3 * l + 2, npts(l));
        sweep(l, rhs[l], nullptr, xa, 0);
        for (int k = 1; k < smooth; ++k) {
            sweep(l, rhs[l], xa, xb, 1);
            PINT_CUDA_CHECK(cudaMemcpyAsync(xa, xb, npts(l) * sizeof(double),
                                            cudaMemcpyDeviceToDevice, c->stream));
        }
        sweep(l, rhs[l], xa, rl, 2);
        double* bc = gen_buf(c, 3 * (l + 1) + 2 + 3 * L, npts(l + 1));
        k_g_restrict<D><<<grid_of(npts(l + 1)), GT, 0, c->stream>>>(s.m[l], s.m[l + 1], count, rl, bc);
        PINT_LAUNCHED(c);
        xs[l] = xa;
        bs[l] = xb;
        rhs[l + 1] = bc;
    }
    for (int l = L - 2; l >= 0; --l) {
        const bool direct = l + 1 == L - 1;
        const double* ec = direct ? rhs[l + 1] : xs[l + 1];
        k_g_prolong_add<D><<<grid_of(npts(l)), GT, 0, c->stream>>>(
            s.m[l], s.m[l + 1], count, tab(l + 1), tw, s.sid, direct, ec, xs[l]);
        PINT_LAUNCHED(c);
        for (int k = 0; k < smooth; ++k) {
            sweep(l, rhs[l], xs[l], bs[l], 1);
            PINT_CUDA_CHECK(cudaMemcpyAsync(xs[l], bs[l], npts(l) * sizeof(double),
                                            cudaMemcpyDeviceToDevice, c->stream));
        }
    }
    PINT_CUDA_CHECK(cudaGetLastError());
}

template <int D>
void run_generic(pint_ctx* c, MgSet& s, int count, const double* b, double* out, int epi,
                 double scale, const double* pin, const double* aux, int acc_slot) {
    const long long total = (long long)count * c->n;
    const int L = s.levels;
    double* x = gen_buf(c, 6 * L + 8, total);
    cycle_generic<D>(c, s, count, b, x);
    for (int k = 1; k < s.cycles; ++k) {
        double* r = gen_buf(c, 6 * L + 9, total);
        double* t = gen_buf(c, 6 * L + 10, total);
        const int tw = D == 2 ? PINT_TW : 28;
        k_g_sweep<D><<<grid_of(total), GT, 0, c->stream>>>(c->m, count, s.tab, tw, s.sid, b, x, r, 2);
        PINT_LAUNCHED(c);
        cycle_generic<D>(c, s, count, r, t);
        k_g_add<<<grid_of(total), GT, 0, c->stream>>>(total, x, t);
        PINT_LAUNCHED(c);
    }
    const bool dot = epi == EPI_UZAWA_P || epi == EPI_DOT_TAU || epi == EPI_SCALE_DOT ||
                     epi == EPI_SCALE_DOTONLY;
    const int g = grid_of(total);
    double* part = nullptr;
    if (dot) {
        ensure_partials(c, (size_t)g);
        part = c->d_part;
    }
    k_g_epilogue<<<g, GT, 0, c->stream>>>(c->n, count, epi, scale, c->d_steps, c->d_rsteps, x, b,
                                          pin, aux, out, part);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
    if (dot) reduce_partials(c, g, acc_slot);
}

}  // namespace

bool vcycle_is_generic(const pint_ctx* c, int which) {
    const MgSet& s = c->mg[which];
    return s.cycles != 1 || s.smooth != 1;
}

void vcycle_generic(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
                    double scale, const double* pin, const double* aux, int acc_slot) {
    MgSet& s = c->mg[which];
    if (!s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    if (c->field)
        pint_throw(PINT_INPUT, "cycles / smooth_steps other than 1 are not available for "
                               "per-point stiffness fields");
    if (c->dims == 2)
        run_generic<2>(c, s, count, b, out, epi, scale, pin, aux, acc_slot);
    else
        run_generic<3>(c, s, count, b, out, epi, scale, pin, aux, acc_slot);
}

}  // namespace pint
