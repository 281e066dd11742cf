// Diagnostic-mode exact spatial solves on the device: the reference's
// sequential implicit-Euler oracle and discrete parabolic S-norm.
//
// The reference evaluates both with SuperLU factorisations on the host:
//   sequential_euler_solve  (solvers.py:158-174):
//       (M + tau_n A_n) u_n = M u_{n-1} + tau_n load_n,   n = 1..N in order
//   s_norm / s_bilinear     (operators.py:155-183):
//       |v|_S^2 = sum_n tau_n g_n . A_n^{-1} g_n          g_n = M (v_n - v_{n-1}) / tau_n
//               + sum_n v_n . tau_n A_n v_n                (energy, apply_Abd)
//               + v_N . M v_N + sum_n dv_n . M dv_n        (jump form, v_0 = 0)
// Here every SPD solve is a multigrid-preconditioned conjugate gradient run
// to the rounding floor (relative residual <= tol, default 1e-14): the
// preconditioner is one V-cycle of the package's own multigrid (the A~ set
// for A_n, the EULER set of M + tau_n A_n), batched over all planes with a
// per-plane CG recurrence (alpha_n, beta_n live in device arrays, so one
// launch serves every plane).  The result equals the direct solve to ~1e-14
// relative, far inside the 1e-8 final-solution bar these quantities check.
// Off the hot path: thread-per-point kernels, no band pipelines.
#include <algorithm>
#include <cmath>
#include <vector>

#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

namespace {

constexpr int NT = 256;

// y_b = s_b * (S_{sid[b]} x_b) [ y = base - y when base ] for planes b of
// m^d points; S a 9-point (2D) / 27-point (3D) stencil row `stride` apart,
// summed in CSR column order from 0 (z, y, x slowest to fastest)
template <int D>
__global__ void __launch_bounds__(NT)
    k_st_apply(int m, long long planes, const double* __restrict__ tab, int stride,
               const int* __restrict__ sid, const double* __restrict__ scale,
               const double* __restrict__ x, const double* __restrict__ base,
               double* __restrict__ y) {
    const long long n = D == 2 ? (long long)m * m : (long long)m * m * m;
    const long long total = planes * n;
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT) {
        const long long b = g / n;
        const long long i = g - b * n;
        const double* c = tab + (sid ? (long long)__ldg(sid + b) * stride : 0);
        const double* v = x + b * n;
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
        if (scale) r = __ldg(scale + b) * r;
        y[g] = base ? base[g] - r : r;
    }
}

// out[b] = sum_i a_b[i] w_b[i] per plane, fixed-order (deterministic)
__global__ void __launch_bounds__(NT)
    k_plane_dot(long long n, const double* __restrict__ a, const double* __restrict__ w,
                double* __restrict__ out) {
    const long long b = blockIdx.x;
    const double* pa = a + b * n;
    const double* pw = w + b * n;
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += NT) s += pa[i] * pw[i];
    s = block_sum<NT>(s);
    if (threadIdx.x == 0) out[b] = s;
}

// x += alpha p; r -= alpha q with alpha_b = rz_b / pq_b (0 on a converged plane)
__global__ void __launch_bounds__(NT)
    k_cg_xr(long long n, long long total, const double* __restrict__ rz,
            const double* __restrict__ pq, const double* __restrict__ p,
            const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r) {
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT) {
        const long long b = g / n;
        const double d = pq[b];
        const double al = d > 0.0 ? rz[b] / d : 0.0;
        x[g] += al * p[g];
        r[g] -= al * q[g];
    }
}

// p = z + beta p with beta_b = rz_new_b / rz_old_b
__global__ void __launch_bounds__(NT)
    k_cg_p(long long n, long long total, const double* __restrict__ rz_new,
           const double* __restrict__ rz_old, const double* __restrict__ z,
           double* __restrict__ p) {
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT) {
        const long long b = g / n;
        const double d = rz_old[b];
        const double be = d > 0.0 ? rz_new[b] / d : 0.0;
        p[g] = z[g] + be * p[g];
    }
}

// out_b = (v_b - v_{b-1}) * s (v_{-1} = 0), s = 1 or per-plane 1/tau applied later
__global__ void __launch_bounds__(NT)
    k_time_diff(long long n, long long total, const double* __restrict__ v,
                double* __restrict__ out) {
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT)
        out[g] = g >= n ? v[g] - v[g - n] : v[g];
}

// out_b = a_b / tau_b
__global__ void __launch_bounds__(NT)
    k_div_planes(long long n, long long total, const double* __restrict__ a,
                 const double* __restrict__ tau, double* __restrict__ out) {
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT)
        out[g] = a[g] / tau[g / n];
}

// b = M prev + tau * load  (solvers.py:171: mass.dot(prev) + tau * load[n])
__global__ void __launch_bounds__(NT)
    k_add_scaled(long long total, const double* __restrict__ mp, double tau,
                 const double* __restrict__ load, double* __restrict__ b) {
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < total;
         g += (long long)gridDim.x * NT)
        b[g] = mp[g] + tau * load[g];
}

int grid_for(long long total) {
    return (int)std::max<long long>(1, std::min<long long>((total + NT - 1) / NT, 148LL * 16));
}

double* scratch(pint_ctx* c, int slot, size_t count) {
    auto& cap = c->ex_cap[slot];
    if (cap < count) {
        if (c->ex_buf[slot]) cudaFree(c->ex_buf[slot]);
        c->ex_buf[slot] = nullptr;
        PINT_CUDA_CHECK(cudaMalloc(&c->ex_buf[slot], count * sizeof(double) + 16));
        cap = count;
    }
    return c->ex_buf[slot];
}

}  // namespace

void st_apply(pint_ctx* c, const double* tab, int stride, const int* sid, const double* scale,
              long long planes, const double* x, const double* base, double* y) {
    const long long total = planes * (long long)c->n;
    if (c->dims == 2)
        k_st_apply<2><<<grid_for(total), NT, 0, c->stream>>>(c->m, planes, tab, stride, sid,
                                                             scale, x, base, y);
    else
        k_st_apply<3><<<grid_for(total), NT, 0, c->stream>>>(c->m, planes, tab, stride, sid,
                                                             scale, x, base, y);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

static void plane_dot(pint_ctx* c, long long planes, const double* a, const double* w,
                      double* out) {
    k_plane_dot<<<(unsigned)planes, NT, 0, c->stream>>>(c->n, a, w, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
}

// Solve S_b x_b = rhs_b on planes b < planes of multigrid set `which` (level-0
// rows of its tables are the operators, sid the per-plane set index) by
// V-cycle-preconditioned CG.  x may alias nothing else.  Returns the number
// of iterations; throws PINT_NOT_SPD on a non-positive curvature.
int spd_solve(pint_ctx* c, int which, long long planes, const double* rhs, double* x,
              double tol, int max_iter, double* rel_out) {
    MgSet& s = c->mg[which];
    if (!s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    const int stride = c->dims == 2 ? PINT_TW : 28;
    const long long n = c->n, total = planes * n;
    double* r = scratch(c, 0, total);
    double* z = scratch(c, 1, total);
    double* p = scratch(c, 2, total);
    double* q = scratch(c, 3, total);
    double* sc = scratch(c, 4, 5 * (size_t)planes);
    double *rz = sc, *rzn = sc + planes, *pq = sc + 2 * planes, *rr = sc + 3 * planes,
           *bb = sc + 4 * planes;
    const size_t bytes = total * sizeof(double);
    PINT_CUDA_CHECK(cudaMemcpyAsync(r, rhs, bytes, cudaMemcpyDeviceToDevice, c->stream));
    PINT_CUDA_CHECK(cudaMemsetAsync(x, 0, bytes, c->stream));
    plane_dot(c, planes, rhs, rhs, bb);
    std::vector<double> hbb(planes), hrr(planes);
    PINT_CUDA_CHECK(cudaMemcpyAsync(hbb.data(), bb, planes * sizeof(double),
                                    cudaMemcpyDeviceToHost, c->stream));
    vcycle(c, which, (int)planes, r, z, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
    PINT_CUDA_CHECK(cudaMemcpyAsync(p, z, bytes, cudaMemcpyDeviceToDevice, c->stream));
    plane_dot(c, planes, r, z, rz);
    const int g = grid_for(total);
    double worst = 1.0;
    int it = 0;
    double prev = HUGE_VAL;
    int stall = 0;
    for (it = 1; it <= max_iter; ++it) {
        st_apply(c, s.tab, stride, s.sid, nullptr, planes, p, nullptr, q);
        plane_dot(c, planes, p, q, pq);
        k_cg_xr<<<g, NT, 0, c->stream>>>(n, total, rz, pq, p, q, x, r);
        PINT_LAUNCHED(c);
        plane_dot(c, planes, r, r, rr);
        PINT_CUDA_CHECK(cudaMemcpyAsync(hrr.data(), rr, planes * sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        worst = 0.0;
        for (long long b = 0; b < planes; ++b) {
            if (!std::isfinite(hrr[b])) pint_throw(PINT_NOT_SPD, "exact solve diverged: operator is not SPD");
            if (hbb[b] > 0.0) worst = std::max(worst, std::sqrt(hrr[b] / hbb[b]));
        }
        if (worst <= tol) break;
        // stagnation at the rounding floor: no 10 % gain over 3 iterations
        if (worst > 0.9 * prev) {
            if (++stall >= 3) break;
        } else {
            stall = 0;
            prev = worst;
        }
        vcycle(c, which, (int)planes, r, z, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        plane_dot(c, planes, r, z, rzn);
        k_cg_p<<<g, NT, 0, c->stream>>>(n, total, rzn, rz, z, p);
        PINT_LAUNCHED(c);
        std::swap(rz, rzn);
    }
    PINT_CUDA_CHECK(cudaGetLastError());
    if (rel_out) *rel_out = worst;
    return std::min(it, max_iter);
}

// u_n = (M + tau_n A_n)^{-1} (M u_{n-1} + tau_n load_n), n = 0..N-1, with the
// EULER multigrid set; load / u0 / out are device arrays ([N][n], [n], [N][n])
int sequential_euler(pint_ctx* c, const double* load, const double* u0, double* out,
                     double tol, int max_iter, double* worst_rel) {
    MgSet& s = c->mg[PINT_MG_EULER];
    if (!s.ready) pint_throw(PINT_INPUT, "EULER multigrid set not configured");
    const long long n = c->n;
    double* b = scratch(c, 5, n);
    double* mp = scratch(c, 6, n);
    int* const sid0 = s.sid;
    int most = 0;
    double worst = 0.0;
    try {
        for (int t = 0; t < c->N; ++t) {
            const double* prev = t == 0 ? u0 : out + (long long)(t - 1) * n;
            st_apply(c, c->d_mass, 0, nullptr, nullptr, 1, prev, nullptr, mp);
            k_add_scaled<<<grid_for(n), NT, 0, c->stream>>>(n, mp, c->h_steps[t],
                                                             load + (long long)t * n, b);
            PINT_LAUNCHED(c);
            s.sid = sid0 + t;  // the single plane solved uses step t's operator set
            double rel = 0.0;
            most = std::max(most, spd_solve(c, PINT_MG_EULER, 1, b, out + (long long)t * n, tol,
                                            max_iter, &rel));
            worst = std::max(worst, rel);
        }
    } catch (...) {
        s.sid = sid0;
        throw;
    }
    s.sid = sid0;
    if (worst_rel) *worst_rel = worst;
    return most;
}

// S-bilinear form s(v, v) of a device block vector (operators.py:155-183)
double s_norm_sq(pint_ctx* c, const double* v, double tol, int max_iter, int* iters) {
    const long long n = c->n, N = c->N, total = N * n;
    double* dv = scratch(c, 7, total);
    double* t1 = scratch(c, 8, total);
    double* sol = scratch(c, 9, total);
    double* pd = scratch(c, 10, 4 * (size_t)N);
    const int g = grid_for(total);
    std::vector<double> h(4 * N);
    // energy: sum v . (tau_n A_n v_n)
    launch_timeop(c, OP_ABD, v, nullptr, nullptr, t1);
    plane_dot(c, N, v, t1, pd);
    // jump: v_N . M v_N + sum dv . M dv
    k_time_diff<<<g, NT, 0, c->stream>>>(n, total, v, dv);
    PINT_LAUNCHED(c);
    st_apply(c, c->d_mass, 0, nullptr, nullptr, N, dv, nullptr, t1);  // M dv
    plane_dot(c, N, dv, t1, pd + N);
    st_apply(c, c->d_mass, 0, nullptr, nullptr, 1, v + (N - 1) * n, nullptr, sol);
    plane_dot(c, 1, v + (N - 1) * n, sol, pd + 2 * N);
    // dual: sum tau_n g_n . A_n^{-1} g_n, g_n = M dv_n / tau_n
    k_div_planes<<<g, NT, 0, c->stream>>>(n, total, t1, c->d_steps, dv);
    PINT_LAUNCHED(c);
    const int it = spd_solve(c, PINT_MG_ATILDE, N, dv, sol, tol, max_iter, nullptr);
    if (iters) *iters = it;
    plane_dot(c, N, dv, sol, pd + 3 * N);
    PINT_CUDA_CHECK(cudaMemcpyAsync(h.data(), pd, 4 * N * sizeof(double), cudaMemcpyDeviceToHost,
                                    c->stream));
    PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    double energy = 0.0, jump = h[2 * N], dual = 0.0;
    for (long long b = 0; b < N; ++b) {
        energy += h[b];
        jump += h[N + b];
        dual += c->h_steps[b] * h[3 * N + b];
    }
    return dual + energy + jump;
}

// x_b = A_n^{-1} rhs_b / tau_n  (exact A_bd^{-1}, operators.py:113-122)
int abd_inverse(pint_ctx* c, const double* rhs, double* out, double tol, int max_iter) {
    const long long n = c->n, total = (long long)c->N * n;
    double* t = scratch(c, 8, total);
    const int it = spd_solve(c, PINT_MG_ATILDE, c->N, rhs, t, tol, max_iter, nullptr);
    k_div_planes<<<grid_for(total), NT, 0, c->stream>>>(n, total, t, c->d_steps, out);
    PINT_LAUNCHED(c);
    PINT_CUDA_CHECK(cudaGetLastError());
    return it;
}

void exact_free(pint_ctx* c) {
    for (int i = 0; i < PINT_EX_BUFS; ++i) {
        if (c->ex_buf[i]) cudaFree(c->ex_buf[i]);
        c->ex_buf[i] = nullptr;
        c->ex_cap[i] = 0;
    }
}

}  // namespace pint
