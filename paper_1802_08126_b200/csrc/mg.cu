// Batched geometric-multigrid V-cycle over all time steps / DST modes.
//
// Reference: MgVCycleSolver._vcycle / apply (spatial.py:148-169) with the
// 2D hierarchy of build_mg_hierarchy (spatial.py:100-113): one pre- and one
// post-smoothing damped-Jacobi sweep (dinv = damping/diag, spatial.py:142),
// residual restriction by P^T (unscaled bilinear full weighting), bilinear
// prolongation P = kron(P1, P1) (spatial.py:75-84,110), Galerkin coarse
// operators (9-point stencils, supplied per level and operator set by the
// host), and a 1x1 direct solve b/a on the coarsest grid (SpdFactor,
// spatial.py:143,149-150).
//
// One launch per level and direction covers every plane of the batch
// (grid.z = plane): the N independent per-step (A~) or per-mode (H~) solves
// of the reference's thread-pool loops (solvers.py:149, schur.py:75) run as
// one kernel.  Each CTA stages its tile of the level's right-hand side (and
// coarse correction) in shared memory with a halo, so pre-smoothing,
// residual and restriction (k_mg_pre) and prolongation plus post-smoothing
// (k_mg_post) are each a single pass over the level.  Operation order
// follows scipy's CSR/CSC matvec exactly (sum from 0 in column order, no FMA),
// so the V-cycle is bit-identical to the reference's.
#include "pint_device.cuh"
#include "pint_internal.cuh"

namespace pint {

constexpr int CX = 32, CY = 8;                   // threads per CTA: 32 x 8
constexpr int PRE_BY = 2 * CY + 3, PRE_BX = 2 * CX + 3;   // rhs tile 19 x 67
constexpr int PRE_RY = 2 * CY + 1, PRE_RX = 2 * CX + 1;   // residual tile 17 x 65
constexpr int PRE_BP = PRE_BX + 1, PRE_RP = PRE_RX + 1;   // pitches
constexpr int POST_Y = CY + 2, POST_X = CX + 2, POST_P = POST_X + 1;  // 10 x 34
constexpr int POST_EY = CY / 2 + 2, POST_EX = CX / 2 + 2, POST_EP = POST_EX + 1;  // 6 x 18

// Pre-smoothing x0 = dinv*b, residual r = b - A x0, restriction b_c = P^T r.
__global__ void __launch_bounds__(CX* CY)
    k_mg_pre(int m, int mc, const double* __restrict__ b, double* __restrict__ bc,
             const double* __restrict__ tab, const int* __restrict__ sid) {
    __shared__ double sb[PRE_BY * PRE_BP];
    __shared__ double sr[PRE_RY * PRE_RP];
    const int plane = blockIdx.z;
    const int tid = threadIdx.y * CX + threadIdx.x;
    const double* tb = tab + (size_t)__ldg(sid + plane) * PINT_TW;
    double ca[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) ca[k] = __ldg(tb + k);
    const double d = __ldg(tb + 9);
    const double* bp = b + (size_t)plane * m * m;
    const int fy0 = 2 * blockIdx.y * CY - 1, fx0 = 2 * blockIdx.x * CX - 1;
    // x0 = dinv*b staged directly (b itself is needed only at the residual points)
    for (int idx = tid; idx < PRE_BY * PRE_BX; idx += CX * CY) {
        const int iy = idx / PRE_BX, ix = idx - iy * PRE_BX;
        const int gy = fy0 + iy, gx = fx0 + ix;
        sb[iy * PRE_BP + ix] =
            (gy >= 0 && gy < m && gx >= 0 && gx < m) ? __ldg(bp + (size_t)gy * m + gx) : 0.0;
    }
    __syncthreads();
    // residual on the 17 x 65 fine points covered by this coarse tile
    for (int idx = tid; idx < PRE_RY * PRE_RX; idx += CX * CY) {
        const int iy = idx / PRE_RX, ix = idx - iy * PRE_RX;
        const int gy = fy0 + 1 + iy, gx = fx0 + 1 + ix;
        double r = 0.0;
        if (gy < m && gx < m) {
            const double* s0 = sb + iy * PRE_BP + ix;
            const double* s1 = s0 + PRE_BP;
            const double* s2 = s1 + PRE_BP;
            double a = ca[0] * (d * s0[0]);
            a = a + ca[1] * (d * s0[1]);
            a = a + ca[2] * (d * s0[2]);
            a = a + ca[3] * (d * s1[0]);
            a = a + ca[4] * (d * s1[1]);
            a = a + ca[5] * (d * s1[2]);
            a = a + ca[6] * (d * s2[0]);
            a = a + ca[7] * (d * s2[1]);
            a = a + ca[8] * (d * s2[2]);
            r = s1[1] - a;
        }
        sr[iy * PRE_RP + ix] = r;
    }
    __syncthreads();
    const int X = blockIdx.x * CX + threadIdx.x, Y = blockIdx.y * CY + threadIdx.y;
    if (X < mc && Y < mc) {
        const double* r0 = sr + (2 * threadIdx.y) * PRE_RP + 2 * threadIdx.x;
        const double* r1 = r0 + PRE_RP;
        const double* r2 = r1 + PRE_RP;
        // P^T r: csc_matvec order = ascending fine index (row-major)
        double s = 0.25 * r0[0];
        s = s + 0.5 * r0[1];
        s = s + 0.25 * r0[2];
        s = s + 0.5 * r1[0];
        s = s + 1.0 * r1[1];
        s = s + 0.5 * r1[2];
        s = s + 0.25 * r2[0];
        s = s + 0.5 * r2[1];
        s = s + 0.25 * r2[2];
        bc[(size_t)plane * mc * mc + (size_t)Y * mc + X] = s;
    }
}

// Prolongation x = x0 + P e and post-smoothing x += dinv*(b - A x), with the
// finest-level epilogues of A~^{-1}, the Uzawa p-update and H~^{-1}.
struct PostArgs {
    int m, mc;
    const double* b;
    const double* ec;       // coarse correction, or coarse rhs when coarse_direct
    int coarse_direct;      // e = b_c / a_c (1x1 coarsest solve)
    const double* tab;      // this level [n_sets][10]
    const double* tabc;     // coarse level [n_sets][10] (centre used when direct)
    const int* sid;
    double* out;
    int epi;
    double scale;
    const double* steps;
    const double* pin;
    const double* aux;
    double* part;
};

__device__ __forceinline__ void prolong_terms(int f, int& j0, double& w0, int& j1, double& w1,
                                              int& cnt) {
    if (f & 1) {
        j0 = (f - 1) >> 1;
        w0 = 1.0;
        cnt = 1;
    } else {
        j0 = (f >> 1) - 1;
        w0 = 0.5;
        j1 = f >> 1;
        w1 = 0.5;
        cnt = 2;
    }
}

__global__ void __launch_bounds__(CX* CY) k_mg_post(PostArgs a) {
    __shared__ double sb[POST_Y * POST_P];
    __shared__ double sx[POST_Y * POST_P];
    __shared__ double se[POST_EY * POST_EP];
    const int m = a.m, mc = a.mc;
    const int plane = blockIdx.z;
    const int tid = threadIdx.y * CX + threadIdx.x;
    const int set = __ldg(a.sid + plane);
    const double* tb = a.tab + (size_t)set * PINT_TW;
    double ca[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) ca[k] = __ldg(tb + k);
    const double d = __ldg(tb + 9);
    const int y0 = blockIdx.y * CY, x0 = blockIdx.x * CX;
    const int cy0 = y0 / 2 - 1, cx0 = x0 / 2 - 1;
    const double* ep = a.ec + (size_t)plane * mc * mc;
    const double acoarse = a.coarse_direct ? __ldg(a.tabc + (size_t)set * PINT_TW + 4) : 1.0;
    for (int idx = tid; idx < POST_EY * POST_EX; idx += CX * CY) {
        const int iy = idx / POST_EX, ix = idx - iy * POST_EX;
        const int gy = cy0 + iy, gx = cx0 + ix;
        double v = 0.0;
        if (gy >= 0 && gy < mc && gx >= 0 && gx < mc) {
            v = __ldg(ep + (size_t)gy * mc + gx);
            if (a.coarse_direct) v = v / acoarse;
        }
        se[iy * POST_EP + ix] = v;
    }
    const double* bp = a.b + (size_t)plane * m * m;
    for (int idx = tid; idx < POST_Y * POST_X; idx += CX * CY) {
        const int iy = idx / POST_X, ix = idx - iy * POST_X;
        const int gy = y0 - 1 + iy, gx = x0 - 1 + ix;
        sb[iy * POST_P + ix] =
            (gy >= 0 && gy < m && gx >= 0 && gx < m) ? __ldg(bp + (size_t)gy * m + gx) : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < POST_Y * POST_X; idx += CX * CY) {
        const int iy = idx / POST_X, ix = idx - iy * POST_X;
        const int gy = y0 - 1 + iy, gx = x0 - 1 + ix;
        double xv = 0.0;
        if (gy >= 0 && gy < m && gx >= 0 && gx < m) {
            int jy0, jy1 = 0, ny, jx0, jx1 = 0, nx;
            double wy0, wy1 = 0.0, wx0, wx1 = 0.0;
            prolong_terms(gy, jy0, wy0, jy1, wy1, ny);
            prolong_terms(gx, jx0, wx0, jx1, wx1, nx);
            jy0 -= cy0;
            jy1 -= cy0;
            jx0 -= cx0;
            jx1 -= cx0;
            // P e: csr_matvec over ascending coarse index (Jy major, Jx minor)
            double pe = (wy0 * wx0) * se[jy0 * POST_EP + jx0];
            if (nx == 2) pe = pe + (wy0 * wx1) * se[jy0 * POST_EP + jx1];
            if (ny == 2) {
                pe = pe + (wy1 * wx0) * se[jy1 * POST_EP + jx0];
                if (nx == 2) pe = pe + (wy1 * wx1) * se[jy1 * POST_EP + jx1];
            }
            xv = d * sb[iy * POST_P + ix] + pe;
        }
        sx[iy * POST_P + ix] = xv;
    }
    __syncthreads();
    const int gy = y0 + threadIdx.y, gx = x0 + threadIdx.x;
    const bool inside = gy < m && gx < m;
    double acc = 0.0;
    if (inside) {
        const int ly = threadIdx.y + 1, lx = threadIdx.x + 1;
        const double bv = sb[ly * POST_P + lx];
        const double xv = sx[ly * POST_P + lx];
        const double r = bv - stencil9_smem<POST_P>(ca, sx, ly, lx);
        const double xn = xv + d * r;
        const size_t gi = (size_t)plane * m * m + (size_t)gy * m + gx;
        switch (a.epi) {
            case EPI_PLAIN:
                a.out[gi] = xn;
                break;
            case EPI_DIV_TAU:
                a.out[gi] = xn / __ldg(a.steps + plane);
                break;
            case EPI_UZAWA_P: {
                const double dp = xn / __ldg(a.steps + plane);
                a.out[gi] = __ldg(a.pin + gi) + dp;
                acc = bv * dp;
                break;
            }
            case EPI_DOT_TAU: {
                const double dp = xn / __ldg(a.steps + plane);
                acc = bv * dp;
                break;
            }
            case EPI_SCALE:
                a.out[gi] = a.scale * xn;
                break;
            case EPI_SCALE_DOT: {
                const double w = a.scale * xn;
                a.out[gi] = w;
                acc = __ldg(a.aux + gi) * w;
                break;
            }
            case EPI_SCALE_DOTONLY: {
                const double w = a.scale * xn;
                acc = __ldg(a.aux + gi) * w;
                break;
            }
        }
    }
    if (a.part != nullptr) {
        const double s = block_sum<CX * CY>(acc);
        if (tid == 0)
            a.part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
    }
}

static bool epi_has_dot(int epi) {
    return epi == EPI_UZAWA_P || epi == EPI_DOT_TAU || epi == EPI_SCALE_DOT ||
           epi == EPI_SCALE_DOTONLY;
}

void vcycle(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
            double scale, const double* pin, const double* aux, int acc_slot) {
    MgSet& s = c->mg[which];
    if (!s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
    const int L = s.levels;
    const dim3 blk(CX, CY);
    auto lvl_tab = [&](int l) { return s.tab + (size_t)l * s.n_sets * PINT_TW; };
    // descend: pre-smooth + restrict, level l -> l+1
    const double* bl = b;
    for (int l = 0; l + 1 < L; ++l) {
        const int mf = s.m[l], mcc = s.m[l + 1];
        const dim3 g((mcc + CX - 1) / CX, (mcc + CY - 1) / CY, count);
        {
            ProfScope prof(c, l == 0 ? K_MG_PRE_FINE : K_MG_PRE_COARSE,
                           8.0 * count * ((double)mf * mf + (double)mcc * mcc));
            k_mg_pre<<<g, blk, 0, c->stream>>>(mf, mcc, bl, c->lev_b[l + 1], lvl_tab(l), s.sid);
        }
        PINT_LAUNCHED(c);
        bl = c->lev_b[l + 1];
    }
    PINT_CUDA_CHECK(cudaGetLastError());
    // ascend: prolong + post-smooth, level l+1 -> l
    for (int l = L - 2; l >= 0; --l) {
        PostArgs a{};
        a.m = s.m[l];
        a.mc = s.m[l + 1];
        a.b = (l == 0) ? b : c->lev_b[l];
        a.coarse_direct = (l + 1 == L - 1);
        a.ec = a.coarse_direct ? c->lev_b[l + 1] : c->lev_x[l + 1];
        a.tab = lvl_tab(l);
        a.tabc = lvl_tab(l + 1);
        a.sid = s.sid;
        a.out = (l == 0) ? out : c->lev_x[l];
        a.epi = (l == 0) ? epi : EPI_PLAIN;
        a.scale = scale;
        a.steps = c->d_steps;
        a.pin = pin;
        a.aux = aux;
        const dim3 g((a.m + CX - 1) / CX, (a.m + CY - 1) / CY, count);
        const bool dot = (l == 0) && epi_has_dot(epi);
        if (dot) {
            ensure_partials(c, (size_t)g.x * g.y * g.z);
            a.part = c->d_part;
        }
        {
            const double fine = (double)a.m * a.m, coarse = (double)a.mc * a.mc;
            double words = fine + coarse;                       // b in, coarse correction in
            if (a.epi != EPI_DOT_TAU && a.epi != EPI_SCALE_DOTONLY) words += fine;  // x out
            if (a.epi == EPI_UZAWA_P) words += fine;            // p in
            if (a.epi == EPI_SCALE_DOT || a.epi == EPI_SCALE_DOTONLY) words += fine;  // aux in
            ProfScope prof(c, l == 0 ? K_MG_POST_FINE : K_MG_POST_COARSE, 8.0 * count * words);
            k_mg_post<<<g, blk, 0, c->stream>>>(a);
        }
        PINT_LAUNCHED(c);
        if (dot) reduce_partials(c, (int)(g.x * g.y * g.z), acc_slot);
    }
    PINT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pint
