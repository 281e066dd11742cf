// Internal declarations shared by the libpint translation units.
//
// Layout conventions (SURVEY.md 7 / DESIGN.md "Data layout"):
//   * a block vector is a time-major slab double[N][n], n = m*m (2D), the
//     C-order (N, dim) array of the reference (linalg.py:1-6);
//   * a spatial plane is row-major m x m, x fastest (problems.py:133-135);
//   * stencils are 9 coefficients in CSR column order of an interior row
//     (SW, S, SE, W, C, E, NW, N, NE), absent entries 0;  the CSR row sum is
//     evaluated in exactly that order, starting from 0, without FMA
//     contraction (the library is compiled with -fmad=false), which makes
//     every stencil / multigrid result bit-identical to scipy's csr_matvec
//     on the same coefficients (tests/test_gpu_parity.py).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "pint.h"

#define PINT_S2 9   // 2D stencil size
#define PINT_TW 10  // table row: 9 coefficients + dinv
#define PINT_FSEP_MAX 3  // terms of a separable stiffness family (pint_field_separable)
#define PINT_EX_BUFS 11  // work buffers of the diagnostic exact solves (exact_solve.cu)

struct PintFail {
    int code;
    std::string msg;
};

[[noreturn]] void pint_throw(int code, const std::string& msg);
void pint_check_cuda(cudaError_t e, const char* what);

#define PINT_CUDA_CHECK(x) pint_check_cuda((x), #x)

// epilogues of the finest post-smoothing kernel of a V-cycle
enum PostEpi : int {
    EPI_PLAIN = 0,      // out = x
    EPI_DIV_TAU = 1,    // out = x / tau_n                (solvers.py:147)
    EPI_UZAWA_P = 2,    // dp = x/tau_n; out = pin + dp; acc += b*dp   (solvers.py:225-226,233)
    EPI_DOT_TAU = 3,    // dp = x/tau_n; acc += b*dp, nothing stored (ref norm, solvers.py:212-214)
    EPI_SCALE = 4,      // out = s*x                      (schur.py:73)
    EPI_SCALE_DOT = 5,  // w = s*x; out = w; acc += aux*w (mode-space form of sum z.y)
    EPI_SCALE_DOTONLY = 6,  // w = s*x; acc += aux*w, nothing stored (ref norm)
};

struct MgSet {
    int levels = 0;
    std::vector<int> m;       // interior points per side, fine to coarse
    int n_sets = 0;
    double* tab = nullptr;    // device [levels][n_sets][PINT_TW]
    int* sid = nullptr;       // device [B]
    std::vector<int> shape;   // per level: which stencil positions can be non-zero
    std::vector<uint32_t> shape3;  // 3D: per level, 27-bit union of non-zero positions
    int cycles = 1, smooth = 1;    // spatial.py:148-169; != 1 runs mg_generic.cu
    bool ready = false;
};

// field-mode (per-point coefficient) multigrid set: coarse Galerkin rows of
// every set on every level >= 1 (field2d.cu)
struct FieldMg {
    int levels = 0;
    std::vector<int> m;
    double damping = 0.0;
    std::vector<double*> f9;  // [l] device [N][9][m_l^2], l >= 1 (f9[0] unused); separable: [sep][9][m_l^2]
    double* d_mu = nullptr;   // H~: per-mode weights [N]
    int sep = 0;              // separable form: number of term tables (0: per-set rows)
    double* d_sc = nullptr;   // separable: term weights [N][sep] (A~: the family's; H~: (mu_k, tau_ref), owned)
    bool own_sc = false;
    bool ready = false;
};

struct DstPlan {
    int N = 0;
    bool fast = false;        // power of two -> FFT path
    double2* tw = nullptr;    // e^{-2 pi i j / N}, j < N
    double2* tq = nullptr;    // (cos, sin)(pi k / 2N), k < N
    int* rev = nullptr;       // output position of DFT index k after the DIF stages
    double* dense = nullptr;  // sin((2k-1) n pi / 2N), k-major (non power of two)
    int radix2_first = 0;
    int pairs = 0;            // column pairs per CTA
    int reg_lg = 0;           // log2 N when the register-radix kernel runs (0: k_dst_fft)
    int reg_p = 0;            // its column pairs per CTA
    double2* twp[3] = {nullptr, nullptr, nullptr};  // its per-pass twiddle tables
};

// kernel families timed individually in profiling mode (pint_profile)
enum KernelId : int {
    K_TIMEOP_K = 0, K_TIMEOP_KT, K_TIMEOP_ABD, K_TIMEOP_R1, K_TIMEOP_Z, K_FOLD, K_AREF,
    K_MG_PRE_FINE, K_MG_PRE_COARSE, K_MG_POST_FINE, K_MG_POST_COARSE,
    K_DST_T, K_DST, K_REDUCE, K_MG_TAIL, K_COUNT
};

struct KStat {
    double ms = 0.0;
    double bytes = 0.0;   // algorithmic bytes
    long long count = 0;
};

struct ProfRec {
    int kid;
    double bytes;
    cudaEvent_t a, b;
};

namespace pint {
struct HostXfer;
}

struct pint_ctx {
    int dev = 0, rank = 0, world = 1;
    int exact = 0;  // 1: bit-exact (no FMA) band kernels; 0: FMA-contracted (pint_set_arith)
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;  // created by the context; `stream` may be a caller's
    std::string err;
    long long launches = 0;
    pint::HostXfer* xfer = nullptr;  // pinned staging for host block vectors (hostcopy.cu)

    // problem
    int dims = 0, m = 0, n = 0, N = 0;
    // time partition (pint_set_partition): this context owns global steps
    // [n0, n0 + N) of N_global; neighbouring ranks' ghost planes sit at local
    // plane -1 / N of the u and p slabs passed to the residual kernels
    int n0 = 0, N_global = 0;
    bool has_prev = false, has_next = false;
    double tau_ref = 0.0;
    int n_a = 0;
    std::vector<double> h_steps, h_mass, h_ast, h_aref;
    double* d_steps = nullptr;   // [N]
    double* d_rsteps = nullptr;  // [N] 1/tau_n when tau_n is a power of two (x/tau == x*(1/tau) exactly), else 0
    double* d_mass = nullptr;    // [9]
    double* d_ast = nullptr;     // [n_a][9]
    int* d_asid = nullptr;       // [N]
    double* d_ascale = nullptr;  // [N]
    double* d_aref = nullptr;    // [9]
    bool problem_ready = false;

    MgSet mg[3];  // PINT_MG_ATILDE, PINT_MG_HTILDE, PINT_MG_EULER
    // field mode (pint_field_set / pint_field_assemble): per-point stiffness
    bool field = false;
    double* d_fa = nullptr;      // [N][3][n] compact fine A_n (centre, east, north)
    double* d_fref = nullptr;    // [3][n] compact A_ref
    // separable family A_n = sum_r sc[n][r] A(w_r) (pint_field_separable): the
    // R compact term fields and the weights replace d_fa
    int fsep_R = 0;
    double* d_fsep = nullptr;    // [R][3][n]
    double* d_fsc = nullptr;     // [N][R]
    std::vector<double> h_fsc;
    double* d_unit = nullptr;    // {1.0, 0.0}
    bool fref_ready = false;
    FieldMg fmg[2];
    double* d_ft = nullptr;      // [N][n] fine-level V-cycle work slab
    std::vector<double*> lev_t;  // coarse-level work planes
    DstPlan dst;
    DstPlan dst_raw;   // plan of the problem-free pint_dst_raw entry

    // level work buffers (levels >= 1): rhs and solution, N planes each
    std::vector<double*> lev_b, lev_x;
    std::vector<double*> gen_scratch;  // mg_generic.cu work vectors
    std::vector<size_t> gen_cap;
    std::vector<size_t> lev_cap;

    // slabs [N][n]
    double *d_f = nullptr, *d_p = nullptr, *d_u = nullptr;
    double *d_r1 = nullptr, *d_z = nullptr, *d_w1 = nullptr, *d_w2 = nullptr;
    double *d_stage_in = nullptr, *d_stage_out = nullptr, *d_vec = nullptr;
    double *d_t3a = nullptr, *d_t3b = nullptr;  // 3D multigrid work slabs
    double *d_mu3 = nullptr, *d_mp3 = nullptr;  // 3D: M u, M p of planes -1..N (ops3d.cu)
    const double* mu3_src = nullptr;            // u that d_mu3 was computed from
    bool mu3_trust = false;                     // caller guarantees u unchanged since (Uzawa step)
    size_t t3_cap = 0;

    // reductions
    double* d_part = nullptr;    // partial sums
    size_t part_cap = 0;
    double* d_acc = nullptr;     // [4] final sums
    double* h_acc = nullptr;     // pinned [4]

    double ref = 0.0;
    bool uz_ready = false;
    // CUDA graph of one Uzawa step (pint_uzawa_step), captured on the second
    // step and replayed while its key (omega, timing, stream) holds
    cudaGraphExec_t g_exec = nullptr;
    double g_omega = 0.0;
    bool g_timing = false;
    cudaStream_t g_stream = nullptr;
    long long g_launches = 0;
    int uz_steps = 0;

    // phase timing
    bool timing = false;
    cudaEvent_t ev[8] = {};
    double ms_dst = 0, ms_mg = 0, ms_other = 0;

    // per-kernel profiling (events around every launch)
    bool profile = false;
    std::vector<cudaEvent_t> prof_pool;
    std::vector<ProfRec> prof_open;
    KStat kstat[K_COUNT];

    // diagnostic exact solves (exact_solve.cu)
    double* ex_buf[PINT_EX_BUFS] = {};
    size_t ex_cap[PINT_EX_BUFS] = {};
};

// RAII event pair around one launch when ctx->profile is on
struct ProfScope {
    pint_ctx* c;
    ProfRec r{};
    bool on;
    ProfScope(pint_ctx* ctx, int kid, double bytes);
    ~ProfScope();
};
void pint_prof_drain(pint_ctx* c);   // after a stream sync: accumulate elapsed times

// ---- kernels / launchers (all on ctx->stream) ------------------------------
namespace pint {

enum TimeOp : int { OP_K = 0, OP_KT = 1, OP_ABD = 2, OP_R1 = 3, OP_Z = 4, OP_MASS0 = 5 };

// time-global stencil operators (stencil_ops.cu)
void launch_timeop(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                   double* out);
void launch_fold_rhs(pint_ctx* c, const double* load, const double* u_init, double* f);
void launch_aref(pint_ctx* c, const double* in, double* out, int count);
void launch_axpy(pint_ctx* c, double* u, const double* y, double omega, long long count);
void launch_lincomb(pint_ctx* c, double* out, const double* x0, double a1, const double* x1,
                    double a2, const double* x2, double sc, bool use_sc, long long count);
void launch_dot(pint_ctx* c, const double* a, const double* b, long long count, int slot);
// TMA band versions (timeop_band.cu), used for 64 <= m <= 512
bool band_timeop_supported(const pint_ctx* c);
void launch_band_timeop(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                        double* out);
void launch_band_apply(pint_ctx* c, const double* st_dev, const double* st_host, const double* in,
                       double* out, int count);

// multigrid (mg.cu)
// V-cycle over planes [0,count) of set `which`; finest post kernel uses `epi`.
// pin: EPI_UZAWA_P input p;  aux: EPI_SCALE_DOT partner vector; acc_slot: d_acc index
// aref_in: the right-hand side is A_ref * b, formed inside the finest pre / post
// kernels (only when vcycle_aref_fusable)
void vcycle(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
            double scale, const double* pin, const double* aux, int acc_slot,
            bool aref_in = false);
bool vcycle_aref_fusable(const pint_ctx* c, int which);
void mg_compute_shapes(MgSet& set, const double* tables);
// The 2D band kernels (timeop_band.cu, mg_band.cu) are compiled twice
// (Makefile): `exact` with -fmad=false (every row sum bit-identical to
// scipy's CSR products) and `fast` with FMA contraction (<= 1e-15 relative
// per operator; the default arithmetic, pint_set_arith).  The functions above
// dispatch on pint_ctx::exact (variant.cu).
#define PINT_VARIANT_API                                                                          \
    bool band_timeop_supported(const pint_ctx* c);                                                \
    void launch_band_timeop(pint_ctx* c, int op, const double* u, const double* p,               \
                            const double* f, double* out);                                       \
    void launch_band_apply(pint_ctx* c, const double* st_dev, const double* st_host,             \
                           const double* in, double* out, int count);                            \
    void vcycle(pint_ctx* c, int which, int count, const double* b, double* out, int epi,         \
                double scale, const double* pin, const double* aux, int acc_slot, bool aref_in); \
    bool vcycle_aref_fusable(const pint_ctx* c, int which);                                      \
    void mg_compute_shapes(MgSet& set, const double* tables);
namespace exact {
PINT_VARIANT_API
}
namespace fast {
PINT_VARIANT_API
}
// general cycles / smooth_steps (mg_generic.cu)
bool vcycle_is_generic(const pint_ctx* c, int which);
void vcycle_generic(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
                    double scale, const double* pin, const double* aux, int acc_slot);
// 3D (ops3d.cu)
void launch_timeop3(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                    double* out);
void launch_apply3(pint_ctx* c, const double* st, const double* in, double* out, int count);
void launch_fold3(pint_ctx* c, const double* load, const double* u0, double* f);
void vcycle3(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
             double scale, const double* pin, const double* aux, int acc_slot);

// field mode, 2D per-point stiffness (field2d.cu)
void field_assemble(pint_ctx* c, int step0, int count, const double* w_dev, double* dst = nullptr);
void field_sep_step(pint_ctx* c, int step, double* out);  // out[3][n] = compact field of one step of a separable family
void field_galerkin(pint_ctx* c, int which);
void launch_timeop_field(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                         double* out);
void launch_aref_field(pint_ctx* c, const double* in, double* out, int count);
void vcycle_field(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
                  double scale, const double* pin, const double* aux, int acc_slot);

// sine transforms (dst.cu)
void dst_plan_build(DstPlan& d, int N);
void dst_plan_free(DstPlan& d);
// kind 0..3 as in pint_dst; out = beta*base + alpha*T(in) when base != nullptr
void dst_apply(pint_ctx* c, int kind, const double* in, double* out, const double* base,
               double alpha);
// same on an arbitrary (N, ncols) slab with plan d
// host <-> device block-vector copies through pinned multi-threaded staging (hostcopy.cu)
void copy_h2d(pint_ctx* c, void* dev, const void* host, size_t bytes);
void copy_d2h(pint_ctx* c, void* host, const void* dev, size_t bytes);  // synchronous
void host_xfer_free(pint_ctx* c);
void host_prefault_async(pint_ctx* c, void* p, size_t bytes);
void host_prefault_join(pint_ctx* c);
void dst_run(pint_ctx* c, const DstPlan& d, int kind, long long ncols, const double* in,
             double* out, const double* base, double alpha);

// diagnostic-mode exact solves (exact_solve.cu): multigrid-preconditioned CG
void st_apply(pint_ctx* c, const double* tab, int stride, const int* sid, const double* scale,
              long long planes, const double* x, const double* base, double* y);
int spd_solve(pint_ctx* c, int which, long long planes, const double* rhs, double* x,
              double tol, int max_iter, double* rel_out);
int sequential_euler(pint_ctx* c, const double* load, const double* u0, double* out,
                     double tol, int max_iter, double* worst_rel);
double s_norm_sq(pint_ctx* c, const double* v, double tol, int max_iter, int* iters);
int abd_inverse(pint_ctx* c, const double* rhs, double* out, double tol, int max_iter);
void exact_free(pint_ctx* c);

// reductions (stencil_ops.cu)
void reduce_partials(pint_ctx* c, int nparts, int slot);
void ensure_partials(pint_ctx* c, size_t nparts);

}  // namespace pint

#define PINT_LAUNCHED(c) ((c)->launches++)
