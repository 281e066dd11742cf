// C ABI of libpint.so (include/pint.h): context, problem upload, operator
// entry points and the device-resident Uzawa driver.
//
// The Uzawa iteration (uzawa_solve, solvers.py:177-264) runs as this launch
// sequence per iteration, all on the context stream, state resident in HBM:
//   r1 = (K u - A p) - f                        k_timeop<OP_R1>
//   p  = p + V_A(r1)/tau ; s1 = sum r1.dp       V-cycle (A~ set), fused epilogue
//   z  = (f - K^T p) - ((K u + K^T u) + A u)    k_timeop<OP_Z>
//   zh = S z                                    DST^T   (dst.py:86-93)
//   y1 = V_H(zh) ; b2 = A_ref y1                V-cycle (H~ set), k_aref
//   w  = (2 tau_ref/N) V_H(b2) ; s2 = sum zh.w  V-cycle, fused epilogue
//   u  = u + omega * S^T w                      DST, fused axpy epilogue
//   res = sqrt(max(s1 + s2, 0))                 (sum z.y == sum zh.w, S orthogonal pairing)
// i.e. y = H~^{-1} z is never materialised in time space and dp is never stored.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include <stdexcept>
#include <string>

#include "pint_internal.cuh"

void pint_throw(int code, const std::string& msg) { throw PintFail{code, msg}; }

void pint_check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        pint_throw(PINT_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static const char* kKernelNames[K_COUNT] = {
    "timeop_K", "timeop_Kt", "timeop_Abd", "timeop_r1", "timeop_z", "fold_rhs", "aref",
    "mg_pre_fine", "mg_pre_coarse", "mg_post_fine", "mg_post_coarse",
    "dst_inverse_transpose", "dst_inverse", "reduce", "mg_tail"};

ProfScope::ProfScope(pint_ctx* ctx, int kid, double bytes) : c(ctx), on(ctx->profile) {
    if (!on) return;
    if (c->prof_pool.size() < 2) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            PINT_CUDA_CHECK(cudaEventCreate(&e));
            c->prof_pool.push_back(e);
        }
    }
    r.kid = kid;
    r.bytes = bytes;
    r.a = c->prof_pool.back();
    c->prof_pool.pop_back();
    r.b = c->prof_pool.back();
    c->prof_pool.pop_back();
    PINT_CUDA_CHECK(cudaEventRecord(r.a, c->stream));
}

ProfScope::~ProfScope() {
    if (!on) return;
    cudaEventRecord(r.b, c->stream);
    c->prof_open.push_back(r);
}

void pint_prof_drain(pint_ctx* c) {
    for (ProfRec& r : c->prof_open) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            c->kstat[r.kid].ms += ms;
            c->kstat[r.kid].bytes += r.bytes;
            c->kstat[r.kid].count += 1;
        }
        c->prof_pool.push_back(r.a);
        c->prof_pool.push_back(r.b);
    }
    c->prof_open.clear();
}

namespace {

template <typename F>
int guarded(pint_ctx* c, F&& f) {
    if (c == nullptr) return PINT_INPUT;
    try {
        PINT_CUDA_CHECK(cudaSetDevice(c->dev));
        f();
        c->err.clear();
        return PINT_OK;
    } catch (const PintFail& e) {
        c->err = e.msg;
        c->mu3_trust = false;
        return e.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        c->mu3_trust = false;
        return PINT_CUDA;
    }
}

bool is_device_ptr(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void dfree(void* p) {
    if (p) cudaFree(p);
}

template <typename T>
T* dalloc(size_t count) {
    T* p = nullptr;
    PINT_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T) + 16));
    return p;
}

template <typename T>
T* upload(pint_ctx* c, const T* h, size_t count) {
    T* d = dalloc<T>(count);
    PINT_CUDA_CHECK(cudaMemcpy(d, h, count * sizeof(T), cudaMemcpyHostToDevice));
    (void)c;
    return d;
}

size_t slab(const pint_ctx* c) { return (size_t)c->N * c->n; }

// Input block vector: device pointer used in place, host pointer staged.
const double* stage_in(pint_ctx* c, const double* p, double* staging, size_t count) {
    if (p == nullptr) pint_throw(PINT_INPUT, "null input");
    if (is_device_ptr(p)) return p;
    pint::copy_h2d(c, staging, p, count * sizeof(double));
    return staging;
}

// any-kind source/destination: device pointers copy on the stream, host
// pointers go through the pinned multi-threaded staging (hostcopy.cu)
void copy_in(pint_ctx* c, double* dev, const double* src, size_t bytes) {
    if (is_device_ptr(src))
        PINT_CUDA_CHECK(cudaMemcpyAsync(dev, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    else
        pint::copy_h2d(c, dev, src, bytes);
}
void copy_out(pint_ctx* c, double* dst, const double* dev, size_t bytes) {
    if (is_device_ptr(dst))
        PINT_CUDA_CHECK(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToDevice, c->stream));
    else
        pint::copy_d2h(c, dst, dev, bytes);
}

struct OutBuf {
    double* dev;
    double* host;
};

OutBuf stage_out(pint_ctx* c, double* p, double* staging) {
    if (p == nullptr) pint_throw(PINT_INPUT, "null output");
    if (is_device_ptr(p)) return {p, nullptr};
    (void)c;
    return {staging, p};
}

void finish_out(pint_ctx* c, const OutBuf& o, size_t count) {
    if (o.host) pint::copy_d2h(c, o.host, o.dev, count * sizeof(double));
    PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    pint_prof_drain(c);
}

void require_problem(pint_ctx* c) {
    if (!c->problem_ready) pint_throw(PINT_INPUT, "problem not set");
}

void free_slabs(pint_ctx* c) {
    double** s[] = {&c->d_f,  &c->d_p,        &c->d_u,         &c->d_r1,  &c->d_z,  &c->d_w1,
                    &c->d_w2, &c->d_stage_in, &c->d_stage_out, &c->d_vec, &c->d_t3a, &c->d_t3b,
                    &c->d_mu3, &c->d_mp3};
    for (double** p : s) {
        dfree(*p);
        *p = nullptr;
    }
    c->t3_cap = 0;
    c->mu3_src = nullptr;
    for (double* p : c->lev_b) dfree(p);
    for (double* p : c->lev_x) dfree(p);
    c->lev_b.clear();
    c->lev_x.clear();
    c->lev_cap.clear();
    for (double* p : c->gen_scratch) dfree(p);
    c->gen_scratch.clear();
    c->gen_cap.clear();
}

void free_field_set(FieldMg& F) {
    for (double* p : F.f9) dfree(p);
    dfree(F.d_mu);
    if (F.own_sc) dfree(F.d_sc);
    F = FieldMg{};
}

void free_field(pint_ctx* c) {
    for (FieldMg& F : c->fmg) free_field_set(F);
    dfree(c->d_fa);
    dfree(c->d_fref);
    dfree(c->d_ft);
    dfree(c->d_fsep);
    dfree(c->d_fsc);
    dfree(c->d_unit);
    for (double* p : c->lev_t) dfree(p);
    c->lev_t.clear();
    c->d_fa = c->d_fref = c->d_ft = c->d_fsep = c->d_fsc = c->d_unit = nullptr;
    c->fsep_R = 0;
    c->h_fsc.clear();
    c->field = false;
    c->fref_ready = false;
}

void graph_reset(pint_ctx* c) {
    if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
    c->g_exec = nullptr;
}

void free_problem(pint_ctx* c) {
    graph_reset(c);
    dfree(c->d_steps);
    dfree(c->d_rsteps);
    c->d_rsteps = nullptr;
    dfree(c->d_mass);
    dfree(c->d_ast);
    dfree(c->d_asid);
    dfree(c->d_ascale);
    dfree(c->d_aref);
    c->d_steps = c->d_mass = c->d_ast = c->d_ascale = c->d_aref = nullptr;
    c->d_asid = nullptr;
    for (MgSet& s : c->mg) {
        dfree(s.tab);
        dfree(s.sid);
        s = MgSet{};
    }
    free_field(c);
    free_slabs(c);
    pint::exact_free(c);
    pint::dst_plan_free(c->dst);
    c->problem_ready = false;
    c->uz_ready = false;
}

// level buffers sized for N planes of every level >= 1 of either set
void ensure_levels(pint_ctx* c, const std::vector<int>& m) {
    if (c->lev_b.size() < m.size()) {
        c->lev_b.resize(m.size(), nullptr);
        c->lev_x.resize(m.size(), nullptr);
        c->lev_cap.resize(m.size(), 0);
    }
    for (size_t l = 1; l < m.size(); ++l) {
        const size_t need = (size_t)c->N * m[l] * m[l] * (c->dims == 3 ? m[l] : 1);
        if (c->lev_cap[l] >= need) continue;
        dfree(c->lev_b[l]);
        dfree(c->lev_x[l]);
        c->lev_b[l] = dalloc<double>(need);
        c->lev_x[l] = dalloc<double>(need);
        c->lev_cap[l] = need;
    }
}

void rec(pint_ctx* c, int i) {
    // External: inside a captured Uzawa step this becomes a real event-record
    // node of the graph (a plain record would only be a capture dependency)
    if (!c->timing) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    PINT_CUDA_CHECK(cudaStreamIsCapturing(c->stream, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        PINT_CUDA_CHECK(cudaEventRecordWithFlags(c->ev[i], c->stream, cudaEventRecordExternal));
    else
        PINT_CUDA_CHECK(cudaEventRecord(c->ev[i], c->stream));
}

float elapsed(pint_ctx* c, int a, int b) {
    float ms = 0.f;
    PINT_CUDA_CHECK(cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]));
    return ms;
}

// H~^{-1} pieces shared by apply, ref-norm and the Uzawa step
// zh = S z (into w1); y1 = V_H(zh) (w2); b2 = A_ref y1 (scratch); w = s V_H(b2)
void schur_mode_space(pint_ctx* c, const double* z, double* scratch, int epi, double* wout,
                      int slot) {
    const double s = 2.0 * c->tau_ref / c->N;   // schur.py:67
    rec(c, 1);
    pint::dst_apply(c, 1, z, c->d_w1, nullptr, 1.0);
    rec(c, 2);
    if (pint::vcycle_aref_fusable(c, PINT_MG_HTILDE) && scratch != wout) {
        // b2 = A_ref y1 formed inside the second V-cycle's finest kernels
        // (schur.py:72-73).  y1 is read on halo rows by every band of the
        // second V-cycle, so it must not share a buffer with that V-cycle's
        // output: y1 goes to `scratch`, w to `wout`.
        pint::vcycle(c, PINT_MG_HTILDE, c->N, c->d_w1, scratch, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        pint::vcycle(c, PINT_MG_HTILDE, c->N, scratch, wout, epi, s, nullptr, c->d_w1, slot, true);
    } else {
        pint::vcycle(c, PINT_MG_HTILDE, c->N, c->d_w1, c->d_w2, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        pint::launch_aref(c, c->d_w2, scratch, c->N);
        pint::vcycle(c, PINT_MG_HTILDE, c->N, scratch, wout, epi, s, nullptr, c->d_w1, slot);
    }
    rec(c, 3);
}

void ensure_uzawa_buffers(pint_ctx* c) {
    const size_t S = slab(c);
    if (!c->d_f) c->d_f = dalloc<double>(S);
    if (!c->d_p) c->d_p = dalloc<double>(S);
    if (!c->d_u) c->d_u = dalloc<double>(S);
    if (!c->d_r1) c->d_r1 = dalloc<double>(S);
    if (!c->d_z) c->d_z = dalloc<double>(S);
    if (!c->d_w1) c->d_w1 = dalloc<double>(S);
    if (!c->d_w2) c->d_w2 = dalloc<double>(S);
}

void ensure_stage(pint_ctx* c) {
    const size_t S = slab(c);
    if (!c->d_stage_in) c->d_stage_in = dalloc<double>(S);
    if (!c->d_stage_out) c->d_stage_out = dalloc<double>(S);
}

bool set_ready(const pint_ctx* c, int which) {
    return c->field ? c->fmg[which].ready : c->mg[which].ready;
}

void require_sets(pint_ctx* c) {
    if (!set_ready(c, PINT_MG_ATILDE) || !set_ready(c, PINT_MG_HTILDE))
        pint_throw(PINT_INPUT, "both multigrid sets (A~ and H~) must be configured");
}

}  // namespace

extern "C" {

int pint_abi_version(void) { return 1; }

int pint_ctx_create(int device, int rank, int world, const void* nccl_id, pint_ctx** out) {
    (void)nccl_id;
    if (out == nullptr) return PINT_INPUT;
    *out = nullptr;
    if (world != 1 || rank != 0) return PINT_INPUT;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return PINT_CUDA;
    }
    pint_ctx* c = new pint_ctx();
    if (const char* e = getenv("PINT_EXACT")) c->exact = atoi(e) != 0;
    c->dev = device;
    c->rank = rank;
    c->world = world;
    const int st = guarded(c, [&] {
        PINT_CUDA_CHECK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        PINT_CUDA_CHECK(cudaMalloc(&c->d_acc, 8 * sizeof(double)));
        PINT_CUDA_CHECK(cudaMallocHost(&c->h_acc, 8 * sizeof(double)));
        for (auto& e : c->ev) PINT_CUDA_CHECK(cudaEventCreate(&e));
    });
    if (st != PINT_OK) {
        delete c;
        return st;
    }
    *out = c;
    return PINT_OK;
}

int pint_ctx_destroy(pint_ctx* c) {
    if (c == nullptr) return PINT_OK;
    cudaSetDevice(c->dev);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_problem(c);
    pint::dst_plan_free(c->dst_raw);
    dfree(c->d_part);
    dfree(c->d_acc);
    if (c->h_acc) cudaFreeHost(c->h_acc);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->prof_pool) cudaEventDestroy(e);
    pint::host_xfer_free(c);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return PINT_OK;
}

const char* pint_last_error(const pint_ctx* c) { return c ? c->err.c_str() : "null context"; }

int pint_sync(pint_ctx* c) {
    return guarded(c, [&] { PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream)); });
}

long long pint_launch_count(const pint_ctx* c) { return c ? c->launches : 0; }

int pint_set_stream(pint_ctx* c, void* stream, int own) {
    return guarded(c, [&] {
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        // stream 0 is the legacy default stream (torch's default): a valid choice
        c->stream = own ? c->own_stream : static_cast<cudaStream_t>(stream);
        graph_reset(c);
    });
}

int pint_set_arith(pint_ctx* c, int exact) {
    return guarded(c, [&] {
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        c->exact = exact != 0;
        graph_reset(c);
    });
}

int pint_get_arith(const pint_ctx* c) { return c ? c->exact : -1; }

int pint_profile(pint_ctx* c, int on) {
    return guarded(c, [&] {
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        pint_prof_drain(c);
        c->profile = on != 0;
        for (KStat& k : c->kstat) k = KStat{};
    });
}

int pint_kernel_stat(pint_ctx* c, int id, const char** name, double* ms_total,
                     long long* launches, double* alg_bytes_total) {
    return guarded(c, [&] {
        if (id < 0 || id >= K_COUNT) pint_throw(PINT_INPUT, "kernel id out of range");
        if (name) *name = kKernelNames[id];
        if (ms_total) *ms_total = c->kstat[id].ms;
        if (launches) *launches = c->kstat[id].count;
        if (alg_bytes_total) *alg_bytes_total = c->kstat[id].bytes;
    });
}

int pint_kernel_count(void) { return K_COUNT; }

int pint_uzawa_run(pint_ctx* c, double omega, int iters, double* res_num, double* ms_out) {
    return guarded(c, [&] {
        if (!c->uz_ready) pint_throw(PINT_INPUT, "pint_uzawa_begin not called");
        cudaEvent_t a, b;
        PINT_CUDA_CHECK(cudaEventCreate(&a));
        PINT_CUDA_CHECK(cudaEventCreate(&b));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        PINT_CUDA_CHECK(cudaEventRecord(a, c->stream));
        for (int j = 0; j < iters; ++j) {
            double num = 0.0;
            const int st = pint_uzawa_step(c, omega, &num);
            if (st != PINT_OK) pint_throw(st, c->err);
            if (res_num) res_num[j] = num;
        }
        PINT_CUDA_CHECK(cudaEventRecord(b, c->stream));
        PINT_CUDA_CHECK(cudaEventSynchronize(b));
        float ms = 0.f;
        PINT_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (ms_out) *ms_out = ms;
    });
}

int pint_set_timing(pint_ctx* c, int on) {
    return guarded(c, [&] { c->timing = on != 0; });
}

int pint_phase_ms(pint_ctx* c, double* ms3) {
    return guarded(c, [&] {
        if (!ms3) pint_throw(PINT_INPUT, "null output");
        ms3[0] = c->ms_dst;
        ms3[1] = c->ms_mg;
        ms3[2] = c->ms_other;
    });
}

int pint_problem_set(pint_ctx* c, int dims, int m, int N, const double* steps, const double* mass,
                     int n_a, const double* a_st, const int* a_sid, const double* a_scale,
                     const double* aref, double tau_ref) {
    return guarded(c, [&] {
        if (dims != 2 && dims != 3) pint_throw(PINT_INPUT, "dims must be 2 or 3");
        if (m < 1 || N < 1 || n_a < 1) pint_throw(PINT_INPUT, "bad problem dimensions");
        if (!steps || !mass || !a_st || !a_sid || !a_scale || !aref)
            pint_throw(PINT_INPUT, "null problem array");
        for (int t = 0; t < N; ++t) {
            if (!(steps[t] > 0.0)) pint_throw(PINT_INPUT, "time-step lengths must be positive");
            if (a_sid[t] < 0 || a_sid[t] >= n_a) pint_throw(PINT_INPUT, "bad stiffness index");
        }
        free_problem(c);
        c->dims = dims;
        c->m = m;
        c->n = dims == 2 ? m * m : m * m * m;
        const int S = dims == 2 ? 9 : 27;
        c->N = N;
        c->tau_ref = tau_ref;
        c->n_a = n_a;
        c->n0 = 0;
        c->N_global = N;
        c->has_prev = c->has_next = false;
        c->h_steps.assign(steps, steps + N);
        c->h_mass.assign(mass, mass + S);
        c->h_ast.assign(a_st, a_st + (size_t)n_a * S);
        c->h_aref.assign(aref, aref + S);
        c->d_steps = upload(c, steps, N);
        {
            // x / tau is computed as x * (1/tau) only where that is bit-identical:
            // tau a power of two (then 1/tau is exact and both round once)
            std::vector<double> r(N, 0.0);
            for (int t = 0; t < N; ++t) {
                int e = 0;
                const double mant = std::frexp(steps[t], &e);
                if (mant == 0.5 && e > -1000 && e < 1000) r[t] = std::ldexp(1.0, 1 - e);
            }
            c->d_rsteps = upload(c, r.data(), N);
        }
        c->d_mass = upload(c, mass, S);
        c->d_ast = upload(c, a_st, (size_t)n_a * S);
        c->d_asid = upload(c, a_sid, N);
        c->d_ascale = upload(c, a_scale, N);
        c->d_aref = upload(c, aref, S);
        pint::dst_plan_build(c->dst, N);
        c->problem_ready = true;
    });
}

int pint_mg_set(pint_ctx* c, int which, int levels, const int* level_m, int n_sets,
                const double* tables, const int* sid) {
    return guarded(c, [&] {
        require_problem(c);
        graph_reset(c);
        if (which != PINT_MG_ATILDE && which != PINT_MG_HTILDE && which != PINT_MG_EULER)
            pint_throw(PINT_INPUT, "unknown multigrid set");
        if (levels < 2 || !level_m || !tables || !sid || n_sets < 1)
            pint_throw(PINT_INPUT, "bad multigrid description");
        if (level_m[0] != c->m) pint_throw(PINT_DIMENSION, "finest level does not match problem");
        for (int l = 0; l + 1 < levels; ++l)
            if (level_m[l] != 2 * level_m[l + 1] + 1)
                pint_throw(PINT_INPUT, "levels must halve the cell count");
        const int TW = c->dims == 2 ? PINT_TW : 28;
        for (int b = 0; b < c->N; ++b)
            if (sid[b] < 0 || sid[b] >= n_sets) pint_throw(PINT_INPUT, "bad operator-set index");
        const size_t ntab = (size_t)levels * n_sets * TW;
        for (int s = 0; s < n_sets; ++s) {
            const double a = tables[((size_t)(levels - 1) * n_sets + s) * TW + (TW - 1) / 2];
            if (!(a > 0.0)) pint_throw(PINT_NOT_SPD, "non-positive pivot: operator is not SPD");
        }
        MgSet& s = c->mg[which];
        dfree(s.tab);
        dfree(s.sid);
        s = MgSet{};
        s.levels = levels;
        s.m.assign(level_m, level_m + levels);
        s.n_sets = n_sets;
        s.tab = upload(c, tables, ntab);
        s.sid = upload(c, sid, c->N);
        if (c->dims == 2) pint::mg_compute_shapes(s, tables);
        if (c->dims == 3)
            for (int l = 0; l < levels; ++l) {
                uint32_t mask = 0;
                for (int q = 0; q < n_sets; ++q)
                    for (int k = 0; k < 27; ++k)
                        if (tables[((size_t)l * n_sets + q) * TW + k] != 0.0) mask |= 1u << k;
                s.shape3.push_back(mask);
            }
        ensure_levels(c, s.m);
        s.ready = true;
    });
}

// ---------------------------------------------------------------------------
// field mode: per-point 2D stiffness (field2d.cu)
// ---------------------------------------------------------------------------
static void enable_field(pint_ctx* c) {
    require_problem(c);
    if (c->dims != 2) pint_throw(PINT_INPUT, "per-point stiffness fields are 2D");
    if (!c->field) {
        c->d_fref = dalloc<double>((size_t)3 * c->n);
        c->field = true;
    }
}

// per-step compact fields [N][3][n] (not held by separable families)
static void ensure_step_fields(pint_ctx* c) {
    if (c->fsep_R) pint_throw(PINT_INPUT, "the stiffness family was declared separable");
    if (!c->d_fa) {
        c->d_fa = dalloc<double>((size_t)c->N * 3 * c->n);
        PINT_CUDA_CHECK(cudaMemsetAsync(c->d_fa, 0, (size_t)c->N * 3 * c->n * sizeof(double),
                                        c->stream));
    }
}


int pint_mg_set_options(pint_ctx* c, int which, int cycles, int smooth_steps) {
    return guarded(c, [&] {
        require_problem(c);
        if (which != PINT_MG_ATILDE && which != PINT_MG_HTILDE && which != PINT_MG_EULER)
            pint_throw(PINT_INPUT, "unknown multigrid set");
        if (cycles < 1 || smooth_steps < 1)
            pint_throw(PINT_INPUT, "cycles and smooth_steps must be >= 1");
        if (c->field && (cycles != 1 || smooth_steps != 1))
            pint_throw(PINT_INPUT, "cycles / smooth_steps other than 1 are not available for "
                                   "per-point stiffness fields");
        MgSet& s = c->mg[which];
        if (!c->field && !s.ready) pint_throw(PINT_INPUT, "multigrid set not configured");
        graph_reset(c);  // the captured step holds the launches of the previous setting
        s.cycles = cycles;
        s.smooth = smooth_steps;
    });
}

int pint_field_set(pint_ctx* c, int step0, int count, const double* fields) {
    return guarded(c, [&] {
        enable_field(c);
        ensure_step_fields(c);
        if (step0 < 0 || count < 0 || step0 + count > c->N || !fields)
            pint_throw(PINT_DIMENSION, "bad step range");
        const size_t cnt = (size_t)count * 3 * c->n;
        PINT_CUDA_CHECK(cudaMemcpyAsync(c->d_fa + (size_t)step0 * 3 * c->n, fields,
                                        cnt * sizeof(double), cudaMemcpyDefault, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int pint_field_assemble(pint_ctx* c, int step0, int count, const double* cell_w) {
    return guarded(c, [&] {
        enable_field(c);
        ensure_step_fields(c);
        if (step0 < 0 || count < 0 || step0 + count > c->N || !cell_w)
            pint_throw(PINT_DIMENSION, "bad step range");
        if (count == 0) return;
        const size_t cw = (size_t)(c->m + 1) * (c->m + 1) * count;
        const double* d = cell_w;
        double* tmp = nullptr;
        if (!is_device_ptr(cell_w)) {
            tmp = dalloc<double>(cw);
            PINT_CUDA_CHECK(cudaMemcpyAsync(tmp, cell_w, cw * sizeof(double),
                                            cudaMemcpyHostToDevice, c->stream));
            d = tmp;
        }
        pint::field_assemble(c, step0, count, d);
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        dfree(tmp);
    });
}

int pint_field_separable(pint_ctx* c, int terms, const double* cell_w, const double* weights) {
    return guarded(c, [&] {
        enable_field(c);
        if (terms < 1 || terms > PINT_FSEP_MAX || !cell_w || !weights)
            pint_throw(PINT_INPUT, "bad separable family (1 .. PINT_FSEP_MAX terms)");
        if (c->d_fa) pint_throw(PINT_INPUT, "per-step stiffness fields are already set");
        graph_reset(c);
        for (FieldMg& F : c->fmg) free_field_set(F);  // their tables belong to the old family
        const size_t cw = (size_t)(c->m + 1) * (c->m + 1) * terms;
        double* tmp = dalloc<double>(cw);
        PINT_CUDA_CHECK(cudaMemcpyAsync(tmp, cell_w, cw * sizeof(double), cudaMemcpyDefault,
                                        c->stream));
        dfree(c->d_fsep);
        dfree(c->d_fsc);
        c->d_fsep = dalloc<double>((size_t)terms * 3 * c->n);
        pint::field_assemble(c, 0, terms, tmp, c->d_fsep);
        c->h_fsc.assign((size_t)c->N * terms, 0.0);
        if (is_device_ptr(weights)) {
            PINT_CUDA_CHECK(cudaMemcpyAsync(c->h_fsc.data(), weights, c->h_fsc.size() * sizeof(double),
                                            cudaMemcpyDeviceToHost, c->stream));
            PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        } else {
            std::copy(weights, weights + c->h_fsc.size(), c->h_fsc.begin());
        }
        c->d_fsc = upload(c, c->h_fsc.data(), c->h_fsc.size());
        if (!c->d_unit) {
            const double unit[2] = {1.0, 0.0};
            c->d_unit = upload(c, unit, 2);
        }
        c->fsep_R = terms;
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        dfree(tmp);
    });
}

int pint_field_aref(pint_ctx* c, int step, const double* fields) {
    return guarded(c, [&] {
        enable_field(c);
        const size_t cnt = (size_t)3 * c->n;
        if (fields) {
            PINT_CUDA_CHECK(cudaMemcpyAsync(c->d_fref, fields, cnt * sizeof(double),
                                            cudaMemcpyDefault, c->stream));
        } else {
            if (step < 0 || step >= c->N) pint_throw(PINT_DIMENSION, "bad A_ref step");
            if (c->fsep_R) {
                pint::field_sep_step(c, step, c->d_fref);
            } else {
                if (!c->d_fa) pint_throw(PINT_INPUT, "no stiffness fields set");
                PINT_CUDA_CHECK(cudaMemcpyAsync(c->d_fref, c->d_fa + (size_t)step * cnt,
                                                cnt * sizeof(double), cudaMemcpyDeviceToDevice,
                                                c->stream));
            }
        }
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        c->fref_ready = true;
    });
}

int pint_mg_set_field(pint_ctx* c, int which, int levels, const int* level_m, double damping,
                      const double* mu) {
    return guarded(c, [&] {
        require_problem(c);
        if (!c->field) pint_throw(PINT_INPUT, "no stiffness fields set");
        // the captured step graph holds this set's buffers and damping
        graph_reset(c);
        if (which != PINT_MG_ATILDE && which != PINT_MG_HTILDE)
            pint_throw(PINT_INPUT, "unknown multigrid set");
        if (levels < 2 || !level_m || !(damping > 0.0)) pint_throw(PINT_INPUT, "bad multigrid description");
        if (level_m[0] != c->m) pint_throw(PINT_DIMENSION, "finest level does not match problem");
        for (int l = 0; l + 1 < levels; ++l)
            if (level_m[l] != 2 * level_m[l + 1] + 1)
                pint_throw(PINT_INPUT, "levels must halve the cell count");
        if (level_m[levels - 1] != 1) pint_throw(PINT_INPUT, "coarsest level must be a single point");
        if (which == PINT_MG_HTILDE && (!mu || !c->fref_ready))
            pint_throw(PINT_INPUT, "H~ needs mode weights and the A_ref field");
        FieldMg& F = c->fmg[which];
        free_field_set(F);
        F.levels = levels;
        F.m.assign(level_m, level_m + levels);
        F.damping = damping;
        F.f9.assign(levels, nullptr);
        if (!c->fsep_R && !c->d_fa) pint_throw(PINT_INPUT, "no stiffness fields set");
        // separable family: R term tables per level, weights (1 .. , s_n) for A~
        // and (mu_k, tau_ref) for H_k = mu_k M + tau_ref A_ref
        F.sep = !c->fsep_R ? 0 : which == PINT_MG_ATILDE ? c->fsep_R : 2;
        const size_t rows = F.sep ? (size_t)F.sep : (size_t)c->N;
        for (int l = 1; l < levels; ++l)
            F.f9[l] = dalloc<double>(rows * 9 * level_m[l] * level_m[l]);
        if (mu) F.d_mu = upload(c, mu, c->N);
        std::vector<double> hsc;
        if (F.sep && which == PINT_MG_ATILDE) {
            F.d_sc = c->d_fsc;
            hsc = c->h_fsc;
        } else if (F.sep) {
            hsc.resize((size_t)c->N * 2);
            for (int k = 0; k < c->N; ++k) {
                hsc[2 * (size_t)k] = mu[k];
                hsc[2 * (size_t)k + 1] = c->tau_ref;
            }
            F.d_sc = upload(c, hsc.data(), hsc.size());
            F.own_sc = true;
        }
        pint::field_galerkin(c, which);
        // coarsest pivots (spatial.py:143 factorises the 1x1 operator)
        std::vector<double> piv(rows * 9);
        PINT_CUDA_CHECK(cudaMemcpyAsync(piv.data(), F.f9[levels - 1], piv.size() * sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        for (int s = 0; s < c->N; ++s) {
            double pv = 0.0;
            if (F.sep)
                for (int r = 0; r < F.sep; ++r) pv += hsc[(size_t)s * F.sep + r] * piv[(size_t)r * 9 + 4];
            else
                pv = piv[(size_t)s * 9 + 4];
            if (!(pv > 0.0)) pint_throw(PINT_NOT_SPD, "non-positive pivot: operator is not SPD");
        }
        ensure_levels(c, F.m);
        if (!c->d_ft) c->d_ft = dalloc<double>(slab(c));
        if (c->lev_t.size() < (size_t)levels) c->lev_t.resize(levels, nullptr);
        for (int l = 1; l < levels; ++l) {
            dfree(c->lev_t[l]);
            c->lev_t[l] = dalloc<double>((size_t)c->N * level_m[l] * level_m[l]);
        }
        F.ready = true;
    });
}

int pint_fold_rhs(pint_ctx* c, const double* load, const double* u_init, double* f) {
    return guarded(c, [&] {
        require_problem(c);
        ensure_stage(c);
        if (u_init == nullptr) pint_throw(PINT_INPUT, "null u_init");
        const double* dl = stage_in(c, load, c->d_stage_in, slab(c));
        const double* dui = u_init;
        if (!is_device_ptr(u_init)) {
            if (!c->d_vec) c->d_vec = dalloc<double>(c->n);
            PINT_CUDA_CHECK(cudaMemcpyAsync(c->d_vec, u_init, c->n * sizeof(double),
                                            cudaMemcpyHostToDevice, c->stream));
            dui = c->d_vec;
        }
        // the fold is element-wise in load, so a host result can overwrite the staged load
        OutBuf o = stage_out(c, f, c->d_stage_in);
        pint::launch_fold_rhs(c, dl, dui, o.dev);
        finish_out(c, o, slab(c));
    });
}

static int timeop_entry(pint_ctx* c, int op, const double* in, double* out) {
    return guarded(c, [&] {
        require_problem(c);
        ensure_stage(c);
        const double* d = stage_in(c, in, c->d_stage_in, slab(c));
        OutBuf o = stage_out(c, out, c->d_stage_out);
        if (o.dev == d) pint_throw(PINT_INPUT, "in-place operator application is not supported");
        pint::launch_timeop(c, op, d, nullptr, nullptr, o.dev);
        finish_out(c, o, slab(c));
    });
}

int pint_apply_K(pint_ctx* c, const double* in, double* out) {
    return timeop_entry(c, pint::OP_K, in, out);
}
int pint_apply_Kt(pint_ctx* c, const double* in, double* out) {
    return timeop_entry(c, pint::OP_KT, in, out);
}
int pint_apply_Abd(pint_ctx* c, const double* in, double* out) {
    return timeop_entry(c, pint::OP_ABD, in, out);
}

int pint_vcycle(pint_ctx* c, int which, int count, const double* in, double* out) {
    return guarded(c, [&] {
        require_problem(c);
        if (which != 0 && which != 1) pint_throw(PINT_INPUT, "unknown multigrid set");
        if (count < 1 || count > c->N) pint_throw(PINT_DIMENSION, "bad plane count");
        ensure_stage(c);
        const size_t cnt = (size_t)count * c->n;
        const double* d = stage_in(c, in, c->d_stage_in, cnt);
        OutBuf o = stage_out(c, out, c->d_stage_out);
        pint::vcycle(c, which, count, d, o.dev, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        finish_out(c, o, cnt);
    });
}

int pint_atilde_inv(pint_ctx* c, const double* in, double* out) {
    return guarded(c, [&] {
        require_problem(c);
        ensure_stage(c);
        const double* d = stage_in(c, in, c->d_stage_in, slab(c));
        OutBuf o = stage_out(c, out, c->d_stage_out);
        pint::vcycle(c, PINT_MG_ATILDE, c->N, d, o.dev, EPI_DIV_TAU, 1.0, nullptr, nullptr, 0);
        finish_out(c, o, slab(c));
    });
}

int pint_htilde_inv(pint_ctx* c, const double* in, double* out) {
    return guarded(c, [&] {
        require_problem(c);
        if (!set_ready(c, PINT_MG_HTILDE)) pint_throw(PINT_INPUT, "H~ multigrid set not configured");
        ensure_stage(c);
        ensure_uzawa_buffers(c);
        const double* d = stage_in(c, in, c->d_stage_in, slab(c));
        OutBuf o = stage_out(c, out, c->d_stage_out);
        schur_mode_space(c, d, c->d_z, EPI_SCALE, c->d_w2, 0);
        pint::dst_apply(c, 0, c->d_w2, o.dev, nullptr, 1.0);
        finish_out(c, o, slab(c));
    });
}

int pint_dst(pint_ctx* c, int kind, const double* in, double* out) {
    return guarded(c, [&] {
        require_problem(c);
        ensure_stage(c);
        const double* d = stage_in(c, in, c->d_stage_in, slab(c));
        OutBuf o = stage_out(c, out, c->d_stage_out);
        pint::dst_apply(c, kind, d, o.dev, nullptr, 1.0);
        finish_out(c, o, slab(c));
    });
}

static int dst_raw_impl(pint_ctx* c, int kind, int N, long long ncols, const double* in,
                        double* out, const double* base, double alpha) {
    return guarded(c, [&] {
        if (N < 1 || ncols < 1) pint_throw(PINT_DIMENSION, "bad transform shape");
        if (base && (!is_device_ptr(base) || !is_device_ptr(out)))
            pint_throw(PINT_INPUT, "the fused update needs device pointers");
        if (c->dst_raw.N != N) pint::dst_plan_build(c->dst_raw, N);
        const size_t cnt = (size_t)N * (size_t)ncols;
        double* tmp_in = nullptr;
        double* tmp_out = nullptr;
        const double* d = in;
        double* o = out;
        if (!is_device_ptr(in)) {
            tmp_in = dalloc<double>(cnt);
            PINT_CUDA_CHECK(cudaMemcpyAsync(tmp_in, in, cnt * sizeof(double),
                                            cudaMemcpyHostToDevice, c->stream));
            d = tmp_in;
        }
        if (!is_device_ptr(out)) {
            tmp_out = dalloc<double>(cnt);
            o = tmp_out;
        }
        pint::dst_run(c, c->dst_raw, kind, ncols, d, o, base, alpha);
        if (tmp_out)
            PINT_CUDA_CHECK(cudaMemcpyAsync(out, tmp_out, cnt * sizeof(double),
                                            cudaMemcpyDeviceToHost, c->stream));
        // device in / out: stream-ordered, no host wait
        if (tmp_in || tmp_out) {
            PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
            dfree(tmp_in);
            dfree(tmp_out);
        }
    });
}

int pint_dst_raw(pint_ctx* c, int kind, int N, long long ncols, const double* in, double* out) {
    return dst_raw_impl(c, kind, N, ncols, in, out, nullptr, 1.0);
}

// out = base + alpha * T(in) on an (N, ncols) column slab (base may alias out)
int pint_dst_raw_axpy(pint_ctx* c, int kind, int N, long long ncols, const double* in,
                      double* out, const double* base, double alpha) {
    return dst_raw_impl(c, kind, N, ncols, in, out, base, alpha);
}

// ---------------------------------------------------------------------------
// time-partitioned building blocks (driven by paper_1802_08126_b200/distributed.py)
// ---------------------------------------------------------------------------
static void drain_if_profiling(pint_ctx* c);

static void require_device(const void* p, const char* what) {
    if (p == nullptr || !is_device_ptr(p))
        pint_throw(PINT_INPUT, std::string(what) + " must be a device pointer");
}

int pint_set_partition(pint_ctx* c, int n0, int N_global, int has_prev, int has_next) {
    return guarded(c, [&] {
        require_problem(c);
        if (n0 < 0 || N_global < n0 + c->N)
            pint_throw(PINT_DIMENSION, "partition does not contain the local steps");
        if ((has_prev != 0) != (n0 > 0) || (has_next != 0) != (n0 + c->N < N_global))
            pint_throw(PINT_INPUT, "ghost flags disagree with the partition");
        c->n0 = n0;
        c->N_global = N_global;
        c->has_prev = has_prev != 0;
        c->has_next = has_next != 0;
    });
}

int pint_residual_r1(pint_ctx* c, const double* u, const double* p, const double* f, double* r1) {
    return guarded(c, [&] {
        require_problem(c);
        require_device(u, "u");
        require_device(p, "p");
        require_device(f, "f");
        require_device(r1, "r1");
        pint::launch_timeop(c, pint::OP_R1, u, p, f, r1);
        drain_if_profiling(c);
    });
}

int pint_residual_z(pint_ctx* c, const double* u, const double* p, const double* f, double* z) {
    return guarded(c, [&] {
        require_problem(c);
        require_device(u, "u");
        require_device(p, "p");
        require_device(f, "f");
        require_device(z, "z");
        pint::launch_timeop(c, pint::OP_Z, u, p, f, z);
        drain_if_profiling(c);
    });
}

// stream-ordered: without profiling nothing here waits for the device
static void drain_if_profiling(pint_ctx* c) {
    if (!c->profile) return;
    PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    pint_prof_drain(c);
}

// deliver d_acc[slot]: to a device pointer as a stream-ordered copy (no host
// wait: the caller all-reduces it on the same stream), to a host pointer
// after a stream sync, nowhere for NULL
static void deliver_acc(pint_ctx* c, int slot, double* dst) {
    drain_if_profiling(c);
    if (!dst) return;
    if (is_device_ptr(dst)) {
        PINT_CUDA_CHECK(cudaMemcpyAsync(dst, c->d_acc + slot, sizeof(double),
                                        cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    PINT_CUDA_CHECK(cudaMemcpyAsync(c->h_acc, c->d_acc + slot, sizeof(double),
                                    cudaMemcpyDeviceToHost, c->stream));
    PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    *dst = c->h_acc[0];
}

int pint_atilde_update(pint_ctx* c, const double* r1, double* p, double* dot) {
    return guarded(c, [&] {
        require_problem(c);
        if (!set_ready(c, PINT_MG_ATILDE)) pint_throw(PINT_INPUT, "A~ multigrid set not configured");
        require_device(r1, "r1");
        if (p) require_device(p, "p");
        pint::vcycle(c, PINT_MG_ATILDE, c->N, r1, p, p ? EPI_UZAWA_P : EPI_DOT_TAU, 1.0, p,
                     nullptr, 0);
        deliver_acc(c, 0, dot);
    });
}

int pint_htilde_modes(pint_ctx* c, const double* zh, double* w, double* dot) {
    return guarded(c, [&] {
        require_problem(c);
        if (!set_ready(c, PINT_MG_HTILDE)) pint_throw(PINT_INPUT, "H~ multigrid set not configured");
        require_device(zh, "zh");
        if (w) require_device(w, "w");
        ensure_uzawa_buffers(c);
        const int Ng = c->N_global > 0 ? c->N_global : c->N;
        const double s = 2.0 * c->tau_ref / Ng;  // schur.py:67 with the global N
        pint::vcycle(c, PINT_MG_HTILDE, c->N, zh, c->d_w2, EPI_PLAIN, 1.0, nullptr, nullptr, 0);
        if (pint::vcycle_aref_fusable(c, PINT_MG_HTILDE)) {
            pint::vcycle(c, PINT_MG_HTILDE, c->N, c->d_w2, w, w ? EPI_SCALE_DOT : EPI_SCALE_DOTONLY,
                         s, nullptr, zh, 1, true);
        } else {
            pint::launch_aref(c, c->d_w2, c->d_z, c->N);
            pint::vcycle(c, PINT_MG_HTILDE, c->N, c->d_z, w, w ? EPI_SCALE_DOT : EPI_SCALE_DOTONLY,
                         s, nullptr, zh, 1);
        }
        deliver_acc(c, 1, dot);
    });
}

int pint_axpy(pint_ctx* c, double* u, const double* y, double omega, long long count) {
    return guarded(c, [&] {
        require_device(u, "u");
        require_device(y, "y");
        pint::launch_axpy(c, u, y, omega, count);
    });
}

int pint_dot(pint_ctx* c, const double* a, const double* b, long long count, double* out) {
    return guarded(c, [&] {
        require_device(a, "a");
        require_device(b, "b");
        if (!out || count < 0) pint_throw(PINT_INPUT, "bad dot arguments");
        pint::launch_dot(c, a, b, count, 3);
        PINT_CUDA_CHECK(cudaMemcpyAsync(c->h_acc + 3, c->d_acc + 3, sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        *out = c->h_acc[3];
    });
}

int pint_lincomb(pint_ctx* c, double* out, long long count, const double* x0, double a1,
                 const double* x1, double a2, const double* x2, double scale, int use_scale) {
    return guarded(c, [&] {
        require_device(out, "out");
        require_device(x0, "x0");
        if (x1) require_device(x1, "x1");
        if (x2) require_device(x2, "x2");
        if (count < 0) pint_throw(PINT_INPUT, "bad count");
        pint::launch_lincomb(c, out, x0, a1, x1, a2, x2, scale, use_scale != 0, count);
    });
}

int pint_apply_saddle(pint_ctx* c, const double* p, const double* u, double* top,
                      double* bottom) {
    return guarded(c, [&] {
        require_problem(c);
        require_device(p, "p");
        require_device(u, "u");
        require_device(top, "top");
        require_device(bottom, "bottom");
        ensure_uzawa_buffers(c);
        const long long S = (long long)slab(c);
        // top = Abd p - K u ;  bottom = -Kt p - ((K u + Kt u) + Abd u)   (operators.py:107-111)
        // are the two fused Uzawa residuals with a zero right-hand side:
        //   r1(f = 0) = (K u - Abd p) - 0 = -(top)          (a - b == -(b - a) exactly)
        //   z(f = 0)  = (0 - Kt p) - ((K u + Kt u) + Abd u) = bottom
        // two launches + one negation instead of six operator passes and four
        // vector combinations (MINRES applies this twice per iteration)
        double* zero = c->d_w1;
        PINT_CUDA_CHECK(cudaMemsetAsync(zero, 0, (size_t)S * sizeof(double), c->stream));
        c->mu3_trust = false;
        pint::launch_timeop(c, pint::OP_R1, u, p, zero, top);
        c->mu3_trust = true;   // the same u: the 3D path reuses M u
        pint::launch_timeop(c, pint::OP_Z, u, p, zero, bottom);
        c->mu3_trust = false;
        pint::launch_lincomb(c, top, top, 0.0, nullptr, 0.0, nullptr, -1.0, true, S);
    });
}

int pint_uzawa_begin(pint_ctx* c, const double* f, const double* p0, const double* u0,
                     double* ref_out) {
    return guarded(c, [&] {
        require_problem(c);
        require_sets(c);
        // host staging slabs are not part of the iteration's working set:
        // release them first (config 4 needs the room; they come back on demand)
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        dfree(c->d_stage_in);
        dfree(c->d_stage_out);
        c->d_stage_in = c->d_stage_out = nullptr;
        if (!c->d_f || !c->d_r1 || !c->d_w2) graph_reset(c);  // buffers (re)allocated below
        ensure_uzawa_buffers(c);
        const size_t S = slab(c), bytes = S * sizeof(double);
        copy_in(c, c->d_f, f, bytes);
        if (p0)
            copy_in(c, c->d_p, p0, bytes);
        else
            PINT_CUDA_CHECK(cudaMemsetAsync(c->d_p, 0, bytes, c->stream));
        if (u0)
            copy_in(c, c->d_u, u0, bytes);
        else
            PINT_CUDA_CHECK(cudaMemsetAsync(c->d_u, 0, bytes, c->stream));
        // ref = sqrt(max(f.A~^-1 f + f.H~^-1 f, 0))   (solvers.py:212-217)
        pint::vcycle(c, PINT_MG_ATILDE, c->N, c->d_f, nullptr, EPI_DOT_TAU, 1.0, nullptr,
                     nullptr, 0);
        schur_mode_space(c, c->d_f, c->d_z, EPI_SCALE_DOTONLY, nullptr, 1);
        PINT_CUDA_CHECK(cudaMemcpyAsync(c->h_acc, c->d_acc, 2 * sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        const double q = c->h_acc[0] + c->h_acc[1];
        c->ref = std::sqrt(q > 0.0 ? q : 0.0);
        c->uz_ready = true;
        c->uz_steps = 0;
        c->ms_dst = c->ms_mg = c->ms_other = 0.0;
        if (ref_out) *ref_out = c->ref;
    });
}

// one Uzawa iteration (solvers.py:224-233), stream-ordered, no host sync
void uzawa_step_enqueue(pint_ctx* c, double omega) {
    rec(c, 0);
    // u is not written between the two residuals: the 3D path may reuse M u
    c->mu3_trust = true;
    pint::launch_timeop(c, pint::OP_R1, c->d_u, c->d_p, c->d_f, c->d_r1);
    rec(c, 4);
    pint::vcycle(c, PINT_MG_ATILDE, c->N, c->d_r1, c->d_p, EPI_UZAWA_P, 1.0, c->d_p, nullptr, 0);
    rec(c, 5);
    pint::launch_timeop(c, pint::OP_Z, c->d_u, c->d_p, c->d_f, c->d_z);
    c->mu3_trust = false;
    schur_mode_space(c, c->d_z, c->d_z, EPI_SCALE_DOT, c->d_w2, 1);
    pint::dst_apply(c, 0, c->d_w2, c->d_u, c->d_u, omega);
    rec(c, 6);
    PINT_CUDA_CHECK(cudaMemcpyAsync(c->h_acc, c->d_acc, 2 * sizeof(double),
                                    cudaMemcpyDeviceToHost, c->stream));
}

bool graphs_enabled() {
    static const int v = getenv("PINT_NO_GRAPH") ? 0 : 1;
    return v != 0;
}

// The ~30 launches of a step are replayed as one CUDA graph: the first step
// of a solve runs eagerly (it sizes every lazily allocated buffer), the
// second is captured; the graph lives until the problem, the multigrid
// tables, the stream or the arithmetic change (graph_reset).
void uzawa_step_launch(pint_ctx* c, double omega) {
    const bool want = graphs_enabled() && !c->profile;
    if (want && c->g_exec && c->g_omega == omega && c->g_timing == c->timing &&
        c->g_stream == c->stream) {
        PINT_CUDA_CHECK(cudaGraphLaunch(c->g_exec, c->stream));
        c->launches += c->g_launches;
        return;
    }
    if (!want || c->uz_steps < 1) {
        uzawa_step_enqueue(c, omega);
        return;
    }
    graph_reset(c);
    const long long l0 = c->launches;
    cudaGraph_t g = nullptr;
    PINT_CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
        uzawa_step_enqueue(c, omega);
    } catch (...) {
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
    }
    PINT_CUDA_CHECK(cudaStreamEndCapture(c->stream, &g));
    const cudaError_t ie = cudaGraphInstantiate(&c->g_exec, g, 0);
    cudaGraphDestroy(g);
    PINT_CUDA_CHECK(ie);
    c->g_launches = c->launches - l0;
    c->g_omega = omega;
    c->g_timing = c->timing;
    c->g_stream = c->stream;
    PINT_CUDA_CHECK(cudaGraphLaunch(c->g_exec, c->stream));
}

int pint_uzawa_step(pint_ctx* c, double omega, double* res_num_out) {
    return guarded(c, [&] {
        if (!c->uz_ready) pint_throw(PINT_INPUT, "pint_uzawa_begin not called");
        uzawa_step_launch(c, omega);
        ++c->uz_steps;
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        pint_prof_drain(c);
        if (c->timing) {
            // events: 0 start, 4 r1 done, 5 A~ done, 1 z done, 2 DST^T done, 3 modes done, 6 end
            c->ms_dst += elapsed(c, 1, 2) + elapsed(c, 3, 6);
            c->ms_mg += elapsed(c, 4, 5) + elapsed(c, 2, 3);
            c->ms_other += elapsed(c, 0, 4) + elapsed(c, 5, 1);
        }
        const double q = c->h_acc[0] + c->h_acc[1];
        if (res_num_out) *res_num_out = std::sqrt(q > 0.0 ? q : 0.0);
    });
}

int pint_host_prefault(pint_ctx* c, void* host, long long bytes) {
    return guarded(c, [&] {
        if (!host || bytes < 0) pint_throw(PINT_INPUT, "bad host buffer");
        if (is_device_ptr(host)) return;
        pint::host_prefault_async(c, host, (size_t)bytes);
    });
}

int pint_host_prefault_join(pint_ctx* c) {
    return guarded(c, [&] { pint::host_prefault_join(c); });
}

int pint_uzawa_end(pint_ctx* c, double* p, double* u) {
    return guarded(c, [&] {
        if (!c->uz_ready) pint_throw(PINT_INPUT, "pint_uzawa_begin not called");
        const size_t bytes = slab(c) * sizeof(double);
        if (p) copy_out(c, p, c->d_p, bytes);
        if (u) copy_out(c, u, c->d_u, bytes);
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int pint_uzawa(pint_ctx* c, const double* f, double* p, double* u, double omega, double tol,
               int max_iter, int use_initial, double* res_hist, int* iters, int* converged,
               double* phase_ms) {
    int st = pint_uzawa_begin(c, f, use_initial ? p : nullptr, use_initial ? u : nullptr, nullptr);
    if (st != PINT_OK) return st;
    if (iters) *iters = 0;
    if (converged) *converged = 0;
    if (c->ref == 0.0) {
        if (converged) *converged = 1;
        return pint_uzawa_end(c, p, u);
    }
    double first = -1.0;
    const bool was_timing = c->timing;
    c->timing = phase_ms != nullptr;
    for (int j = 0; j < max_iter; ++j) {
        double num = 0.0;
        st = pint_uzawa_step(c, omega, &num);
        if (st != PINT_OK) break;
        const double res = num / c->ref;
        if (res_hist) res_hist[j] = res;
        if (iters) *iters = j + 1;
        if (first < 0.0) first = res > 1e-300 ? res : 1e-300;
        if (res > 1e6 * first) {
            char buf[128];
            snprintf(buf, sizeof buf, "residual grew to %.3e from %.3e", res, first);
            c->err = buf;
            st = PINT_DIVERGED;
            break;
        }
        if (res < tol) {
            if (converged) *converged = 1;
            break;
        }
    }
    c->timing = was_timing;
    if (phase_ms) {
        phase_ms[0] = c->ms_dst;
        phase_ms[1] = c->ms_mg;
        phase_ms[2] = c->ms_other;
    }
    if (st == PINT_DIVERGED) {
        std::string keep = c->err;
        pint_uzawa_end(c, p, u);
        c->err = keep;
        return st;
    }
    if (st != PINT_OK) return st;
    return pint_uzawa_end(c, p, u);
}

// ---------------------------------------------------------------------------
// diagnostic mode: exact solves on the device (exact_solve.cu)
// ---------------------------------------------------------------------------
static void require_exact_capable(pint_ctx* c) {
    require_problem(c);
    if (c->field) pint_throw(PINT_INPUT, "exact solves are not built for per-point stiffness fields");
}

int pint_sequential_euler(pint_ctx* c, const double* load, const double* u_init, double* u_out,
                          double tol, int max_iter, int* iters, double* worst_rel) {
    return guarded(c, [&] {
        require_exact_capable(c);
        if (!load || !u_init || !u_out) pint_throw(PINT_INPUT, "null argument");
        ensure_stage(c);
        const double* dl = stage_in(c, load, c->d_stage_in, slab(c));
        const double* du0 = u_init;
        if (!is_device_ptr(u_init)) {
            if (!c->d_vec) c->d_vec = dalloc<double>(c->n);
            PINT_CUDA_CHECK(cudaMemcpyAsync(c->d_vec, u_init, c->n * sizeof(double),
                                            cudaMemcpyHostToDevice, c->stream));
            du0 = c->d_vec;
        }
        OutBuf o = stage_out(c, u_out, c->d_stage_out);
        double rel = 0.0;
        const int it = pint::sequential_euler(c, dl, du0, o.dev, tol, max_iter, &rel);
        finish_out(c, o, slab(c));
        if (iters) *iters = it;
        if (worst_rel) *worst_rel = rel;
    });
}

// |a - b|_S (b may be NULL): S-norm of operators.py:182-183
int pint_s_norm(pint_ctx* c, const double* a, const double* b, double tol, int max_iter,
                double* out) {
    return guarded(c, [&] {
        require_exact_capable(c);
        if (!set_ready(c, PINT_MG_ATILDE)) pint_throw(PINT_INPUT, "A~ multigrid set not configured");
        if (!a || !out) pint_throw(PINT_INPUT, "null argument");
        ensure_stage(c);
        const size_t S = slab(c);
        const double* da = stage_in(c, a, c->d_stage_in, S);
        const double* v = da;
        if (b) {
            const double* db = stage_in(c, b, c->d_stage_out, S);
            pint::launch_lincomb(c, c->d_stage_out, da, -1.0, db, 0.0, nullptr, 1.0, false,
                                 (long long)S);
            v = c->d_stage_out;
        }
        const double q = pint::s_norm_sq(c, v, tol, max_iter, nullptr);
        *out = std::sqrt(q > 0.0 ? q : 0.0);
    });
}

// |u_j - u_star|_S of the Uzawa iterate held by the context (diagnostic mode
// of uzawa_solve, solvers.py:236-244); u_star device or host
int pint_uzawa_s_error(pint_ctx* c, const double* u_star, double tol, int max_iter, double* out) {
    return guarded(c, [&] {
        if (!c->uz_ready) pint_throw(PINT_INPUT, "pint_uzawa_begin not called");
        require_exact_capable(c);
        ensure_stage(c);
        const size_t S = slab(c);
        const double* ds = stage_in(c, u_star, c->d_stage_in, S);
        pint::launch_lincomb(c, c->d_stage_out, c->d_u, -1.0, ds, 0.0, nullptr, 1.0, false,
                             (long long)S);
        const double q = pint::s_norm_sq(c, c->d_stage_out, tol, max_iter, nullptr);
        *out = std::sqrt(q > 0.0 ? q : 0.0);
    });
}

// exact A_bd^{-1} (operators.py:113-122)
int pint_abd_inverse(pint_ctx* c, const double* in, double* out, double tol, int max_iter) {
    return guarded(c, [&] {
        require_exact_capable(c);
        if (!set_ready(c, PINT_MG_ATILDE)) pint_throw(PINT_INPUT, "A~ multigrid set not configured");
        ensure_stage(c);
        const double* d = stage_in(c, in, c->d_stage_in, slab(c));
        OutBuf o = stage_out(c, out, c->d_stage_out);
        if (o.dev == d) pint_throw(PINT_INPUT, "in-place operator application is not supported");
        pint::abd_inverse(c, d, o.dev, tol, max_iter);
        finish_out(c, o, slab(c));
    });
}

}  // extern "C"
