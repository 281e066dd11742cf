// Dispatch of the 2D band kernels between the bit-exact build (pint::exact,
// -fmad=false: every stencil / multigrid row sum equals scipy's CSR product
// bit for bit) and the FMA build (pint::fast, the default arithmetic).  The
// fast build changes each operator by at most a few ulps (<= 1e-15
// relative); the Uzawa iteration counts and residual histories stay inside
// the reference's own DST-path noise.
#include "pint_internal.cuh"

namespace pint {

bool band_timeop_supported(const pint_ctx* c) {
    return c->exact ? exact::band_timeop_supported(c) : fast::band_timeop_supported(c);
}

void launch_band_timeop(pint_ctx* c, int op, const double* u, const double* p, const double* f,
                        double* out) {
    if (c->exact) exact::launch_band_timeop(c, op, u, p, f, out);
    else fast::launch_band_timeop(c, op, u, p, f, out);
}

void launch_band_apply(pint_ctx* c, const double* st_dev, const double* st_host, const double* in,
                       double* out, int count) {
    if (c->exact) exact::launch_band_apply(c, st_dev, st_host, in, out, count);
    else fast::launch_band_apply(c, st_dev, st_host, in, out, count);
}

void vcycle(pint_ctx* c, int which, int count, const double* b, double* out, int epi,
            double scale, const double* pin, const double* aux, int acc_slot, bool aref_in) {
    if (vcycle_is_generic(c, which)) {
        if (aref_in) pint_throw(PINT_INPUT, "fused A_ref input needs the V(1,1) kernels");
        vcycle_generic(c, which, count, b, out, epi, scale, pin, aux, acc_slot);
        return;
    }
    if (c->exact) exact::vcycle(c, which, count, b, out, epi, scale, pin, aux, acc_slot, aref_in);
    else fast::vcycle(c, which, count, b, out, epi, scale, pin, aux, acc_slot, aref_in);
}

bool vcycle_aref_fusable(const pint_ctx* c, int which) {
    if (vcycle_is_generic(c, which)) return false;
    return c->exact ? exact::vcycle_aref_fusable(c, which) : fast::vcycle_aref_fusable(c, which);
}

void mg_compute_shapes(MgSet& set, const double* tables) { exact::mg_compute_shapes(set, tables); }

}  // namespace pint
