// Host <-> device block-vector transfers for the reference-facing API.
//
// The reference's callers hand numpy arrays (pageable host memory) to
// uzawa_solve and get numpy arrays back (solvers.py:177-264); a slab is
// 0.5-8.6 GB at the BASELINE configs.  A plain cudaMemcpy of pageable memory
// runs through the driver's single staging thread (~10-20 GB/s) and the
// destination's first-touch page faults are taken by that one thread.  Here
// the copy is split into chunks that T host threads move through their own
// pair of pinned buffers while the copy engine streams the previous chunk:
//   H2D: memcpy(pinned[slot] <- host chunk); cudaMemcpyAsync(dev <- pinned[slot])
//   D2H: cudaMemcpyAsync(pinned[slot] <- dev chunk); wait; memcpy(host <- pinned[slot])
// All DMAs are issued on the context stream, so they are ordered with the
// kernels around them exactly like the single cudaMemcpyAsync they replace.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "pint_internal.cuh"

namespace pint {

struct HostXfer {
    int threads = 0;
    size_t chunk = 0;
    std::vector<char*> pinned;      // 2 per thread
    std::vector<cudaEvent_t> done;  // DMA completion per pinned buffer
    std::vector<std::thread> faulting;  // background first-touch of host outputs
};

namespace {

constexpr size_t kSmall = 8u << 20;  // below this one plain async copy is cheaper

HostXfer* xfer_of(pint_ctx* c) {
    if (c->xfer) return c->xfer;
    auto* x = new HostXfer;
    int t = (int)std::thread::hardware_concurrency();
    if (const char* e = getenv("PINT_COPY_THREADS")) t = atoi(e);
    x->threads = std::max(1, std::min(t > 0 ? t : 4, 16));
    x->chunk = 8u << 20;
    x->pinned.assign(2 * x->threads, nullptr);
    x->done.assign(2 * x->threads, nullptr);
    for (int i = 0; i < 2 * x->threads; ++i) {
        PINT_CUDA_CHECK(cudaHostAlloc(&x->pinned[i], x->chunk, cudaHostAllocPortable));
        PINT_CUDA_CHECK(cudaEventCreateWithFlags(&x->done[i], cudaEventDisableTiming));
    }
    c->xfer = x;
    return x;
}

// run body(t) on T threads (t = 0 on the caller), rethrowing the first error
template <typename F>
void fan_out(pint_ctx* c, int T, F body) {
    std::vector<std::thread> pool;
    std::vector<std::string> errs(T);
    std::vector<int> codes(T, PINT_OK);
    auto run = [&](int t) {
        try {
            cudaSetDevice(c->dev);
            body(t);
        } catch (const PintFail& e) {
            codes[t] = e.code;
            errs[t] = e.msg;
        }
    };
    for (int t = 1; t < T; ++t) pool.emplace_back(run, t);
    run(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < T; ++t)
        if (codes[t] != PINT_OK) pint_throw(codes[t], errs[t]);
}

}  // namespace

// First touch of a fresh host output buffer (numpy's np.empty) costs a page
// fault + zeroing per 4 KiB page; doing it inside the D2H copy halves its
// rate.  The caller can have it done by background threads while the device
// iterates; copy_d2h joins them first.
void host_prefault_async(pint_ctx* c, void* p, size_t bytes) {
    HostXfer* x = xfer_of(c);
    const int T = std::max(1, x->threads / 2);  // leave cores to the launching thread
    const size_t per = ((bytes + T - 1) / T + 4095) & ~size_t(4095);
    for (int t = 0; t < T; ++t) {
        const size_t off = (size_t)t * per;
        if (off >= bytes) break;
        const size_t len = std::min(per, bytes - off);
        char* base = static_cast<char*>(p) + off;
        x->faulting.emplace_back([base, len] {
            for (size_t i = 0; i < len; i += 4096) base[i] = 0;
        });
    }
}

void host_prefault_join(pint_ctx* c) {
    if (!c->xfer) return;
    for (auto& th : c->xfer->faulting) th.join();
    c->xfer->faulting.clear();
}

void host_xfer_free(pint_ctx* c) {
    HostXfer* x = c->xfer;
    if (!x) return;
    host_prefault_join(c);
    for (auto* p : x->pinned)
        if (p) cudaFreeHost(p);
    for (auto e : x->done)
        if (e) cudaEventDestroy(e);
    delete x;
    c->xfer = nullptr;
}

void copy_h2d(pint_ctx* c, void* dev, const void* host, size_t bytes) {
    if (bytes < kSmall) {
        PINT_CUDA_CHECK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c->stream));
        return;
    }
    HostXfer* x = xfer_of(c);
    const size_t C = x->chunk, nck = (bytes + C - 1) / C;
    const int T = (int)std::min<size_t>(x->threads, nck);
    fan_out(c, T, [&](int t) {
        int it = 0;
        for (size_t k = t; k < nck; k += T, ++it) {
            const int slot = 2 * t + (it & 1);
            // the slot's previous DMA may belong to this call (it >= 2) or to an
            // earlier copy_h2d issued without a stream sync in between; an
            // event that was never recorded returns at once
            PINT_CUDA_CHECK(cudaEventSynchronize(x->done[slot]));
            const size_t off = k * C, len = std::min(C, bytes - off);
            std::memcpy(x->pinned[slot], static_cast<const char*>(host) + off, len);
            PINT_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dev) + off, x->pinned[slot], len,
                                            cudaMemcpyHostToDevice, c->stream));
            PINT_CUDA_CHECK(cudaEventRecord(x->done[slot], c->stream));
        }
    });
}

void copy_d2h(pint_ctx* c, void* host, const void* dev, size_t bytes) {
    host_prefault_join(c);
    if (bytes < kSmall) {
        PINT_CUDA_CHECK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
        PINT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        return;
    }
    HostXfer* x = xfer_of(c);
    const size_t C = x->chunk, nck = (bytes + C - 1) / C;
    const int T = (int)std::min<size_t>(x->threads, nck);
    fan_out(c, T, [&](int t) {
        size_t pend_off = 0, pend_len = 0;
        int pend_slot = -1, it = 0;
        auto drain = [&]() {
            if (pend_slot < 0) return;
            PINT_CUDA_CHECK(cudaEventSynchronize(x->done[pend_slot]));
            std::memcpy(static_cast<char*>(host) + pend_off, x->pinned[pend_slot], pend_len);
            pend_slot = -1;
        };
        for (size_t k = t; k < nck; k += T, ++it) {
            const int slot = 2 * t + (it & 1);
            const size_t off = k * C, len = std::min(C, bytes - off);
            PINT_CUDA_CHECK(cudaMemcpyAsync(x->pinned[slot], static_cast<const char*>(dev) + off,
                                            len, cudaMemcpyDeviceToHost, c->stream));
            PINT_CUDA_CHECK(cudaEventRecord(x->done[slot], c->stream));
            drain();  // previous chunk of this thread, while this one is in flight
            pend_slot = slot;
            pend_off = off;
            pend_len = len;
        }
        drain();
    });
}

}  // namespace pint
