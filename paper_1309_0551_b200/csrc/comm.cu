// Native t-slab NN sweep over NCCL (BASELINE configs[4]; SURVEY.md 8(b) comm handles, 8(e)).
//
// The C-ABI counterpart of paper_1309_0551_b200/slab.py for host programs that
// do not run Python: a communicator handle wraps an NCCL communicator, one
// rank per GPU, and su3g_slab_nn_sweep_* performs one application of D on the
// rank's t-slab with the schedule of SURVEY.md 8(e):
//
//   stream S (caller's):  pack w = U_t^dag v on the last local slice  (su3g_nn_halo_w)
//                         record E_pack
//   comm stream C:        wait E_pack; group{ send v(t=0) -> r-1, recv v_hi <- r+1,
//                                             send w      -> r+1, recv w_lo <- r-1 }
//                         record E_halo
//   S:                    interior slices [1, nt-1)  -- overlaps the exchange
//   S:                    wait E_halo; boundary slices 0 and nt-1 with the halos
//
// The halos are the same values the periodic single-GPU kernel reads, computed
// with the same arithmetic, so the sharded result is bit-identical to the
// unsharded sweep.  NCCL is resolved at su3g_comm_init time with dlopen
// ("libnccl.so.2", normally already mapped by the host process; SU3G_NCCL_LIB
// overrides), so the library itself loads without NCCL.  A one-rank
// communicator exchanges with itself, which runs the whole schedule on one GPU.
#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include <nccl.h>

#include "su3g_common.cuh"

namespace su3g {

void set_sm_reserve(int n);
int sm_reserve();

namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
    decltype(&ncclCommAbort) commAbort = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int load_nccl() {
    std::lock_guard<std::mutex> lock(g_nccl_mu);
    if (g_nccl.handle) return SU3G_OK;
    const char* env = std::getenv("SU3G_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
        if (n && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return fail_invalid(std::string("comm: cannot load NCCL (libnccl.so.2; set SU3G_NCCL_LIB): ") + dlerror());
    NcclApi a;
    a.handle = h;
    bool ok = true;
#define SU3G_SYM(field, name)                                                 \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));            \
    ok = ok && a.field != nullptr
    SU3G_SYM(getUniqueId, "ncclGetUniqueId");
    SU3G_SYM(commInitRank, "ncclCommInitRank");
    SU3G_SYM(commDestroy, "ncclCommDestroy");
    SU3G_SYM(groupStart, "ncclGroupStart");
    SU3G_SYM(groupEnd, "ncclGroupEnd");
    SU3G_SYM(send, "ncclSend");
    SU3G_SYM(recv, "ncclRecv");
    SU3G_SYM(errorString, "ncclGetErrorString");
    SU3G_SYM(getAsyncError, "ncclCommGetAsyncError");
    SU3G_SYM(commAbort, "ncclCommAbort");
#undef SU3G_SYM
    if (!ok) return fail_invalid("comm: NCCL library lacks a required symbol");
    g_nccl = a;
    return SU3G_OK;
}

int nccl_fail(const char* what, ncclResult_t r) {
    set_error(std::string(what) + ": NCCL error " + std::to_string(int(r)) + " (" +
              (g_nccl.errorString ? g_nccl.errorString(r) : "?") + ")");
    return SU3G_ENCCL;
}

int cuda_fail(const char* what, cudaError_t e) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return static_cast<int>(e);
}

}  // namespace

}  // namespace su3g

struct su3g_comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    void* faces = nullptr;  // w_send | v_hi | w_lo, each 6*F reals
    size_t faces_bytes = 0;
};

using namespace su3g;

namespace {

template <typename T>
int slab_sweep(su3g_comm_t c, const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int mode,
               cudaStream_t st) {
    if (c == nullptr || c->nccl == nullptr) return fail_invalid("slab_nn_sweep: null or destroyed communicator");
    if (!U || !v || !out) return fail_invalid("slab_nn_sweep: null pointer");
    if (nx < 1 || ny < 1 || nz < 1 || nt < 1) return fail_invalid("slab_nn_sweep: lattice extents must be >= 1");
    if (out == v) return fail_invalid("slab_nn_sweep: out must not alias v");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != c->device) return fail_invalid("slab_nn_sweep: current device differs from the communicator's");
    // a communicator that failed asynchronously (peer died, network error) must not be fed more work
    ncclResult_t async_err = ncclSuccess;
    if (ncclResult_t r = g_nccl.getAsyncError(c->nccl, &async_err)) return nccl_fail("slab_nn_sweep: async query", r);
    if (async_err != ncclSuccess && async_err != ncclInProgress)
        return nccl_fail("slab_nn_sweep: communicator in error state", async_err);
    const int64_t F = int64_t(nx) * ny * nz;
    const size_t face = size_t(6 * F) * sizeof(T);
    if (c->faces_bytes < 3 * face) {
        cudaStreamSynchronize(c->comm_stream);
        if (c->faces) cudaFree(c->faces);
        c->faces = nullptr;
        c->faces_bytes = 0;
        if (cudaError_t e = cudaMalloc(&c->faces, 3 * face)) return cuda_fail("slab_nn_sweep: halo buffers", e);
        c->faces_bytes = 3 * face;
    }
    T* w_send = static_cast<T*>(c->faces);
    T* v_hi = w_send + 6 * F;
    T* w_lo = v_hi + 6 * F;
    const ncclDataType_t dt = sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
    const int lo = (c->rank - 1 + c->nranks) % c->nranks, hi = (c->rank + 1) % c->nranks;
    constexpr bool F32 = sizeof(T) == 4;
    auto sweep = [&](int t0, int t1, const T* vh, const T* wl) -> int {
        if (F32)
            return su3g_nn_sweep_f32(reinterpret_cast<const float*>(U), reinterpret_cast<const float*>(v),
                                     reinterpret_cast<float*>(out), nx, ny, nz, nt, t0, t1,
                                     reinterpret_cast<const float*>(vh), reinterpret_cast<const float*>(wl), mode, st);
        return su3g_nn_sweep_f64(reinterpret_cast<const double*>(U), reinterpret_cast<const double*>(v),
                                 reinterpret_cast<double*>(out), nx, ny, nz, nt, t0, t1,
                                 reinterpret_cast<const double*>(vh), reinterpret_cast<const double*>(wl), mode, st);
    };

    // 1. pack w on the last local slice, publish it and v to the comm stream
    int rc = F32 ? su3g_nn_halo_w_f32(reinterpret_cast<const float*>(U), reinterpret_cast<const float*>(v),
                                      reinterpret_cast<float*>(w_send), nx, ny, nz, nt, mode, st)
                 : su3g_nn_halo_w_f64(reinterpret_cast<const double*>(U), reinterpret_cast<const double*>(v),
                                      reinterpret_cast<double*>(w_send), nx, ny, nz, nt, mode, st);
    if (rc) return rc;
    if (cudaError_t e = cudaEventRecord(c->ev_pack, st)) return cuda_fail("slab_nn_sweep: record", e);
    if (cudaError_t e = cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0)) return cuda_fail("slab_nn_sweep: wait", e);
    // 2. halo exchange on the comm stream (v's t=0 face is the contiguous first 6F reals)
    ncclResult_t r = g_nccl.groupStart();
    if (r == ncclSuccess) r = g_nccl.send(v, size_t(6 * F), dt, lo, c->nccl, c->comm_stream);
    if (r == ncclSuccess) r = g_nccl.recv(v_hi, size_t(6 * F), dt, hi, c->nccl, c->comm_stream);
    if (r == ncclSuccess) r = g_nccl.send(w_send, size_t(6 * F), dt, hi, c->nccl, c->comm_stream);
    if (r == ncclSuccess) r = g_nccl.recv(w_lo, size_t(6 * F), dt, lo, c->nccl, c->comm_stream);
    const ncclResult_t r2 = g_nccl.groupEnd();
    if (r != ncclSuccess) return nccl_fail("slab_nn_sweep: send/recv", r);
    if (r2 != ncclSuccess) return nccl_fail("slab_nn_sweep: group", r2);
    if (cudaError_t e = cudaEventRecord(c->ev_halo, c->comm_stream)) return cuda_fail("slab_nn_sweep: record", e);
    // 3. interior while the halos move (leave SMs for NCCL's kernels on a multi-rank run)
    if (nt > 2) {
        const int saved = sm_reserve();
        if (c->nranks > 1) set_sm_reserve(4);
        rc = sweep(1, nt - 1, nullptr, nullptr);
        set_sm_reserve(saved);
        if (rc) return rc;
    }
    // 4. boundary slices once the halos are in
    if (cudaError_t e = cudaStreamWaitEvent(st, c->ev_halo, 0)) return cuda_fail("slab_nn_sweep: wait", e);
    // both boundary slices in one launch (su3g_nn_sweep_edges)
    if (F32)
        return su3g_nn_sweep_edges_f32(reinterpret_cast<const float*>(U), reinterpret_cast<const float*>(v),
                                       reinterpret_cast<float*>(out), nx, ny, nz, nt,
                                       reinterpret_cast<const float*>(v_hi), reinterpret_cast<const float*>(w_lo),
                                       nullptr, mode, st);
    return su3g_nn_sweep_edges_f64(reinterpret_cast<const double*>(U), reinterpret_cast<const double*>(v),
                                   reinterpret_cast<double*>(out), nx, ny, nz, nt,
                                   reinterpret_cast<const double*>(v_hi), reinterpret_cast<const double*>(w_lo),
                                   nullptr, mode, st);
}

}  // namespace

extern "C" {

int su3g_comm_unique_id(void* id_out) {
    if (id_out == nullptr) return fail_invalid("comm_unique_id: null pointer");
    if (int rc = load_nccl()) return rc;
    ncclUniqueId id;
    if (ncclResult_t r = g_nccl.getUniqueId(&id)) return nccl_fail("comm_unique_id", r);
    std::memcpy(id_out, &id, sizeof(id));
    return SU3G_OK;
}

int su3g_comm_init(int32_t nranks, int32_t rank, const void* id, su3g_comm_t* comm_out) {
    if (comm_out == nullptr || id == nullptr) return fail_invalid("comm_init: null pointer");
    *comm_out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail_invalid("comm_init: need 0 <= rank < nranks");
    if (int rc = load_nccl()) return rc;
    auto* c = new su3g_comm();
    c->rank = rank;
    c->nranks = nranks;
    cudaGetDevice(&c->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    if (ncclResult_t r = g_nccl.commInitRank(&c->nccl, nranks, uid, rank)) {
        delete c;
        return nccl_fail("comm_init", r);
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        su3g_comm_destroy(c);
        return cuda_fail("comm_init", e);
    }
    *comm_out = c;
    return SU3G_OK;
}

int su3g_comm_destroy(su3g_comm_t c) {
    if (c == nullptr) return SU3G_OK;
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    int rc = SU3G_OK;
    if (c->nccl) {
        if (ncclResult_t r = g_nccl.commDestroy(c->nccl)) rc = nccl_fail("comm_destroy", r);
    }
    if (c->faces) cudaFree(c->faces);
    if (c->ev_pack) cudaEventDestroy(c->ev_pack);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    delete c;
    return rc;
}

int su3g_comm_check(su3g_comm_t c, int64_t timeout_ms) {
    if (c == nullptr || c->nccl == nullptr) return fail_invalid("comm_check: null or destroyed communicator");
    // wait for the last enqueued exchange, polling NCCL's asynchronous error state; a peer that never
    // posts its half leaves the exchange pending forever, so past the deadline the communicator is
    // aborted (its kernels return) and the call fails instead of hanging the caller
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaEventQuery(c->ev_halo);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) return cuda_fail("comm_check: exchange", q);
        ncclResult_t async_err = ncclSuccess;
        if (ncclResult_t r = g_nccl.getAsyncError(c->nccl, &async_err)) return nccl_fail("comm_check: async query", r);
        if (async_err != ncclSuccess && async_err != ncclInProgress) {
            g_nccl.commAbort(c->nccl);
            c->nccl = nullptr;
            return nccl_fail("comm_check: halo exchange failed (communicator aborted)", async_err);
        }
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
        if (timeout_ms >= 0 && ms.count() > timeout_ms) {
            g_nccl.commAbort(c->nccl);
            c->nccl = nullptr;
            set_error("comm_check: halo exchange did not complete within " + std::to_string(timeout_ms) +
                      " ms (communicator aborted)");
            return SU3G_ENCCL;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    return SU3G_OK;
}

int su3g_comm_rank(su3g_comm_t c, int32_t* rank, int32_t* nranks) {
    if (c == nullptr || rank == nullptr || nranks == nullptr) return fail_invalid("comm_rank: null pointer");
    *rank = c->rank;
    *nranks = c->nranks;
    return SU3G_OK;
}

int su3g_slab_nn_sweep_f32(su3g_comm_t c, const float* U, const float* v, float* out, int32_t nx, int32_t ny,
                           int32_t nz, int32_t nt_local, int32_t mode, su3g_stream_t st) {
    return slab_sweep<float>(c, U, v, out, nx, ny, nz, nt_local, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_slab_nn_sweep_f64(su3g_comm_t c, const double* U, const double* v, double* out, int32_t nx, int32_t ny,
                           int32_t nz, int32_t nt_local, int32_t mode, su3g_stream_t st) {
    return slab_sweep<double>(c, U, v, out, nx, ny, nz, nt_local, mode, reinterpret_cast<cudaStream_t>(st));
}

}  // extern "C"
