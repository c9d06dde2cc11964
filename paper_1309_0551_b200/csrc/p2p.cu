// Fused compute + halo push over NVLink for the t-slab NN sweep (BASELINE configs[4]).
//
// The NCCL schedule (comm.cu, slab.py) sends the two halo faces with separate
// send/recv kernels.  Here the kernel that computes a rank's boundary slices
// also delivers the NEXT application's halos straight into its neighbours'
// memory (peer pointers mapped with CUDA IPC), so no communication kernel or
// host round trip exists:
//
//   application e on rank r (stream-ordered):
//     k_p2p_boundary:  wait until this rank's halo window holds application e's
//                      halos (flags >= e+1, ld.acquire.sys); compute out on
//                      t = 0 and t = nt-1 from them; store out(t=0) into rank
//                      r-1's v_hi[(e+1)%2] and w = U_t^dag out(nt-1) into rank
//                      r+1's w_lo[(e+1)%2] (remote stores over NVLink); the
//                      last CTA to finish releases flag e+2 at both peers
//                      (st.release.sys after __threadfence_system).
//     interior:        slices [1, nt-1) with the ordinary kernels, while the
//                      peers' pushes for e+1 land in this rank's window.
//
// Ordering argument (no WAR hazard, no deadlock): a rank pushes into parity
// (e+1)%2 only after both neighbours released flag e+1, i.e. after they
// finished boundary(e-1), the last kernel that read that parity; boundary(e)
// only waits on boundary(e-1) of the neighbours, which never waits on anything
// later.  A fresh source vector is primed (k_p2p_prime) after a host barrier.
// The halo values are exactly the single-GPU kernel's operands (v of the
// neighbour slice; w = U_t^dag v with the same arithmetic), so the result is
// bit-identical to the periodic sweep.  With one rank the peer windows are the
// rank's own, which runs the whole protocol on a single GPU.
#include <algorithm>
#include <cstring>
#include <string>

#include "nn_site.cuh"

namespace su3g {

namespace {

constexpr size_t kCtrlBytes = 128;

struct Ctrl {
    unsigned long long flag_vhi;  // application whose v_hi halo is complete, + 1
    unsigned long long flag_wlo;  // same for w_lo
    unsigned int counter;         // CTAs of the running boundary/prime launch that finished pushing
    unsigned int error;           // 1: a wait timed out (the result of that launch is invalid)
};

size_t face_bytes(int64_t F, size_t esz) { return (size_t(6 * F) * esz + 127) / 128 * 128; }

template <typename T>
struct Window {  // device view of one rank's window
    T* vhi[2];
    T* wlo[2];
    Ctrl* ctrl;
};

template <typename T>
Window<T> window_at(void* base, int64_t F) {
    char* b = static_cast<char*>(base);
    const size_t fb = face_bytes(F, sizeof(T));
    Window<T> w;
    w.vhi[0] = reinterpret_cast<T*>(b);
    w.vhi[1] = reinterpret_cast<T*>(b + fb);
    w.wlo[0] = reinterpret_cast<T*>(b + 2 * fb);
    w.wlo[1] = reinterpret_cast<T*>(b + 3 * fb);
    w.ctrl = reinterpret_cast<Ctrl*>(b + 4 * fb);
    return w;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// bounded spin (about 20 s): a protocol bug reports through ctrl->error instead of hanging the GPU
__device__ __forceinline__ void wait_flags(Ctrl* c, unsigned long long need) {
    for (long long spin = 0; ld_acquire_sys(&c->flag_vhi) < need || ld_acquire_sys(&c->flag_wlo) < need; ++spin) {
        if (spin > (1LL << 27)) {
            atomicExch(&c->error, 1u);
            return;
        }
        __nanosleep(128);
    }
}

// after every CTA pushed: the last one resets the counter and releases `value` at both peers
__device__ __forceinline__ void signal_peers(Ctrl* local, Ctrl* lo, Ctrl* hi, unsigned long long value) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&local->counter, 1u);
        if (prev == gridDim.x - 1) {
            local->counter = 0;
            __threadfence_system();
            st_release_sys(&lo->flag_vhi, value);
            st_release_sys(&hi->flag_wlo, value);
        }
    }
}

template <typename T, bool FUSED>
__device__ __forceinline__ void push_w(const T* __restrict__ U, const T* vsrc, const Geom& g, int64_t s3, T* dst) {
    // w = U_t(x, nt-1)^dag v(x, nt-1), the single-GPU kernel's backward t operand
    T u[18], vv[6], w[6];
    ld_soa<T, 18>(U + (int64_t(g.nt - 1) * 72 + 54) * g.F, g.F, s3, u);
#pragma unroll
    for (int c = 0; c < 6; ++c) vv[c] = vsrc[(int64_t(g.nt - 1) * 6 + c) * g.F + s3];
    amv<T, FUSED>(u, vv, w);
#pragma unroll
    for (int c = 0; c < 6; ++c) dst[c * g.F + s3] = w[c];
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256)
    k_p2p_prime(const T* __restrict__ U, const T* __restrict__ v, Geom g, Window<T> me, Window<T> lo, Window<T> hi,
                long long epoch) {
    const int par = static_cast<int>(epoch & 1);
    for (int64_t s3 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s3 < g.F; s3 += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 6; ++c) lo.vhi[par][c * g.F + s3] = v[c * g.F + s3];  // v(t=0) -> rank r-1
        push_w<T, FUSED>(U, v, g, s3, hi.wlo[par]);                                // w(nt-1) -> rank r+1
    }
    signal_peers(me.ctrl, lo.ctrl, hi.ctrl, static_cast<unsigned long long>(epoch) + 1);
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256)
    k_p2p_boundary(const T* __restrict__ U, const T* __restrict__ v, T* out, Geom g, Window<T> me, Window<T> lo,
                   Window<T> hi, long long epoch) {
    if (threadIdx.x == 0) wait_flags(me.ctrl, static_cast<unsigned long long>(epoch) + 1);
    __syncthreads();
    const int par = static_cast<int>(epoch & 1), nxt = par ^ 1;
    const int nsl = g.nt == 1 ? 1 : 2;
    // grid-stride over the boundary sites: few, persistent CTAs, so few system-scope fences in signal_peers
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < nsl * g.F;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int t = idx < g.F ? 0 : g.nt - 1;
        const int64_t s3 = idx < g.F ? idx : idx - g.F;
        const int x = static_cast<int>(s3 % g.nx);
        const int y = static_cast<int>((s3 / g.nx) % g.ny);
        const int z = static_cast<int>(s3 / (int64_t(g.nx) * g.ny));
        nn_site<T, FUSED, false, true>(U, v, out, g, x, y, z, t, me.vhi[par], me.wlo[par]);
        // next application's halos, computed from this application's output (own thread's stores)
        if (t == 0) {
#pragma unroll
            for (int c = 0; c < 6; ++c) lo.vhi[nxt][c * g.F + s3] = out[c * g.F + s3];
        }
        if (t == g.nt - 1) push_w<T, FUSED>(U, out, g, s3, hi.wlo[nxt]);
    }
    signal_peers(me.ctrl, lo.ctrl, hi.ctrl, static_cast<unsigned long long>(epoch) + 2);
}

template <typename T>
int p2p_check(const char* what, const void* me, const void* lo, const void* hi, int nx, int ny, int nz, int nt,
              int mode) {
    if (!me || !lo || !hi) return fail_invalid(std::string(what) + ": null window");
    if (nx < 1 || ny < 1 || nz < 1 || nt < 1) return fail_invalid(std::string(what) + ": lattice extents must be >= 1");
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid(std::string(what) + ": mode must be SU3G_EXACT or SU3G_FMA");
    return SU3G_OK;
}

template <typename T>
int p2p_prime(const T* U, const T* v, int nx, int ny, int nz, int nt, void* me, void* lo, void* hi, long long epoch,
              int mode, cudaStream_t st) {
    if (int rc = p2p_check<T>("p2p_prime", me, lo, hi, nx, ny, nz, nt, mode)) return rc;
    if (!U || !v) return fail_invalid("p2p_prime: null pointer");
    if (epoch < 0) return fail_invalid("p2p_prime: epoch must be >= 0");
    const Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((g.F + 255) / 256, 4LL * device_info().num_sms)));
    const Window<T> wm = window_at<T>(me, g.F), wl = window_at<T>(lo, g.F), wh = window_at<T>(hi, g.F);
    if (mode == SU3G_FMA) k_p2p_prime<T, true><<<grid, 256, 0, st>>>(U, v, g, wm, wl, wh, epoch);
    else k_p2p_prime<T, false><<<grid, 256, 0, st>>>(U, v, g, wm, wl, wh, epoch);
    note_kernel("k_p2p_prime");
    return check_launch("p2p_prime");
}

template <typename T>
int p2p_sweep(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, void* me, void* lo, void* hi,
              long long epoch, int mode, cudaStream_t st) {
    if (int rc = p2p_check<T>("p2p_nn_sweep", me, lo, hi, nx, ny, nz, nt, mode)) return rc;
    if (!U || !v || !out) return fail_invalid("p2p_nn_sweep: null pointer");
    if (out == v) return fail_invalid("p2p_nn_sweep: out must not alias v");
    if (epoch < 0) return fail_invalid("p2p_nn_sweep: epoch must be >= 0");
    const Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int nsl = nt == 1 ? 1 : 2;
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((nsl * g.F + 255) / 256, 4LL * device_info().num_sms)));
    const Window<T> wm = window_at<T>(me, g.F), wl = window_at<T>(lo, g.F), wh = window_at<T>(hi, g.F);
    // boundary first: its pushes for application e+1 then overlap this rank's interior
    if (mode == SU3G_FMA) k_p2p_boundary<T, true><<<grid, 256, 0, st>>>(U, v, out, g, wm, wl, wh, epoch);
    else k_p2p_boundary<T, false><<<grid, 256, 0, st>>>(U, v, out, g, wm, wl, wh, epoch);
    if (int rc = check_launch("p2p_nn_sweep(boundary)")) return rc;
    if (nt > 2) {
        const int rc = sizeof(T) == 4
                           ? su3g_nn_sweep_f32(reinterpret_cast<const float*>(U), reinterpret_cast<const float*>(v),
                                               reinterpret_cast<float*>(out), nx, ny, nz, nt, 1, nt - 1, nullptr,
                                               nullptr, mode, st)
                           : su3g_nn_sweep_f64(reinterpret_cast<const double*>(U), reinterpret_cast<const double*>(v),
                                               reinterpret_cast<double*>(out), nx, ny, nz, nt, 1, nt - 1, nullptr,
                                               nullptr, mode, st);
        if (rc) return rc;
    }
    return SU3G_OK;
}

}  // namespace

}  // namespace su3g

using namespace su3g;

extern "C" {

int64_t su3g_p2p_window_bytes(int32_t nx, int32_t ny, int32_t nz, int32_t elem_size) {
    if (nx < 1 || ny < 1 || nz < 1 || (elem_size != 4 && elem_size != 8)) return -1;
    return int64_t(4 * face_bytes(int64_t(nx) * ny * nz, size_t(elem_size)) + kCtrlBytes);
}

int64_t su3g_p2p_ctrl_offset(int32_t nx, int32_t ny, int32_t nz, int32_t elem_size) {
    if (nx < 1 || ny < 1 || nz < 1 || (elem_size != 4 && elem_size != 8)) return -1;
    return int64_t(4 * face_bytes(int64_t(nx) * ny * nz, size_t(elem_size)));
}

int su3g_ipc_get_handle(const void* dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out) return fail_invalid("ipc_get_handle: null pointer");
    cudaIpcMemHandle_t h;
    if (cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr))) {
        set_error(std::string("ipc_get_handle: ") + cudaGetErrorString(e));
        return static_cast<int>(e);
    }
    std::memcpy(handle_out, &h, sizeof(h));
    return SU3G_OK;
}

int su3g_ipc_open_handle(const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return fail_invalid("ipc_open_handle: null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess)) {
        set_error(std::string("ipc_open_handle: ") + cudaGetErrorString(e));
        return static_cast<int>(e);
    }
    return SU3G_OK;
}

int su3g_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return SU3G_OK;
    if (cudaError_t e = cudaIpcCloseMemHandle(dev_ptr)) {
        set_error(std::string("ipc_close: ") + cudaGetErrorString(e));
        return static_cast<int>(e);
    }
    return SU3G_OK;
}

int su3g_p2p_prime_f32(const float* U, const float* v, int32_t nx, int32_t ny, int32_t nz, int32_t nt, void* win,
                       void* win_lo, void* win_hi, int64_t epoch, int32_t mode, su3g_stream_t st) {
    return p2p_prime<float>(U, v, nx, ny, nz, nt, win, win_lo, win_hi, epoch, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_p2p_prime_f64(const double* U, const double* v, int32_t nx, int32_t ny, int32_t nz, int32_t nt, void* win,
                       void* win_lo, void* win_hi, int64_t epoch, int32_t mode, su3g_stream_t st) {
    return p2p_prime<double>(U, v, nx, ny, nz, nt, win, win_lo, win_hi, epoch, mode,
                             reinterpret_cast<cudaStream_t>(st));
}
int su3g_p2p_nn_sweep_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                          void* win, void* win_lo, void* win_hi, int64_t epoch, int32_t mode, su3g_stream_t st) {
    return p2p_sweep<float>(U, v, out, nx, ny, nz, nt, win, win_lo, win_hi, epoch, mode,
                            reinterpret_cast<cudaStream_t>(st));
}
int su3g_p2p_nn_sweep_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz,
                          int32_t nt, void* win, void* win_lo, void* win_hi, int64_t epoch, int32_t mode,
                          su3g_stream_t st) {
    return p2p_sweep<double>(U, v, out, nx, ny, nz, nt, win, win_lo, win_hi, epoch, mode,
                             reinterpret_cast<cudaStream_t>(st));
}

}  // extern "C"
