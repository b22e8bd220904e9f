// p2p_exchange.cu -- the split-L exchange over peer memory (SURVEY.md 8(e) phase 2), an alternative
// to the NCCL all_gather of dist.summarize_by_length.
//
// Every rank owns a receive buffer (recv_o [world][B,H,S,d] f32, recv_lse [world][B,H,S] f32), a
// flags array and an acks array (uint32 [world] each) and a device epoch counter.  The buffers are
// shared with the other ranks of the node through CUDA IPC (vista_ipc_*), so a rank holds device
// pointers to every rank's buffers; stores to a peer's pointer travel over NVLink / NVSwitch.
// One exchange step, all on the caller's stream (no host synchronization, CUDA-graph capturable:
// the epoch lives in device memory):
//   push    wait until every peer has acknowledged the previous epoch (acks[r] >= epoch), then
//           store this rank's partial into slot `rank` of every rank's receive buffer
//   signal  epoch += 1; flags_r[rank] = epoch on every rank r (system-scope release)
//   wait    until flags[r] == epoch for every r (acquire): the local receive buffer holds all
//           partials -> vista_summarize_merge over it
//   ack     acks_r[rank] = epoch on every rank r: this rank has consumed the epoch; the peers may
//           overwrite its receive buffer in the next push
// Deadlock-free by construction: every rank runs push, signal, wait, merge, ack in stream order, and
// a push of epoch e+1 only waits for acks of e, which every rank publishes after its own wait for e.
// Fused form (softmax): vista_summarize_partial_peers replaces the push -- the ack wait runs first,
// then the partial's own epilogue / slot-merge / empty-user stores go straight into every rank's
// receive buffer (slot `rank`) over NVLink; signal, wait, merge and ack as above.
// Waits spin with a 4-second watchdog trap (a protocol bug becomes a launch error, not a hang).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "internal.h"

namespace vista {
namespace {

struct XPtrs {
    float* o[kMaxExchangeRanks];
    float* l[kMaxExchangeRanks];
    uint32_t* f[kMaxExchangeRanks];
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// spin until (int32)(p[0] - want) >= 0; trap after 4 s
__device__ __forceinline__ void spin_until_ge(const uint32_t* p, uint32_t want) {
    if ((int32_t)(ld_acquire_sys(p) - want) >= 0) return;
    const uint64_t t0 = gtimer();
    while ((int32_t)(ld_acquire_sys(p) - want) < 0) {
        if (gtimer() - t0 > 4000000000ull) __trap();
    }
}

// acks: this rank's ack array (acks[r] written by rank r); the epoch before this step's signal
__global__ void xpush_kernel(const float4* __restrict__ src_o, size_t n_o4, const float* __restrict__ src_l,
                             size_t n_l, XPtrs dst, int world, int rank, const uint32_t* acks,
                             const uint32_t* epoch) {
    if (threadIdx.x < 32) {
        const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(epoch);
        if ((int)threadIdx.x < world) spin_until_ge(acks + threadIdx.x, e);  // every peer consumed epoch e
    }
    __syncthreads();
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_o4; i += stride) {
        const float4 v = __ldg(src_o + i);
        for (int r = 0; r < world; ++r) reinterpret_cast<float4*>(dst.o[r])[(size_t)rank * n_o4 + i] = v;
    }
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_l; i += stride) {
        const float v = __ldg(src_l + i);
        for (int r = 0; r < world; ++r) dst.l[r][(size_t)rank * n_l + i] = v;
    }
}

__global__ void xsignal_kernel(XPtrs dst, int world, int rank, uint32_t* epoch) {
    if (threadIdx.x != 0) return;
    const uint32_t e = epoch[0] + 1;
    epoch[0] = e;
    __threadfence_system();  // the push kernel's stores (completed before this kernel) are visible system-wide
    for (int r = 0; r < world; ++r) st_release_sys(dst.f[r] + rank, e);
}

__global__ void xwait_kernel(const uint32_t* flags, int world, const uint32_t* epoch) {
    const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(epoch);
    if ((int)threadIdx.x < world) spin_until_ge(flags + threadIdx.x, e);
    __threadfence_system();
}

__global__ void xack_kernel(XPtrs dst, int world, int rank, const uint32_t* epoch) {
    if (threadIdx.x != 0) return;
    const uint32_t e = epoch[0];
    __threadfence_system();  // the merge's reads of the receive buffer (completed before) come first
    for (int r = 0; r < world; ++r) st_release_sys(dst.f[r] + rank, e);
}

// the fused exchange (vista_summarize_partial_peers): before the partial's kernels store into the
// peers' receive buffers, every peer must have consumed the previous epoch
__global__ void xwait_acks_kernel(const uint32_t* acks, int world, const uint32_t* epoch) {
    const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(epoch);
    if ((int)threadIdx.x < world) spin_until_ge(acks + threadIdx.x, e);
}

bool fill(XPtrs& x, int world, float* const* o, float* const* l, uint32_t* const* f) {
    std::memset(&x, 0, sizeof(x));
    for (int r = 0; r < world; ++r) {
        if ((o && !o[r]) || (l && !l[r]) || (f && !f[r])) return false;
        if (o) x.o[r] = o[r];
        if (l) x.l[r] = l[r];
        if (f) x.f[r] = f[r];
    }
    return true;
}

}  // namespace

cudaError_t launch_exchange_wait_acks(int world, const uint32_t* acks, const uint32_t* epoch, cudaStream_t stream) {
    xwait_acks_kernel<<<1, 32, 0, stream>>>(acks, world, epoch);
    return cudaGetLastError();
}

}  // namespace vista

using namespace vista;

extern "C" {

vista_status_t vista_ipc_get_handle(const void* dptr, void* handle) {
    if (!dptr || !handle) return VISTA_ERR_NULL;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)) != cudaSuccess) return VISTA_ERR_CUDA;
    static_assert(sizeof(h) == VISTA_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    return VISTA_OK;
}

vista_status_t vista_ipc_open_handle(const void* handle, void** dptr) {
    if (!handle || !dptr) return VISTA_ERR_NULL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return VISTA_ERR_CUDA;
    return VISTA_OK;
}

vista_status_t vista_ipc_close(void* dptr) {
    if (!dptr) return VISTA_ERR_NULL;
    return cudaIpcCloseMemHandle(dptr) == cudaSuccess ? VISTA_OK : VISTA_ERR_CUDA;
}

vista_status_t vista_exchange_push(int32_t world, int32_t rank, const float* part_o, int64_t n_o,
                                   const float* part_lse, int64_t n_lse, float* const* recv_o,
                                   float* const* recv_lse, const uint32_t* acks, const uint32_t* epoch,
                                   void* stream) {
    if (world < 1 || world > kMaxExchangeRanks || rank < 0 || rank >= world || n_o < 0 || n_lse < 0 || n_o % 4)
        return VISTA_ERR_INVALID;
    if (!part_o || !recv_o || !acks || !epoch || (n_lse > 0 && (!part_lse || !recv_lse))) return VISTA_ERR_NULL;
    if (reinterpret_cast<uintptr_t>(part_o) & 15) return VISTA_ERR_MISALIGNED;
    XPtrs x;
    if (!fill(x, world, recv_o, n_lse > 0 ? recv_lse : nullptr, nullptr)) return VISTA_ERR_NULL;
    for (int r = 0; r < world; ++r)
        if (reinterpret_cast<uintptr_t>(x.o[r]) & 15) return VISTA_ERR_MISALIGNED;
    const size_t n4 = (size_t)n_o / 4;
    int grid = (int)std::min<size_t>((n4 + 255) / 256, 4 * 148);
    if (grid < 1) grid = 1;
    xpush_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const float4*>(part_o), n4, part_lse, (size_t)n_lse, x, world, rank, acks, epoch);
    count_launches(1);
    return cudaGetLastError() == cudaSuccess ? VISTA_OK : VISTA_ERR_CUDA;
}

vista_status_t vista_exchange_signal(int32_t world, int32_t rank, uint32_t* const* flags, uint32_t* epoch,
                                     void* stream) {
    if (world < 1 || world > kMaxExchangeRanks || rank < 0 || rank >= world) return VISTA_ERR_INVALID;
    if (!flags || !epoch) return VISTA_ERR_NULL;
    XPtrs x;
    if (!fill(x, world, nullptr, nullptr, flags)) return VISTA_ERR_NULL;
    xsignal_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, world, rank, epoch);
    count_launches(1);
    return cudaGetLastError() == cudaSuccess ? VISTA_OK : VISTA_ERR_CUDA;
}

vista_status_t vista_exchange_wait(int32_t world, const uint32_t* flags, const uint32_t* epoch, void* stream) {
    if (world < 1 || world > kMaxExchangeRanks) return VISTA_ERR_INVALID;
    if (!flags || !epoch) return VISTA_ERR_NULL;
    xwait_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, world, epoch);
    count_launches(1);
    return cudaGetLastError() == cudaSuccess ? VISTA_OK : VISTA_ERR_CUDA;
}

vista_status_t vista_exchange_ack(int32_t world, int32_t rank, uint32_t* const* acks, const uint32_t* epoch,
                                  void* stream) {
    if (world < 1 || world > kMaxExchangeRanks || rank < 0 || rank >= world) return VISTA_ERR_INVALID;
    if (!acks || !epoch) return VISTA_ERR_NULL;
    XPtrs x;
    if (!fill(x, world, nullptr, nullptr, acks)) return VISTA_ERR_NULL;
    xack_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, world, rank, epoch);
    count_launches(1);
    return cudaGetLastError() == cudaSuccess ? VISTA_OK : VISTA_ERR_CUDA;
}

}  // extern "C"
