// vista_abi.cu -- the C ABI of libvista (include/vista.h): validation, workspace planning,
// dispatch by shape, launch sequencing.  All device work is enqueued on the caller's stream;
// nothing here synchronizes (except the debug entry vista_check_offsets).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "internal.h"

using namespace vista;

namespace {

thread_local char g_cuda_err[256] = "";
thread_local cudaEvent_t g_ev_start = nullptr, g_ev_stop = nullptr;
std::atomic<unsigned long long> g_launches{0};

// Launch the dominant kernel of a call, bracketed by the armed timing events if any.
template <typename F>
cudaError_t timed_main(cudaStream_t s, F&& launch) {
    cudaEvent_t a = g_ev_start, b = g_ev_stop;
    g_ev_start = g_ev_stop = nullptr;
    // under stream capture the records become external event nodes: the graph records them at
    // every replay (a plain record in a capture is only an internal dependency)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const unsigned flags =
        (a || b) && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive
            ? cudaEventRecordExternal
            : cudaEventRecordDefault;
    cudaError_t e;
    if (a && (e = cudaEventRecordWithFlags(a, s, flags)) != cudaSuccess) return e;
    e = launch();
    if (e == cudaSuccess && b) e = cudaEventRecordWithFlags(b, s, flags);
    return e;
}

vista_status_t cuda_fail(cudaError_t e) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return VISTA_ERR_CUDA;
}

int device_sms() {
    static std::mutex mu;
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    std::lock_guard<std::mutex> lock(mu);
    if (!cache[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

vista_status_t validate_desc(const vista_desc_t* d) {
    if (!d) return VISTA_ERR_NULL;
    if (d->abi_version != VISTA_ABI_VERSION) return VISTA_ERR_INVALID;
    if (d->num_users < 0 || d->num_summary < 1 || d->num_heads < 1) return VISTA_ERR_INVALID;
    if (d->in_dtype != VISTA_F32 && d->in_dtype != VISTA_BF16) return VISTA_ERR_INVALID;
    if (d->out_dtype != VISTA_F32 && d->out_dtype != VISTA_BF16) return VISTA_ERR_INVALID;
    if (d->attn != VISTA_SOFTMAX && d->attn != VISTA_QLA) return VISTA_ERR_INVALID;
    if (d->head_dim != 32 && d->head_dim != 64 && d->head_dim != 128) return VISTA_ERR_UNSUPPORTED;
    if (d->attn == VISTA_SOFTMAX && !isnan(d->softmax_scale) && !(d->softmax_scale > 0.f && isfinite(d->softmax_scale)))
        return VISTA_ERR_INVALID;
    if (d->attn == VISTA_QLA) {
        for (int phi : {d->qla_phi1, d->qla_phi2})
            if (phi < VISTA_ACT_IDENTITY || phi > VISTA_ACT_SHIFTED_ELU) return VISTA_ERR_INVALID;
        if (d->qla_normalize != 0 && d->qla_normalize != 1) return VISTA_ERR_INVALID;
    }
    if (d->q_user_stride < 0) return VISTA_ERR_INVALID;
    if (d->q_user_stride > 0 && d->q_user_stride < (int64_t)d->num_summary * d->num_heads * d->head_dim)
        return VISTA_ERR_INVALID;
    return VISTA_OK;
}

Problem make_problem(const vista_desc_t* d, int64_t total_len) {
    Problem p{};
    p.B = d->num_users;
    p.S = d->num_summary;
    p.H = d->num_heads;
    p.d = d->head_dim;
    p.in_bf16 = d->in_dtype == VISTA_BF16;
    p.attn = d->attn;
    p.scale = isnan(d->softmax_scale) ? 1.0f / sqrtf((float)d->head_dim) : d->softmax_scale;
    p.phi1 = d->qla_phi1;
    p.phi2 = d->qla_phi2;
    p.normalize = d->qla_normalize;
    p.q_user_stride = d->q_user_stride;
    p.total_len = total_len;
    p.num_sms = std::min(device_sms(), kMaxPersistentCtas);  // bounds the merge's slot run list
    return p;
}

}  // namespace

namespace vista {
void count_launches(unsigned n) { g_launches += n; }
}  // namespace vista

namespace vista {

cudaError_t set_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const auto key = std::make_tuple(fn, dev, bytes);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

Path choose_path(const Problem& p) {
    const bool tma_ok = p.in_bf16 && p.d == 128 && p.total_len < (int64_t(1) << 31) && (p.q_user_stride % 8) == 0;
    if (p.attn == VISTA_SOFTMAX) return (tma_ok && p.S % 128 == 0) ? PATH_SM100_SOFTMAX : PATH_SIMT_SOFTMAX;
    return tma_ok ? PATH_SM100_QLA : PATH_SIMT_QLA;
}

int sm100_softmax_cluster(int S);
int sm100_softmax_num_clusters(const Problem& p);

Workspace plan_workspace(const Problem& p, bool partial) {
    (void)partial;
    Workspace w{};
    const Path path = choose_path(p);
    size_t off = 0;
    w.num_ctas = 0;
    w.rows_per_unit = 0;
    if (path == PATH_SM100_SOFTMAX || path == PATH_SM100_QLA) {
        w.num_ctas = p.num_sms;
        w.rows_per_unit = 128;
        if (path == PATH_SM100_SOFTMAX) {  // persistent grid of clusters, C * 128 query rows per unit
            w.num_ctas = sm100_softmax_num_clusters(p);
            w.rows_per_unit = sm100_softmax_cluster(p.S) * 128;
        }
    }
    w.uts_off = off;
    off = align256(off + (size_t)(p.B + 1) * sizeof(int64_t));
    w.slot_unit_off = off;
    off = align256(off + (size_t)2 * w.num_ctas * sizeof(int));
    w.slot_o_off = off;
    off = align256(off + (size_t)2 * w.num_ctas * w.rows_per_unit * 128 * sizeof(float));
    w.slot_lse_off = off;
    off = align256(off + (size_t)2 * w.num_ctas * w.rows_per_unit * sizeof(float));
    w.zbuf_off = off;
    if (p.attn == VISTA_QLA) off = align256(off + (size_t)p.B * p.H * p.d * p.d * sizeof(float));
    w.fin_off = off;
    if (p.attn == VISTA_QLA && qla_finalize_uses_tc(p)) off = align256(off + sm100_qla_finalize_workspace(p));
    w.total = off;
    return w;
}

}  // namespace vista

extern "C" {

int vista_abi_version(void) { return VISTA_ABI_VERSION; }

const char* vista_status_string(int s) {
    switch (s) {
        case VISTA_OK: return "VISTA_OK";
        case VISTA_ERR_NULL: return "VISTA_ERR_NULL";
        case VISTA_ERR_INVALID: return "VISTA_ERR_INVALID";
        case VISTA_ERR_UNSUPPORTED: return "VISTA_ERR_UNSUPPORTED";
        case VISTA_ERR_MISALIGNED: return "VISTA_ERR_MISALIGNED";
        case VISTA_ERR_WORKSPACE: return "VISTA_ERR_WORKSPACE";
        case VISTA_ERR_CUDA: return "VISTA_ERR_CUDA";
        case VISTA_ERR_OFFSETS: return "VISTA_ERR_OFFSETS";
    }
    return "VISTA_ERR_UNKNOWN";
}

const char* vista_last_cuda_error(void) { return g_cuda_err; }

const char* vista_dispatch_name(const vista_desc_t* desc) {
    if (validate_desc(desc) != VISTA_OK) return nullptr;
    Problem p = make_problem(desc, 0);
    switch (choose_path(p)) {
        case PATH_SM100_SOFTMAX: return "sm100_softmax";
        case PATH_SM100_QLA: return "sm100_qla";
        case PATH_SIMT_SOFTMAX: return "simt_softmax";
        case PATH_SIMT_QLA: return "simt_qla";
        default: return nullptr;
    }
}

vista_status_t vista_summarize_workspace_size(const vista_desc_t* desc, int64_t total_len, size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (total_len < 0) return VISTA_ERR_INVALID;
    Problem p = make_problem(desc, total_len);
    *bytes = plan_workspace(p, false).total;
    return VISTA_OK;
}

static vista_status_t run(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                          const int64_t* offsets, int64_t total_len, OutSpec outs, void* workspace,
                          size_t workspace_bytes, void* stream, const PeerSpec* peers = nullptr) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (total_len < 0) return VISTA_ERR_INVALID;
    if (!q || !offsets || (!outs.out && desc->num_users > 0)) return VISTA_ERR_NULL;  // B = 0: nothing to write
    if (total_len > 0 && (!k || !v)) return VISTA_ERR_NULL;
    if (outs.mode == OUT_PARTIAL && desc->attn == VISTA_SOFTMAX && !outs.lse && desc->num_users > 0)
        return VISTA_ERR_NULL;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(outs.out)) return VISTA_ERR_MISALIGNED;
    if (outs.lse && (reinterpret_cast<uintptr_t>(outs.lse) & 3)) return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, total_len);
    p.q = q;
    p.k = k;
    p.v = v;
    p.offsets = offsets;
    p.outs = outs;
    if (peers) {
        p.peers = *peers;  // the fused exchange: tcgen05 paths only
        const Path pp = choose_path(p);
        if (pp != PATH_SM100_SOFTMAX && pp != PATH_SM100_QLA) return VISTA_ERR_UNSUPPORTED;
    }
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0) return VISTA_OK;
    const bool partial = outs.mode == OUT_PARTIAL;
    const Workspace w = plan_workspace(p, partial);
    if (w.total > 0 && (!workspace || workspace_bytes < w.total)) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    char* ws = reinterpret_cast<char*>(workspace);
    cudaError_t e = cudaSuccess;
    int nlaunch = 0;
    switch (choose_path(p)) {
        case PATH_SM100_SOFTMAX: {
            if ((e = launch_user_tiles(p, reinterpret_cast<int64_t*>(ws + w.uts_off), nullptr)) != cudaSuccess)
                break;
            if ((e = timed_main(p.stream, [&] { return launch_sm100_softmax(p, w, ws); })) != cudaSuccess) break;
            e = launch_merge_softmax_slots(p, w, ws);
            nlaunch = 3;
            break;
        }
        case PATH_SM100_QLA: {
            if (!partial && qla_finalize_uses_tc(p)) {
                // fused: state epilogue / slot merge write the finalize GEMM's W operand directly
                uint8_t* wbuf = reinterpret_cast<uint8_t*>(ws + w.fin_off);
                if ((e = launch_user_tiles(p, reinterpret_cast<int64_t*>(ws + w.uts_off), nullptr)) != cudaSuccess) break;
                if ((e = timed_main(p.stream, [&] { return launch_sm100_qla_state(p, w, ws, nullptr, wbuf); })) !=
                    cudaSuccess)
                    break;
                if ((e = launch_merge_qla_slots_w(p, w, ws, wbuf)) != cudaSuccess) break;
                e = launch_sm100_qla_finalize_fused(p, wbuf);
                nlaunch = 4;
                break;
            }
            float* zbuf = partial ? reinterpret_cast<float*>(outs.out) : reinterpret_cast<float*>(ws + w.zbuf_off);
            if ((e = launch_user_tiles(p, reinterpret_cast<int64_t*>(ws + w.uts_off), zbuf)) != cudaSuccess) break;
            if ((e = timed_main(p.stream, [&] { return launch_sm100_qla_state(p, w, ws, zbuf); })) != cudaSuccess) break;
            if ((e = launch_merge_qla_slots(p, w, ws, zbuf)) != cudaSuccess) break;
            if (!partial) e = launch_qla_finalize(p, zbuf, 1, 0, nullptr, ws + w.fin_off);
            nlaunch = partial ? 3 : 4;
            break;
        }
        case PATH_SIMT_SOFTMAX:
            e = timed_main(p.stream, [&] { return launch_simt_softmax(p); });
            nlaunch = 1;
            break;
        case PATH_SIMT_QLA: {
            float* zbuf = partial ? reinterpret_cast<float*>(outs.out) : reinterpret_cast<float*>(ws + w.zbuf_off);
            if ((e = timed_main(p.stream, [&] { return launch_simt_qla_state(p, zbuf); })) != cudaSuccess) break;
            if (!partial) e = launch_qla_finalize(p, zbuf, 1, 0, nullptr, ws + w.fin_off);
            nlaunch = partial ? 1 : 2;
            break;
        }
        default: return VISTA_ERR_UNSUPPORTED;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += (unsigned long long)nlaunch;
    return VISTA_OK;
}

vista_status_t vista_summarize_fwd(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                   const int64_t* offsets, int64_t total_len, void* out, float* lse, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    OutSpec o{OUT_FINAL, desc->out_dtype == VISTA_BF16, out, desc->attn == VISTA_SOFTMAX ? lse : nullptr};
    return run(desc, q, k, v, offsets, total_len, o, workspace, workspace_bytes, stream);
}

vista_status_t vista_summarize_fwd_int8(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                        const int64_t* offsets, int64_t total_len, void* out, float* lse,
                                        int8_t* codes, float* scale, float* zero_point, void* workspace,
                                        size_t workspace_bytes, void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    if (desc->num_users > 0 && (!codes || !scale || !zero_point)) return VISTA_ERR_NULL;
    if (!aligned16(codes) || (reinterpret_cast<uintptr_t>(scale) & 3) || (reinterpret_cast<uintptr_t>(zero_point) & 3))
        return VISTA_ERR_MISALIGNED;
    OutSpec o{OUT_FINAL, desc->out_dtype == VISTA_BF16, out, desc->attn == VISTA_SOFTMAX ? lse : nullptr};
    // fused into the epilogues (softmax epilogue, slot merge, empty-user fill) on the tcgen05 softmax
    // path with a bf16, 32-B aligned out; otherwise the export kernel runs after the summarization
    Problem pp = validate_desc(desc) == VISTA_OK ? make_problem(desc, total_len) : Problem{};
    const bool fused = validate_desc(desc) == VISTA_OK && choose_path(pp) == PATH_SM100_SOFTMAX &&
                       desc->out_dtype == VISTA_BF16 && (reinterpret_cast<uintptr_t>(out) & 31) == 0;
    if (fused) {
        o.codes = codes;
        o.qscale = scale;
        o.qzp = zero_point;
    }
    vista_status_t st = run(desc, q, k, v, offsets, total_len, o, workspace, workspace_bytes, stream);
    if (st != VISTA_OK || fused || desc->num_users == 0) return st;
    const int64_t n = (int64_t)desc->num_users * desc->num_summary * desc->num_heads;
    cudaError_t e = launch_quantize_rows(n, desc->head_dim, desc->out_dtype == VISTA_BF16, out, codes, scale,
                                         zero_point, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += 1;
    return VISTA_OK;
}

vista_status_t vista_summarize_partial(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                       const int64_t* offsets, int64_t total_len, float* part_o, float* part_lse,
                                       void* workspace, size_t workspace_bytes, void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    OutSpec o{OUT_PARTIAL, 0, part_o, desc->attn == VISTA_SOFTMAX ? part_lse : nullptr};
    return run(desc, q, k, v, offsets, total_len, o, workspace, workspace_bytes, stream);
}

vista_status_t vista_summarize_partial_peers(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                             const int64_t* offsets, int64_t total_len, int32_t world, int32_t rank,
                                             float* const* recv_o, float* const* recv_lse, const uint32_t* acks,
                                             const uint32_t* epoch, void* workspace, size_t workspace_bytes,
                                             void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    if (world < 1 || world > kMaxExchangeRanks || rank < 0 || rank >= world) return VISTA_ERR_INVALID;
    const bool softmax = desc->attn == VISTA_SOFTMAX;
    if (!recv_o || (softmax && !recv_lse) || !acks || !epoch) return VISTA_ERR_NULL;
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    // per rank slot: softmax O_p [B,H,S,d] + lse_p [B,H,S]; QLA Z_p [B,H,d,d]
    const size_t n_l = softmax ? (size_t)desc->num_users * desc->num_heads * desc->num_summary : 0;
    const size_t n_o = softmax ? n_l * desc->head_dim
                               : (size_t)desc->num_users * desc->num_heads * desc->head_dim * desc->head_dim;
    PeerSpec pe{};
    pe.n = world;
    for (int r = 0; r < world; ++r) {
        if (!recv_o[r] || (softmax && !recv_lse[r])) return VISTA_ERR_NULL;
        if (!aligned16(recv_o[r]) || (softmax && (reinterpret_cast<uintptr_t>(recv_lse[r]) & 3)))
            return VISTA_ERR_MISALIGNED;
        pe.o[r] = recv_o[r] + (size_t)rank * n_o;
        pe.lse[r] = softmax ? recv_lse[r] + (size_t)rank * n_l : nullptr;
    }
    // this rank's own slot: the base the kernels' row offsets are taken from (and what the checks see)
    OutSpec o{OUT_PARTIAL, 0, pe.o[rank], pe.lse[rank]};
    if (total_len < 0) return VISTA_ERR_INVALID;
    const Path path = desc->num_users > 0 ? choose_path(make_problem(desc, total_len)) : PATH_NONE;
    if (desc->num_users > 0 && path != PATH_SM100_SOFTMAX && path != PATH_SM100_QLA)
        return VISTA_ERR_UNSUPPORTED;  // the fused stores exist on the tcgen05 paths
    cudaError_t e = launch_exchange_wait_acks(world, acks, epoch, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    count_launches(1);
    return run(desc, q, k, v, offsets, total_len, o, workspace, workspace_bytes, stream, &pe);
}

// ---- shared key prefix: attention / state over [prefix keys; history] (reading R18).
// Workspace: [sub-run workspace | prefix result | history result | QLA finalize workspace].
namespace {
struct PrefixPlan {
    size_t sub_off, pre_off, preoff_off, main_off, main2_off, fin_off, total;
};
PrefixPlan plan_prefix(const vista_desc_t* desc, int64_t total_len, int64_t P) {
    PrefixPlan pl{};
    vista_desc_t d1 = *desc;
    d1.num_users = 1;
    const Problem pm = make_problem(desc, total_len), p1 = make_problem(&d1, P);
    const size_t sub = std::max(plan_workspace(pm, true).total, plan_workspace(p1, true).total);
    const bool softmax = desc->attn == VISTA_SOFTMAX;
    const size_t B = (size_t)pm.B, H = (size_t)pm.H, S = (size_t)pm.S, d = (size_t)pm.d;
    size_t off = 0;
    pl.sub_off = off;
    off = align256(off + sub);
    pl.pre_off = off;  // softmax: opre [H,S,d] + lpre [H,S]; QLA: zpre [H,d,d]
    off = align256(off + (softmax ? (H * S * d + H * S) : H * d * d) * sizeof(float));
    pl.preoff_off = off;
    off = align256(off + 2 * sizeof(int64_t));
    pl.main_off = off;  // softmax: o [B,H,S,d]; QLA: z [B,H,d,d]
    off = align256(off + (softmax ? B * H * S * d : B * H * d * d) * sizeof(float));
    pl.main2_off = off;  // softmax: lse [B,H,S]; QLA: user_len [B]
    off = align256(off + (softmax ? B * H * S * sizeof(float) : B * sizeof(int64_t)));
    pl.fin_off = off;
    if (!softmax && qla_finalize_uses_tc(pm)) off = align256(off + sm100_qla_finalize_workspace(pm));
    pl.total = off;
    return pl;
}
}  // namespace

vista_status_t vista_summarize_prefix_workspace_size(const vista_desc_t* desc, int64_t total_len, int64_t prefix_len,
                                                     size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (total_len < 0 || prefix_len < 0) return VISTA_ERR_INVALID;
    if (prefix_len == 0) return vista_summarize_workspace_size(desc, total_len, bytes);
    *bytes = plan_prefix(desc, total_len, prefix_len).total;
    return VISTA_OK;
}

static vista_status_t run_prefix(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                 const int64_t* offsets, int64_t total_len, const void* kp, const void* vp,
                                 int64_t P, OutSpec outs, void* workspace, size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (P < 0 || total_len < 0) return VISTA_ERR_INVALID;
    if (P == 0) return run(desc, q, k, v, offsets, total_len, outs, workspace, workspace_bytes, stream);
    if (!kp || !vp) return VISTA_ERR_NULL;
    if (!aligned16(kp) || !aligned16(vp)) return VISTA_ERR_MISALIGNED;
    if (desc->q_user_stride != 0) return VISTA_ERR_UNSUPPORTED;  // the prefix result is shared by all users
    if (!q || !offsets || !outs.out) return VISTA_ERR_NULL;
    if (outs.mode == OUT_PARTIAL && desc->attn == VISTA_SOFTMAX && !outs.lse) return VISTA_ERR_NULL;
    if (desc->num_users == 0) return VISTA_OK;
    const PrefixPlan pl = plan_prefix(desc, total_len, P);
    if (!workspace || workspace_bytes < pl.total) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    char* ws = reinterpret_cast<char*>(workspace);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t sub_bytes = pl.pre_off - pl.sub_off;
    vista_desc_t d1 = *desc;
    d1.num_users = 1;
    int64_t* pre_offsets = reinterpret_cast<int64_t*>(ws + pl.preoff_off);
    cudaError_t e = launch_write_prefix_offsets(pre_offsets, P, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += 1;
    Problem pm = make_problem(desc, total_len);
    pm.q = q;
    pm.offsets = offsets;
    pm.outs = outs;
    pm.stream = s;
    if (desc->attn == VISTA_SOFTMAX) {
        float* opre = reinterpret_cast<float*>(ws + pl.pre_off);
        float* lpre = opre + (size_t)pm.H * pm.S * pm.d;
        float* o = reinterpret_cast<float*>(ws + pl.main_off);
        float* l = reinterpret_cast<float*>(ws + pl.main2_off);
        st = run(&d1, q, kp, vp, pre_offsets, P, OutSpec{OUT_PARTIAL, 0, opre, lpre}, ws + pl.sub_off, sub_bytes, stream);
        if (st != VISTA_OK) return st;
        st = run(desc, q, k, v, offsets, total_len, OutSpec{OUT_PARTIAL, 0, o, l}, ws + pl.sub_off, sub_bytes, stream);
        if (st != VISTA_OK) return st;
        e = launch_merge_prefix(pm, o, l, opre, lpre);
    } else {
        float* zpre = reinterpret_cast<float*>(ws + pl.pre_off);
        const bool partial = outs.mode == OUT_PARTIAL;
        float* z = partial ? reinterpret_cast<float*>(outs.out) : reinterpret_cast<float*>(ws + pl.main_off);
        int64_t* user_len = partial ? nullptr : reinterpret_cast<int64_t*>(ws + pl.main2_off);
        st = run(&d1, q, kp, vp, pre_offsets, P, OutSpec{OUT_PARTIAL, 0, zpre, nullptr}, ws + pl.sub_off, sub_bytes,
                 stream);
        if (st != VISTA_OK) return st;
        st = run(desc, q, k, v, offsets, total_len, OutSpec{OUT_PARTIAL, 0, z, nullptr}, ws + pl.sub_off, sub_bytes,
                 stream);
        if (st != VISTA_OK) return st;
        if ((e = launch_add_prefix_state(pm, z, zpre, P, user_len)) == cudaSuccess && !partial) {
            g_launches += 1;
            e = launch_qla_finalize(pm, z, 1, 0, user_len, ws + pl.fin_off);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += 1;
    return VISTA_OK;
}

vista_status_t vista_summarize_fwd_prefix(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                          const int64_t* offsets, int64_t total_len, const void* k_prefix,
                                          const void* v_prefix, int64_t prefix_len, void* out, float* lse,
                                          void* workspace, size_t workspace_bytes, void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    OutSpec o{OUT_FINAL, desc->out_dtype == VISTA_BF16, out, desc->attn == VISTA_SOFTMAX ? lse : nullptr};
    return run_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, prefix_len, o, workspace, workspace_bytes,
                      stream);
}

vista_status_t vista_summarize_partial_prefix(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                              const int64_t* offsets, int64_t total_len, const void* k_prefix,
                                              const void* v_prefix, int64_t prefix_len, float* part_o,
                                              float* part_lse, void* workspace, size_t workspace_bytes, void* stream) {
    if (!desc) return VISTA_ERR_NULL;
    OutSpec o{OUT_PARTIAL, 0, part_o, desc->attn == VISTA_SOFTMAX ? part_lse : nullptr};
    return run_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, prefix_len, o, workspace, workspace_bytes,
                      stream);
}

// ---- backward (NEXT-2).  QLA: recompute Z (forward partial pass), per-unit dW / dZ / dQ, dK / dV.
// Workspace: [forward sub-run | Z | dZ | dZ bf16 operands (tcgen05 path) | per-user dQ (shared seeds)].
namespace {
struct BwdPlan {
    size_t sub_off, z_off, dz_off, dzop_off, abuf_off, dqu_off, total;
};
BwdPlan plan_bwd(const Problem& p) {
    BwdPlan b{};
    const size_t B = (size_t)p.B, H = (size_t)p.H, S = (size_t)p.S, d = (size_t)p.d;
    size_t off = 0;
    b.sub_off = off;
    off = align256(off + plan_workspace(p, true).total);
    b.z_off = off;
    off = align256(off + B * H * d * d * sizeof(float));
    b.dz_off = off;
    off = align256(off + B * H * d * d * sizeof(float));
    b.dzop_off = off;
    if (qla_bwd_uses_tc(p)) off = align256(off + B * H * d * d * 2);
    b.abuf_off = off;
    if (qla_bwd_uses_tc(p) && p.S % 128 == 0) off = align256(off + qla_prep_q_bytes(p));
    b.dqu_off = off;
    if (p.q_user_stride == 0) off = align256(off + B * S * H * d * sizeof(float));
    b.total = off;
    return b;
}
}  // namespace

vista_status_t vista_summarize_bwd_workspace_size(const vista_desc_t* desc, int64_t total_len, size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (total_len < 0) return VISTA_ERR_INVALID;
    const Problem p = make_problem(desc, total_len);
    if (desc->attn == VISTA_SOFTMAX) {
        *bytes = softmax_bwd_supported(p, desc->out_dtype == VISTA_BF16) ? softmax_bwd_workspace(p)
                                                                         : softmax_bwd_simt_workspace(p);
        return VISTA_OK;
    }
    *bytes = plan_bwd(p).total;
    return VISTA_OK;
}

static vista_status_t qla_bwd(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                              const int64_t* offsets, int64_t total_len, const float* z_saved, const void* dout,
                              float* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream);

vista_status_t vista_summarize_bwd_qla_saved(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                             const int64_t* offsets, int64_t total_len, const float* z_saved,
                                             const void* dout, float* dq, void* dk, void* dv, void* workspace,
                                             size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (desc->attn != VISTA_QLA) return VISTA_ERR_INVALID;
    if (!z_saved) return VISTA_ERR_NULL;
    if (!aligned16(z_saved)) return VISTA_ERR_MISALIGNED;
    return qla_bwd(desc, q, k, v, offsets, total_len, z_saved, dout, dq, dk, dv, workspace, workspace_bytes, stream);
}

vista_status_t vista_summarize_bwd(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                                   const int64_t* offsets, int64_t total_len, const void* out, const float* lse,
                                   const void* dout, float* dq, void* dk, void* dv, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (total_len < 0) return VISTA_ERR_INVALID;
    if (desc->attn == VISTA_SOFTMAX) {
        if (!q || !offsets || !dout || !dq || !out || !lse) return VISTA_ERR_NULL;
        if (total_len > 0 && (!k || !v || !dk || !dv)) return VISTA_ERR_NULL;
        if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(out) ||
            !aligned16(lse) || !aligned16(dq) || !aligned16(dk) || !aligned16(dv))
            return VISTA_ERR_MISALIGNED;
        Problem p = make_problem(desc, total_len);
        p.q = q;
        p.k = k;
        p.v = v;
        p.offsets = offsets;
        p.stream = reinterpret_cast<cudaStream_t>(stream);
        const bool dout_bf16 = desc->out_dtype == VISTA_BF16;
        const bool tc = softmax_bwd_supported(p, dout_bf16);
        if (p.B == 0) return VISTA_OK;
        const size_t need = tc ? softmax_bwd_workspace(p) : softmax_bwd_simt_workspace(p);
        if (!workspace || workspace_bytes < need) return VISTA_ERR_WORKSPACE;
        if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
        cudaEvent_t ev_a = g_ev_start, ev_b = g_ev_stop;
        g_ev_start = g_ev_stop = nullptr;
        int nl = 0;
        cudaError_t e;
        if (tc) {
            e = launch_softmax_bwd(p, out, lse, dout, dq, dk, dv, reinterpret_cast<char*>(workspace), &nl, ev_a, ev_b);
        } else {  // CUDA cores: D, dK/dV (timed), dQ
            e = launch_softmax_bwd_simt(p, dout_bf16, out, lse, dout, dq, dk, dv, reinterpret_cast<char*>(workspace));
            nl = p.total_len > 0 ? 3 : 2;
        }
        if (e != cudaSuccess) return cuda_fail(e);
        g_launches += (unsigned long long)nl;
        return VISTA_OK;
    }
    return qla_bwd(desc, q, k, v, offsets, total_len, nullptr, dout, dq, dk, dv, workspace, workspace_bytes, stream);
}

static vista_status_t qla_bwd(const vista_desc_t* desc, const void* q, const void* k, const void* v,
                              const int64_t* offsets, int64_t total_len, const float* z_saved, const void* dout,
                              float* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream) {
    vista_status_t st = VISTA_OK;
    if (total_len < 0) return VISTA_ERR_INVALID;
    if (!q || !offsets || !dout || !dq) return VISTA_ERR_NULL;
    if (total_len > 0 && (!k || !v || !dk || !dv)) return VISTA_ERR_NULL;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq) || !aligned16(dk) ||
        !aligned16(dv))
        return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, total_len);
    p.q = q;
    p.k = k;
    p.v = v;
    p.offsets = offsets;
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0) return VISTA_OK;
    const BwdPlan b = plan_bwd(p);
    if (!workspace || workspace_bytes < b.total) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    char* ws = reinterpret_cast<char*>(workspace);
    const float* z = z_saved ? z_saved : reinterpret_cast<float*>(ws + b.z_off);
    float* dz = reinterpret_cast<float*>(ws + b.dz_off);
    const bool tc = qla_bwd_uses_tc(p);
    uint8_t* dz_op = tc ? reinterpret_cast<uint8_t*>(ws + b.dzop_off) : nullptr;
    float* dqu = p.q_user_stride == 0 ? reinterpret_cast<float*>(ws + b.dqu_off) : dq;
    // 1. Z = sum_j phi1(k_j)^T v_j (the forward state kernel, partial mode), unless the forward's
    //    state was saved.  The timing hook, if armed, is kept for the dK / dV kernel (the dominant
    //    one of the backward).  The tile starts of the dK / dV kernel come from this run too.
    cudaEvent_t ev_a = g_ev_start, ev_b = g_ev_stop;
    g_ev_start = g_ev_stop = nullptr;
    if (!z_saved) {
        st = run(desc, q, k, v, offsets, total_len, OutSpec{OUT_PARTIAL, 0, const_cast<float*>(z), nullptr},
                 ws + b.sub_off, b.z_off - b.sub_off, stream);
    } else if (qla_bwd_uses_tc(p) && total_len > 0) {
        const Workspace w = plan_workspace(p, true);
        Problem pt = p;
        pt.outs = OutSpec{OUT_PARTIAL, 0, nullptr, nullptr};
        const cudaError_t e0 = launch_user_tiles(pt, reinterpret_cast<int64_t*>(ws + b.sub_off + w.uts_off), nullptr);
        if (e0 != cudaSuccess) st = cuda_fail(e0);
        else g_launches += 1;
    }
    g_ev_start = ev_a;
    g_ev_stop = ev_b;
    if (st != VISTA_OK) return st;
    // 2. per unit: dW, dZ, dA -> dQ_u (tensor cores when bf16, d = 128, S % 128 == 0)
    cudaError_t e;
    int nl = 1;
    if (tc && p.S % 128 == 0) {
        uint8_t* abuf = reinterpret_cast<uint8_t*>(ws + b.abuf_off);
        e = launch_qla_prep_q(p, abuf);
        if (e == cudaSuccess)
            e = launch_sm100_qla_bwd_unit(p, desc->out_dtype == VISTA_BF16, dout, z, abuf, dz_op, dqu);
        ++nl;
    } else {
        e = launch_qla_bwd_unit(p, desc->out_dtype == VISTA_BF16, dout, z, dz, dz_op, dqu);
    }
    // 3. shared seeds: dQ = sum_u dQ_u
    if (e == cudaSuccess && p.q_user_stride == 0) {
        e = launch_qla_bwd_dq_sum(p, dqu, dq);
        ++nl;
    }
    // 4. dK, dV
    if (e == cudaSuccess && total_len > 0) {
        if (tc) {
            const Workspace w = plan_workspace(p, true);
            e = timed_main(p.stream, [&] { return launch_sm100_qla_bwd_kv(p, w, ws + b.sub_off, dz_op, dk, dv); });
        } else {
            e = timed_main(p.stream, [&] { return launch_qla_bwd_kv_simt(p, dz, dk, dv); });
        }
        ++nl;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += (unsigned long long)nl;
    return VISTA_OK;
}

// ---------------------------------------------------------------- QLA at per-user query rows
namespace {
struct RowsPlan {
    size_t sub_off, z_off, w_off, uts_off, total;
};
// with_state: workspace for the Z pass too (vista_qla_rows); else only W_u and the rows' tile starts
RowsPlan plan_rows(const Problem& p, int64_t total_rows, bool with_state) {
    RowsPlan r{};
    const size_t B = (size_t)p.B, H = (size_t)p.H, d = (size_t)p.d;
    const bool tc = qla_rows_uses_tc(p, total_rows);
    size_t off = 0;
    r.sub_off = off;
    if (with_state) off = align256(off + plan_workspace(p, true).total);
    r.z_off = off;
    if (with_state) off = align256(off + B * H * d * d * sizeof(float));
    r.w_off = off;
    if (tc) off = align256(off + B * H * d * d * 2);
    r.uts_off = off;
    if (tc) off = align256(off + (B + 1) * sizeof(int64_t));
    r.total = off;
    return r;
}

// Rows from a state: W_u = phi2(Z_u / N_u) operands, the rows' tile starts, the rows kernel (or the
// SIMT kernel).  N_u from user_len (if given) or p.offsets.
vista_status_t rows_from_z(const vista_desc_t* desc, const Problem& p, const RowsPlan& r, char* ws, const float* z,
                           const int64_t* user_len, const void* q_rows, const int64_t* row_offsets, int64_t total_rows,
                           const void* k_self, const void* v_self, void* out, const void* gate = nullptr) {
    const int out_bf16 = desc->out_dtype == VISTA_BF16;
    cudaError_t e;
    int nl = 0;
    if (qla_rows_uses_tc(p, total_rows)) {
        uint8_t* w_op = reinterpret_cast<uint8_t*>(ws + r.w_off);
        int64_t* uts = reinterpret_cast<int64_t*>(ws + r.uts_off);
        Problem pr = p;
        pr.offsets = row_offsets;
        pr.total_len = total_rows;
        pr.attn = VISTA_QLA;
        pr.outs = OutSpec{OUT_PARTIAL, 0, nullptr, nullptr};
        e = launch_qla_prep_w(p, z, w_op, user_len);
        if (e == cudaSuccess) e = launch_user_tiles(pr, uts, nullptr);
        if (e == cudaSuccess)
            e = timed_main(p.stream, [&] {
                return launch_sm100_qla_rows(p, row_offsets, total_rows, uts, w_op, q_rows, k_self, v_self, out_bf16,
                                             out, user_len, gate);
            });
        nl = 3;
    } else {
        e = timed_main(p.stream, [&] {
            return launch_qla_rows_simt(p, z, row_offsets, total_rows, q_rows, k_self, v_self, out_bf16, out, user_len);
        });
        nl = 1;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += (unsigned long long)nl;
    return VISTA_OK;
}

vista_status_t check_rows_args(const vista_desc_t* desc, int64_t total_rows, const void* q_rows,
                               const int64_t* row_offsets, const void* k_self, const void* v_self, const void* out) {
    if (desc->attn != VISTA_QLA || total_rows < 0) return VISTA_ERR_INVALID;
    if (!row_offsets) return VISTA_ERR_NULL;
    if (total_rows > 0 && (!q_rows || !out)) return VISTA_ERR_NULL;
    if ((k_self == nullptr) != (v_self == nullptr)) return VISTA_ERR_NULL;
    if (!aligned16(q_rows) || !aligned16(k_self) || !aligned16(v_self) || !aligned16(out)) return VISTA_ERR_MISALIGNED;
    return VISTA_OK;
}
}  // namespace

vista_status_t vista_qla_rows_workspace_size(const vista_desc_t* desc, int64_t total_len, int64_t total_rows,
                                             size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (desc->attn != VISTA_QLA || total_len < 0 || total_rows < 0) return VISTA_ERR_INVALID;
    *bytes = plan_rows(make_problem(desc, total_len), total_rows, true).total;
    return VISTA_OK;
}

vista_status_t vista_qla_rows(const vista_desc_t* desc, const void* k, const void* v, const int64_t* offsets,
                              int64_t total_len, const void* q_rows, const int64_t* row_offsets, int64_t total_rows,
                              const void* k_self, const void* v_self, void* out, void* workspace,
                              size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (total_len < 0) return VISTA_ERR_INVALID;
    if ((st = check_rows_args(desc, total_rows, q_rows, row_offsets, k_self, v_self, out)) != VISTA_OK) return st;
    if (!offsets) return VISTA_ERR_NULL;
    if (total_len > 0 && (!k || !v)) return VISTA_ERR_NULL;
    if (!aligned16(k) || !aligned16(v)) return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, total_len);
    p.k = k;
    p.v = v;
    p.offsets = offsets;
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0 || total_rows == 0) return VISTA_OK;
    const RowsPlan r = plan_rows(p, total_rows, true);
    if (!workspace || workspace_bytes < r.total) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    char* ws = reinterpret_cast<char*>(workspace);
    float* z = reinterpret_cast<float*>(ws + r.z_off);
    // 1. Z_u = sum_j phi1(k_j)^T v_j (the forward state path, partial mode); the timing hook, if
    //    armed, is kept for the rows kernel
    cudaEvent_t ev_a = g_ev_start, ev_b = g_ev_stop;
    g_ev_start = g_ev_stop = nullptr;
    st = run(desc, q_rows, k, v, offsets, total_len, OutSpec{OUT_PARTIAL, 0, z, nullptr}, ws + r.sub_off,
             r.z_off - r.sub_off, stream);
    g_ev_start = ev_a;
    g_ev_stop = ev_b;
    if (st != VISTA_OK) return st;
    // 2.-3. W_u, tile starts, rows
    return rows_from_z(desc, p, r, ws, z, nullptr, q_rows, row_offsets, total_rows, k_self, v_self, out);
}

vista_status_t vista_qla_rows_from_state_workspace_size(const vista_desc_t* desc, int64_t total_rows, size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (desc->attn != VISTA_QLA || total_rows < 0) return VISTA_ERR_INVALID;
    *bytes = plan_rows(make_problem(desc, 0), total_rows, false).total;
    return VISTA_OK;
}

vista_status_t vista_qla_rows_from_state(const vista_desc_t* desc, const float* z, const int64_t* user_len,
                                         const void* q_rows, const int64_t* row_offsets, int64_t total_rows,
                                         const void* k_self, const void* v_self, void* out, void* workspace,
                                         size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if ((st = check_rows_args(desc, total_rows, q_rows, row_offsets, k_self, v_self, out)) != VISTA_OK) return st;
    if (desc->num_users > 0 && (!z || !user_len)) return VISTA_ERR_NULL;
    if (!aligned16(z)) return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, 0);
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0 || total_rows == 0) return VISTA_OK;
    const RowsPlan r = plan_rows(p, total_rows, false);
    if (r.total > 0 && (!workspace || workspace_bytes < r.total)) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    return rows_from_z(desc, p, r, reinterpret_cast<char*>(workspace), z, user_len, q_rows, row_offsets, total_rows,
                       k_self, v_self, out);
}

// ---------------------------------------------------------------- multi-layer summarizer (NEXT-3)
namespace {
struct LayersPlan {
    size_t qkvg_off, o_off, z_off, sub_off, rows_off, total;
};
LayersPlan plan_layers(const Problem& p, int64_t R) {
    LayersPlan l{};
    const size_t D = (size_t)p.H * p.d;
    size_t off = 0;
    l.qkvg_off = off;
    off = align256(off + 4 * (size_t)R * D * 2);
    l.o_off = off;
    off = align256(off + (size_t)R * D * 2);
    l.z_off = off;
    off = align256(off + (size_t)p.B * p.H * p.d * p.d * sizeof(float));
    l.sub_off = off;
    Problem ps = p;
    ps.total_len = R;
    ps.attn = VISTA_QLA;
    off = align256(off + plan_workspace(ps, true).total);
    l.rows_off = off;
    off = align256(off + plan_rows(ps, R, false).total);
    l.total = off;
    return l;
}
bool layers_supported(const vista_desc_t* d) {
    return d->in_dtype == VISTA_BF16 && d->head_dim == 128 && d->attn == VISTA_QLA && d->q_user_stride == 0;
}
}  // namespace

vista_status_t vista_summarize_layers_workspace_size(const vista_desc_t* desc, int32_t num_layers, int64_t total_rows,
                                                     size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (num_layers < 0 || total_rows < 0) return VISTA_ERR_INVALID;
    if (!layers_supported(desc)) return VISTA_ERR_UNSUPPORTED;
    *bytes = plan_layers(make_problem(desc, total_rows), total_rows).total;
    return VISTA_OK;
}

vista_status_t vista_summarize_layers(const vista_desc_t* desc, int32_t num_layers, const void* weights, void* x,
                                      const int64_t* x_offsets, int64_t total_rows, void* tokens, void* workspace,
                                      size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (num_layers < 0 || total_rows < 0) return VISTA_ERR_INVALID;
    if (!layers_supported(desc)) return VISTA_ERR_UNSUPPORTED;
    if (!x_offsets || (total_rows > 0 && !x) || (num_layers > 0 && !weights)) return VISTA_ERR_NULL;
    if (!aligned16(weights) || !aligned16(x) || !aligned16(tokens)) return VISTA_ERR_MISALIGNED;
    if (total_rows >= (int64_t(1) << 31)) return VISTA_ERR_UNSUPPORTED;
    Problem p = make_problem(desc, total_rows);
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0) return VISTA_OK;
    const LayersPlan l = plan_layers(p, total_rows);
    if (!workspace || workspace_bytes < l.total) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    char* ws = reinterpret_cast<char*>(workspace);
    const int R = (int)total_rows, D = p.H * p.d;
    const size_t RD = (size_t)R * D;
    __nv_bfloat16* qkvg = reinterpret_cast<__nv_bfloat16*>(ws + l.qkvg_off);
    void* outs[4] = {qkvg, qkvg + RD, qkvg + 2 * RD, qkvg + 3 * RD};  // Q, K, V, G [R, D] each
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(ws + l.o_off);
    float* z = reinterpret_cast<float*>(ws + l.z_off);
    vista_desc_t dq = *desc;  // the QLA state / rows over all rows of every user's segment
    dq.attn = VISTA_QLA;
    dq.in_dtype = VISTA_BF16;
    dq.out_dtype = VISTA_BF16;
    Problem pr = make_problem(&dq, total_rows);
    pr.offsets = x_offsets;
    pr.stream = p.stream;
    const RowsPlan rp = plan_rows(pr, total_rows, false);
    cudaError_t e = cudaSuccess;
    for (int layer = 0; layer < num_layers && R > 0; ++layer) {
        const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(weights) + (size_t)layer * 5 * D * D;
        // 1. [Q | K | V | G] = X [Wq | Wk | Wv | Wg]^T
        // (the timing hook, if armed, brackets the first layer's projection GEMM, the dominant kernel)
        if ((e = timed_main(p.stream, [&] {
                 return launch_sm100_gemm(R, 4 * D, D, x, D, W, 4, outs, nullptr, p.num_sms, p.stream);
             })) != cudaSuccess)
            break;
        g_launches += 1;
        // 2. Z_u = sum over the user's rows of phi1(K)^T V (the state kernel, partial mode)
        cudaEvent_t ev_a = g_ev_start, ev_b = g_ev_stop;
        g_ev_start = g_ev_stop = nullptr;
        st = run(&dq, outs[0], outs[1], outs[2], x_offsets, total_rows, OutSpec{OUT_PARTIAL, 0, z, nullptr},
                 ws + l.sub_off, l.rows_off - l.sub_off, stream);
        g_ev_start = ev_a;
        g_ev_stop = ev_b;
        if (st != VISTA_OK) return st;
        // 3. O_r = (phi1(Q_r) phi2(Z_u / N_u)) (.) sigmoid(G_r) for every row (N_u = the segment's length;
        //    the SGLU gate applied in the rows kernel's epilogue, so O is written once, gated)
        st = rows_from_z(&dq, pr, rp, ws + l.rows_off, z, nullptr, outs[0], x_offsets, total_rows, nullptr, nullptr, o,
                         outs[3]);
        if (st != VISTA_OK) return st;
        // 4. X <- X + O Wo^T (the residual in the GEMM's epilogue)
        void* xo[4] = {x, x, x, x};
        if ((e = launch_sm100_gemm(R, D, D, o, D, W + 4 * (size_t)D * D, 1, xo, x, p.num_sms, p.stream)) != cudaSuccess)
            break;
        g_launches += 1;
    }
    if (e == cudaSuccess && tokens) {
        e = launch_gather_seed_rows(x, x_offsets, p.B, p.S, D, desc->out_dtype == VISTA_BF16, tokens, p.stream);
        g_launches += 1;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    return VISTA_OK;
}

// ---------------------------------------------------------------- stage-2 target-aware attention
vista_status_t vista_target_attend_workspace_size(const vista_desc_t* desc, int64_t total_rows, size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    if (total_rows < 0) return VISTA_ERR_INVALID;
    const Problem p = make_problem(desc, 0);
    *bytes = target_attend_uses_tc(p) ? align256((size_t)(p.B + 1) * sizeof(int64_t)) : 0;
    return VISTA_OK;
}

vista_status_t vista_target_attend(const vista_desc_t* desc, const int8_t* codes, const float* token_scale,
                                   const float* token_zero_point, const void* q, const void* k_self,
                                   const void* v_self, const void* resid, const int64_t* row_offsets,
                                   int64_t total_rows, void* out, float* lse, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (total_rows < 0) return VISTA_ERR_INVALID;
    if (!row_offsets) return VISTA_ERR_NULL;
    if (desc->num_users > 0 && (!codes || !token_scale || !token_zero_point)) return VISTA_ERR_NULL;
    if (total_rows > 0 && (!q || !k_self || !v_self || !out)) return VISTA_ERR_NULL;
    if (!aligned16(codes) || !aligned16(q) || !aligned16(k_self) || !aligned16(v_self) || !aligned16(resid) ||
        !aligned16(out) || (reinterpret_cast<uintptr_t>(token_scale) & 3) ||
        (reinterpret_cast<uintptr_t>(token_zero_point) & 3) || (reinterpret_cast<uintptr_t>(lse) & 3))
        return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, 0);
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0 || total_rows == 0) return VISTA_OK;
    const int out_bf16 = desc->out_dtype == VISTA_BF16;
    cudaError_t e;
    int nl;
    if (target_attend_uses_tc(p) && total_rows < (int64_t(1) << 31)) {
        const size_t need = align256((size_t)(p.B + 1) * sizeof(int64_t));
        if (!workspace || workspace_bytes < need) return VISTA_ERR_WORKSPACE;
        if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
        int64_t* uts = reinterpret_cast<int64_t*>(workspace);
        Problem pr = p;  // tile starts of the candidates' jagged layout
        pr.offsets = row_offsets;
        pr.total_len = total_rows;
        pr.attn = VISTA_QLA;
        pr.outs = OutSpec{OUT_PARTIAL, 0, nullptr, nullptr};
        e = launch_user_tiles(pr, uts, nullptr);
        if (e == cudaSuccess)
            e = timed_main(p.stream, [&] {
                return launch_sm100_target_attend(p, row_offsets, total_rows, uts, codes, token_scale, token_zero_point,
                                                  q, k_self, v_self, resid, out_bf16, out, lse);
            });
        nl = 2;
    } else {
        e = timed_main(p.stream, [&] {
            return launch_simt_target_attend(p, row_offsets, total_rows, codes, token_scale, token_zero_point, q,
                                             k_self, v_self, resid, out_bf16, out, lse);
        });
        nl = 1;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += (unsigned long long)nl;
    return VISTA_OK;
}

static size_t merge_ws_bytes(const Problem& p) {
    return (p.attn == VISTA_QLA && qla_finalize_uses_tc(p)) ? sm100_qla_finalize_workspace(p) : 0;
}

vista_status_t vista_summarize_merge_workspace_size(const vista_desc_t* desc, size_t* bytes) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (!bytes) return VISTA_ERR_NULL;
    *bytes = merge_ws_bytes(make_problem(desc, 0));
    return VISTA_OK;
}

vista_status_t vista_summarize_merge(const vista_desc_t* desc, int32_t num_parts, const float* part_o,
                                     const float* part_lse, const void* q, const int64_t* user_len, void* out,
                                     float* lse, void* workspace, size_t workspace_bytes, void* stream) {
    vista_status_t st = validate_desc(desc);
    if (st != VISTA_OK) return st;
    if (num_parts < 1) return VISTA_ERR_INVALID;
    if (!part_o || !out) return VISTA_ERR_NULL;
    if (desc->attn == VISTA_SOFTMAX && !part_lse) return VISTA_ERR_NULL;
    if (desc->attn == VISTA_QLA && (!q || !user_len)) return VISTA_ERR_NULL;
    if (!aligned16(part_o) || !aligned16(out) || (q && !aligned16(q))) return VISTA_ERR_MISALIGNED;
    Problem p = make_problem(desc, 0);
    p.q = q;
    p.outs = OutSpec{OUT_FINAL, desc->out_dtype == VISTA_BF16, out, desc->attn == VISTA_SOFTMAX ? lse : nullptr};
    p.stream = reinterpret_cast<cudaStream_t>(stream);
    if (p.B == 0) return VISTA_OK;
    const size_t need = merge_ws_bytes(p);
    if (need > 0 && (!workspace || workspace_bytes < need)) return VISTA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return VISTA_ERR_MISALIGNED;
    cudaError_t e;
    if (desc->attn == VISTA_SOFTMAX) {
        e = launch_merge_softmax_parts(p, num_parts, part_o, part_lse);
    } else {
        e = launch_qla_finalize(p, part_o, num_parts, (int64_t)p.B * p.H * p.d * p.d, user_len, workspace);
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches += 1;
    return VISTA_OK;
}

vista_status_t vista_quantize_rows_int8(int64_t n, int32_t d, int32_t in_dtype, const void* x, int8_t* codes,
                                        float* scale, float* zero_point, void* stream) {
    if (n < 0 || d < 1) return VISTA_ERR_INVALID;
    if (in_dtype != VISTA_F32 && in_dtype != VISTA_BF16) return VISTA_ERR_INVALID;
    if (n > 0 && (!x || !codes || !scale || !zero_point)) return VISTA_ERR_NULL;
    cudaError_t e = launch_quantize_rows(n, d, in_dtype == VISTA_BF16, x, codes, scale, zero_point,
                                         reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    if (n > 0) g_launches += 1;
    return VISTA_OK;
}

vista_status_t vista_time_next_main_kernel(void* start_event, void* stop_event) {
    g_ev_start = reinterpret_cast<cudaEvent_t>(start_event);
    g_ev_stop = reinterpret_cast<cudaEvent_t>(stop_event);
    return VISTA_OK;
}

uint64_t vista_launch_counter(void) { return g_launches.load(); }

vista_status_t vista_check_offsets(const int64_t* offsets, int32_t num_users, int64_t total_len, void* stream) {
    if (!offsets) return VISTA_ERR_NULL;
    if (num_users < 0) return VISTA_ERR_INVALID;
    std::vector<int64_t> h((size_t)num_users + 1);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(h.data(), offsets, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (h[0] != 0 || h[num_users] != total_len) return VISTA_ERR_OFFSETS;
    for (int32_t u = 0; u < num_users; ++u)
        if (h[u + 1] < h[u]) return VISTA_ERR_OFFSETS;
    return VISTA_OK;
}

}  // extern "C"
