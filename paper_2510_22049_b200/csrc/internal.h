// internal.h -- host/device declarations shared by the libvista kernels and the C ABI layer.
// Not part of the public ABI (include/vista.h is).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#include "../../include/vista.h"

namespace vista {

constexpr int kTile = 128;  // history items per tile (= TMA box rows = MMA N of the score GEMM)
// Upper bound on every persistent grid (one CTA per SM): the split-L merge lists a unit's run of
// partial slots in a fixed array of 2 * kMaxPersistentCtas + 2 entries (kernels_misc.cu).
constexpr int kMaxPersistentCtas = 159;
constexpr int kMaxExchangeRanks = 8;  // p2p_exchange.cu: ranks of one node
void count_launches(unsigned n);     // the library's launch counter (vista_launch_counter)
// p2p_exchange.cu: spin until every rank acknowledged the current epoch (the fused exchange's first step)
cudaError_t launch_exchange_wait_acks(int world, const uint32_t* acks, const uint32_t* epoch, cudaStream_t stream);

enum OutMode : int { OUT_FINAL = 0, OUT_PARTIAL = 1 };

// Launch with programmatic dependent launch (PDL): the kernel may begin while its predecessor on
// the stream finishes; it must execute `griddepcontrol.wait` before touching the predecessor's
// results.  Hides the launch latency of the short kernels around the main ones.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifdef VISTA_NO_PDL
    cfg.numAttrs = 0;
#else
    cfg.numAttrs = 1;
#endif
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the CURRENT device, set once per
// (function, device, bytes) under a lock (function attributes are per device: a process-wide
// once-only set would leave a second device at the 48 KB default).  vista_abi.cu.
cudaError_t set_smem_attr(const void* fn, int bytes);

// Where a finished (normalized) output row goes.
struct OutSpec {
    int mode;            // OUT_FINAL: out[B,S,H,d] (out_dtype) + lse[B,H,S]; OUT_PARTIAL: part_o[B,H,S,d] f32 + part_lse[B,H,S]
    int out_bf16;        // OUT_FINAL only: 1 -> bf16, 0 -> f32
    void* out;           // FINAL: out;  PARTIAL: part_o (float*)
    float* lse;          // may be NULL in FINAL mode
    // NEXT-1 fused int8 export of the out rows (FINAL mode; NULL = none): codes [B,S,H,d] int8,
    // qscale / qzp [B,S,H] float32 (int8_export.cuh)
    int8_t* codes;
    float* qscale;
    float* qzp;
};

// The fused split-L exchange (vista_summarize_partial_peers): n > 0 -> every partial-mode row and lse
// (softmax) is stored to these n destinations instead of OutSpec out / lse -- the node's receive
// buffers, already offset to this rank's slot.  A separate kernel argument (not in OutSpec), so the
// kernels that never see it compile exactly as before.
struct PeerSpec {
    int n;
    float* o[kMaxExchangeRanks];
    float* lse[kMaxExchangeRanks];
};

// Everything a launch needs (filled by the ABI layer after validation).
struct Problem {
    int B, S, H, d;
    int in_bf16;               // 1: q/k/v bf16, 0: f32
    int attn;                  // vista_attn_t
    float scale;               // softmax scale (> 0)
    int phi1, phi2, normalize; // QLA
    int64_t q_user_stride;     // elements; 0 = shared
    int64_t total_len;
    const void* q;
    const void* k;
    const void* v;
    const int64_t* offsets;
    OutSpec outs;
    PeerSpec peers;            // fused exchange destinations (softmax partial); n = 0: none
    cudaStream_t stream;
    int num_sms;
};



// Workspace carve-up (all offsets 256-B aligned).
struct Workspace {
    size_t uts_off, slot_unit_off, slot_o_off, slot_lse_off, zbuf_off, fin_off, total;
    int num_ctas;      // persistent grid size used by the tiled kernels
    int rows_per_unit; // softmax: query rows per work unit (NQ * 128); QLA: d
};

enum Path : int { PATH_NONE = 0, PATH_SM100_SOFTMAX, PATH_SM100_QLA, PATH_SIMT_SOFTMAX, PATH_SIMT_QLA };

Path choose_path(const Problem& p);
Workspace plan_workspace(const Problem& p, bool partial);

// ---- launchers (return cudaError_t of the launch) ----
// user tile starts: uts[u] = sum_{u'<u} ceil(L_u' / 128); also fills the outputs of empty users
// (softmax: zeros / -inf in outs; QLA: zeros in zbuf if non-NULL).
cudaError_t launch_user_tiles(const Problem& p, int64_t* uts, float* zbuf);
cudaError_t launch_sm100_softmax(const Problem& p, const Workspace& w, char* ws);
// wbuf != NULL: complete units write W = phi2(Z / N) (bf16 finalize operand) instead of Z to zbuf
cudaError_t launch_sm100_qla_state(const Problem& p, const Workspace& w, char* ws, float* zbuf,
                                   uint8_t* wbuf = nullptr);
cudaError_t launch_merge_softmax_slots(const Problem& p, const Workspace& w, char* ws);
cudaError_t launch_merge_qla_slots(const Problem& p, const Workspace& w, char* ws, float* zbuf);
// split units' W = phi2(sum of slots / N) into wbuf (fused finalize path)
cudaError_t launch_merge_qla_slots_w(const Problem& p, const Workspace& w, char* ws, uint8_t* wbuf);
// finalize from the W operands already at ws (sm100_qla_finalize_workspace layout: W then phi1(Q))
cudaError_t launch_sm100_qla_finalize_fused(const Problem& p, uint8_t* ws);
cudaError_t launch_simt_softmax(const Problem& p);
cudaError_t launch_simt_qla_state(const Problem& p, float* zbuf);
// O = phi1(Q) phi2( (sum_{p<P} Z_p) / N_u ) ; Z parts at zparts + p * part_stride (floats),
// N_u from offsets (user_len == NULL) or user_len[u].
cudaError_t launch_qla_finalize(const Problem& p, const float* zparts, int P, int64_t part_stride,
                                const int64_t* user_len, void* ws);
bool qla_finalize_uses_tc(const Problem& p);
// QLA backward (NEXT-2)
cudaError_t launch_qla_bwd_unit(const Problem& p, bool dout_bf16, const void* dout, const float* z, float* dz,
                                uint8_t* dz_op, float* dqu);
cudaError_t launch_qla_bwd_dq_sum(const Problem& p, const float* dqu, float* dq);
cudaError_t launch_qla_bwd_kv_simt(const Problem& p, const float* dz, void* dk, void* dv);
// tcgen05 dK / dV (bf16, d = 128): uts from the forward recompute's workspace; dz_op bf16 operands
cudaError_t launch_sm100_qla_bwd_kv(const Problem& p, const Workspace& w, char* ws, const uint8_t* dz_op, void* dk,
                                    void* dv);
bool qla_bwd_uses_tc(const Problem& p);
// softmax backward (NEXT-2): bf16, d = 128, S % 128 == 0, S <= 1024, bf16 dout
bool softmax_bwd_supported(const Problem& p, bool dout_bf16);
size_t softmax_bwd_workspace(const Problem& p);
// CUDA-core softmax backward for the other shapes (softmax_bwd_simt.cu)
size_t softmax_bwd_simt_workspace(const Problem& p);
cudaError_t launch_softmax_bwd_simt(const Problem& p, bool dout_bf16, const void* out, const float* lse,
                                    const void* dout, float* dq, void* dk, void* dv, char* ws);
cudaError_t launch_softmax_bwd(const Problem& p, const void* out, const float* lse, const void* dout, float* dq,
                               void* dk, void* dv, char* ws, int* nlaunch, cudaEvent_t ev_a, cudaEvent_t ev_b);
// phi1(Q) as bf16 128-row MMA operand blocks (qla_prep_q_kernel); qla_prep_q_bytes of space
size_t qla_prep_q_bytes(const Problem& p);
cudaError_t launch_qla_prep_q(const Problem& p, uint8_t* abuf);
// tcgen05 per-unit backward (dW -> dZ operand, dA -> per-user dQ); needs S % 128 == 0
cudaError_t launch_sm100_qla_bwd_unit(const Problem& p, bool dout_bf16, const void* dout, const float* z,
                                      const uint8_t* abuf, uint8_t* dz_op, float* dqu);
// shared key prefix (vista_summarize_*_prefix)
cudaError_t launch_write_prefix_offsets(int64_t* off, int64_t P, cudaStream_t st);
cudaError_t launch_merge_prefix(const Problem& p, const float* o, const float* lse, const float* opre,
                                const float* lpre);
cudaError_t launch_add_prefix_state(const Problem& p, float* z, const float* zpre, int64_t P, int64_t* user_len);
// tensor-core finalize (bf16, d = 128); ws: sm100_qla_finalize_workspace(p) bytes
size_t sm100_qla_finalize_workspace(const Problem& p);
// QLA at per-user query rows (NEXT-3 / NEXT-4, sm100_qla_rows.cu)
// W_u = phi2(Z_u / N_u) operands; N_u = user_len[u] if given, else from p.offsets
cudaError_t launch_qla_prep_w(const Problem& p, const float* z, uint8_t* wbuf, const int64_t* user_len = nullptr);
bool qla_rows_uses_tc(const Problem& p, int64_t total_rows);
cudaError_t launch_sm100_qla_rows(const Problem& p, const int64_t* row_offsets, int64_t total_rows, const int64_t* uts,
                                  const uint8_t* w_op, const void* q, const void* k_self, const void* v_self,
                                  int out_bf16, void* out, const int64_t* user_len = nullptr,
                                  const void* gate = nullptr);
cudaError_t launch_qla_rows_simt(const Problem& p, const float* z, const int64_t* row_offsets, int64_t total_rows,
                                 const void* q, const void* k_self, const void* v_self, int out_bf16, void* out,
                                 const int64_t* user_len = nullptr);
// multi-layer summarizer (NEXT-3): tcgen05 GEMM C = A B^T (sm100_gemm.cu) and the seed-row gather
cudaError_t launch_sm100_gemm(int M, int N, int K, const void* A, int64_t lda, const void* Bw, int nsplit,
                              void* const* outs, const void* resid, int num_sms, cudaStream_t stream);
cudaError_t launch_gather_seed_rows(const void* x, const int64_t* x_offsets, int B, int S, int D, int out_bf16,
                                    void* tokens, cudaStream_t stream);
// stage-2 target-aware attention over the cached int8 summary tokens (NEXT-4, sm100_target_attend.cu)
bool target_attend_uses_tc(const Problem& p);
cudaError_t launch_sm100_target_attend(const Problem& p, const int64_t* row_offsets, int64_t total_rows,
                                       const int64_t* uts, const int8_t* codes, const float* tscale, const float* tzp,
                                       const void* q, const void* k_self, const void* v_self, const void* resid,
                                       int out_bf16, void* out, float* lse);
cudaError_t launch_simt_target_attend(const Problem& p, const int64_t* row_offsets, int64_t total_rows,
                                      const int8_t* codes, const float* tscale, const float* tzp, const void* q,
                                      const void* k_self, const void* v_self, const void* resid, int out_bf16,
                                      void* out, float* lse);
cudaError_t launch_sm100_qla_finalize(const Problem& p, const float* zparts, int P, int64_t part_stride,
                                      const int64_t* user_len, void* ws);
cudaError_t launch_quantize_rows(int64_t n, int d, int in_bf16, const void* x, int8_t* codes, float* scale, float* zp,
                                 cudaStream_t stream);
// Merge P stacked softmax partials [P,B,H,S,d] / [P,B,H,S] into outs.
cudaError_t launch_merge_softmax_parts(const Problem& p, int P, const float* part_o, const float* part_lse);

}  // namespace vista
