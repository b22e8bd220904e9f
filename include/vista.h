/*
 * vista.h -- C ABI of libvista: B200 (sm_100a) kernels for VISTA stage-1 user-history
 * summarization (arXiv 2510.22049, "VISTA").  Citations are PAPER.md:<line> of the paper source.
 *
 * WHAT IS COMPUTED.  S learned "virtual seed" query tokens, shared across users (PAPER.md:148,
 * Sec. 3.2 "initialized randomly as shared parameters across users"), attend over each user's
 * interaction history (UIH) of L_u item embeddings; the seed rows' outputs are the user's summary
 * tokens.  Two accumulator forms:
 *
 *   VISTA_SOFTMAX  RowSoftmax(Q K^T) V  (Sec. 3.2.1), queries = the S seed rows:
 *                  out[u,i,h,:] = sum_j softmax_j(scale * q_{i,h} . k_{j,h}) v_{j,h,:}
 *                  lse[u,h,i]   = ln sum_j exp(scale * q_{i,h} . k_{j,h})        (natural log)
 *   VISTA_QLA      quasi-linear attention, source part (Sec. 3.2.2; two
 *                  activations PAPER.md:831-836, App. B.2):
 *                  Z = sum_j phi1(k_j)^T v_j (d x d);  Zbar = Z / N_u if qla_normalize
 *                  (the "1/N factor"; N_u = L_u);  out = phi1(Q) phi2(Zbar)
 *
 * No mask and no positional term (full attention).  Users are independent.
 * Empty history (L_u = 0): softmax out = 0 and lse = -inf (the identity of the LSE merge);
 * QLA Zbar = 0 so out = phi1(Q) phi2(0).
 *
 * LAYOUTS (row-major, last dimension contiguous, element strides in parentheses):
 *   q       [S, H, d]     shared seeds (q_user_stride = 0), or user u's block at q + u*q_user_stride
 *   k, v    [total_len, H, d]   jagged history of all users, user u owns rows
 *                               [offsets[u], offsets[u+1])
 *   offsets [B + 1] int64, DEVICE memory; offsets[0] = 0, non-decreasing, offsets[B] = total_len
 *   out     [B, S, H, d]  (out_dtype)
 *   lse     [B, H, S]     float32, may be NULL
 *   part_o  softmax: [B, H, S, d] float32 normalized partial output;
 *           QLA:     [B, H, d, d] float32 unnormalized partial state Z_p
 *   part_lse softmax: [B, H, S] float32 (-inf for an empty shard); QLA: unused (may be NULL)
 *
 * OWNERSHIP AND SYNCHRONIZATION.  All tensor pointers are DEVICE pointers owned by the caller,
 * who also owns the workspace.  The library never allocates or frees device memory on these
 * calls and never synchronizes: every call only enqueues kernels on `stream` (a cudaStream_t,
 * NULL = legacy default stream).  Results are bitwise deterministic for fixed inputs, device and
 * partition.  Calls are reentrant; concurrent calls on different streams need different
 * workspaces.
 *
 * ERRORS.  Return codes only (no exceptions cross the ABI).  Every host-checkable error is
 * reported BEFORE any launch, with no side effect: NULL pointers, B < 0, S < 1, H < 1, an
 * unsupported (dtype, d, attn) combination, misalignment (16 B base for q/k/v/out; TMA needs
 * 16 B strides), too small a workspace.  Offsets are a precondition (not read on the host);
 * vista_check_offsets() validates them (synchronizing, debug only).  Launch failures return
 * VISTA_ERR_CUDA.
 *
 * DISPATCH (by shape, not a backend switch):
 *   bf16, d = 128, softmax, S % 128 == 0  -> TMA + tcgen05/TMEM kernel (sm_100a)
 *   bf16, d = 128, QLA                    -> TMA + tcgen05/TMEM state kernel + finalize
 *   f32 or bf16 with d in {32, 64, 128} otherwise -> SIMT fp32-accumulate kernels
 */
#ifndef VISTA_H_
#define VISTA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VISTA_ABI_VERSION 1

typedef enum {
    VISTA_OK = 0,
    VISTA_ERR_NULL = 1,        /* a required pointer is NULL                          */
    VISTA_ERR_INVALID = 2,     /* bad size / enum / abi_version                       */
    VISTA_ERR_UNSUPPORTED = 3, /* valid but unsupported (dtype, d, attn, S) combination */
    VISTA_ERR_MISALIGNED = 4,  /* a pointer is not 16-byte aligned                    */
    VISTA_ERR_WORKSPACE = 5,   /* workspace_bytes < vista_summarize_workspace_size     */
    VISTA_ERR_CUDA = 6,        /* a CUDA runtime / driver call failed                 */
    VISTA_ERR_OFFSETS = 7      /* vista_check_offsets: offsets violate the precondition */
} vista_status_t;

typedef enum { VISTA_F32 = 0, VISTA_BF16 = 1 } vista_dtype_t;
typedef enum { VISTA_SOFTMAX = 0, VISTA_QLA = 1 } vista_attn_t;
/* phi choices: identity; SiLU x*sigmoid(x); shifted ELU x if x >= 1 else e^{x-1}
 * (App. B.1.5). */
typedef enum { VISTA_ACT_IDENTITY = 0, VISTA_ACT_SILU = 1, VISTA_ACT_SHIFTED_ELU = 2 } vista_act_t;

typedef struct {
    int32_t abi_version;   /* must equal VISTA_ABI_VERSION                                  */
    int32_t num_users;     /* B >= 0                                                        */
    int32_t num_summary;   /* S >= 1  (summary tokens = seed queries)                       */
    int32_t num_heads;     /* H >= 1                                                        */
    int32_t head_dim;      /* d in {32, 64, 128}                                            */
    int32_t in_dtype;      /* vista_dtype_t of q, k, v                                      */
    int32_t out_dtype;     /* vista_dtype_t of out                                          */
    int32_t attn;          /* vista_attn_t                                                  */
    float softmax_scale;   /* softmax only; NaN => 1/sqrt(d) (reading R4)          */
    int32_t qla_phi1;      /* vista_act_t, QLA only                                         */
    int32_t qla_phi2;      /* vista_act_t, QLA only                                         */
    int32_t qla_normalize; /* QLA only: 1 => Zbar = Z / L_u (reading R10), 0 => Zbar = Z     */
    int64_t q_user_stride; /* elements between consecutive users' Q blocks; 0 => shared seeds */
} vista_desc_t;

/* Version of the ABI this library implements (VISTA_ABI_VERSION). */
int vista_abi_version(void);

/* Static, human-readable name of a status code (never NULL). */
const char* vista_status_string(int status);

/* Last CUDA error string recorded by a call that returned VISTA_ERR_CUDA on this thread. */
const char* vista_last_cuda_error(void);

/*
 * Bytes of device workspace vista_summarize_fwd / vista_summarize_partial need for this
 * descriptor and history size.  Depends on (B, S, H, d, attn, total_len) and the current
 * device's SM count.  Writes *bytes; host only, no launch.
 */
vista_status_t vista_summarize_workspace_size(const vista_desc_t* desc, int64_t total_len,
                                              size_t* bytes);

/*
 * Full summarization of B users: writes out [B,S,H,d] and (softmax, if lse != NULL) lse [B,H,S].
 * total_len is the host copy of offsets[B].  Asynchronous on `stream`.
 */
vista_status_t vista_summarize_fwd(const vista_desc_t* desc, const void* q, const void* k,
                                   const void* v, const int64_t* offsets, int64_t total_len,
                                   void* out, float* lse, void* workspace, size_t workspace_bytes,
                                   void* stream);

/*
 * vista_summarize_fwd plus the int8 export of the summary rows (NEXT-1; scheme of
 * vista_quantize_rows_int8 below, applied to out as stored): codes [B,S,H,d] int8 (16-B aligned),
 * scale / zero_point [B,S,H] float32.  On the tcgen05 softmax path with a bf16, 32-B aligned out
 * the export is fused into the epilogues (no second pass over out); otherwise it runs after.
 * Results equal vista_quantize_rows_int8(out) bit for bit.
 */
vista_status_t vista_summarize_fwd_int8(const vista_desc_t* desc, const void* q, const void* k,
                                        const void* v, const int64_t* offsets, int64_t total_len,
                                        void* out, float* lse, int8_t* codes, float* scale,
                                        float* zero_point, void* workspace, size_t workspace_bytes,
                                        void* stream);

/*
 * Partial pass over one shard of every user's history (split-L across GPUs, flash-decoding
 * style).  Same inputs as vista_summarize_fwd; here offsets describe THIS shard's rows of each
 * user.  Writes part_o and (softmax) part_lse, laid out as described above.  Combine the shards
 * of all parts with vista_summarize_merge.
 */
vista_status_t vista_summarize_partial(const vista_desc_t* desc, const void* q, const void* k,
                                       const void* v, const int64_t* offsets, int64_t total_len,
                                       float* part_o, float* part_lse, void* workspace,
                                       size_t workspace_bytes, void* stream);

/*
 * Shared key prefix (optional; SURVEY.md 8(b) / DESIGN.md reading R18).  Every user additionally
 * attends to the same prefix_len keys / values k_prefix, v_prefix [prefix_len, H, d] (e.g. the
 * seeds' own keys in the self-attention over [seeds; UIH]):
 *   softmax: out / lse are those of the attention over the union [prefix; history of u];
 *   QLA:     Z = Z_prefix + Z_u and N_u = prefix_len + L_u (when qla_normalize).
 * An empty user gets the prefix-only result.  prefix_len = 0 is exactly the plain call.  Requires
 * shared seeds (q_user_stride = 0; else VISTA_ERR_UNSUPPORTED).  For split-L, pass the prefix to
 * exactly ONE shard's vista_summarize_partial_prefix.  Workspace: at least
 * vista_summarize_prefix_workspace_size bytes.
 */
vista_status_t vista_summarize_prefix_workspace_size(const vista_desc_t* desc, int64_t total_len,
                                                     int64_t prefix_len, size_t* bytes);
vista_status_t vista_summarize_fwd_prefix(const vista_desc_t* desc, const void* q, const void* k,
                                          const void* v, const int64_t* offsets, int64_t total_len,
                                          const void* k_prefix, const void* v_prefix,
                                          int64_t prefix_len, void* out, float* lse, void* workspace,
                                          size_t workspace_bytes, void* stream);
vista_status_t vista_summarize_partial_prefix(const vista_desc_t* desc, const void* q,
                                              const void* k, const void* v,
                                              const int64_t* offsets, int64_t total_len,
                                              const void* k_prefix, const void* v_prefix,
                                              int64_t prefix_len, float* part_o, float* part_lse,
                                              void* workspace, size_t workspace_bytes,
                                              void* stream);

/*
 * Backward (NEXT-2, stage-1 training).
 * SOFTMAX: gradients of out_i = sum_j softmax_j(scale q_i . k_j) v_j, flash
 *   style from the forward's out and lse (both required): dV = P^T dO, dK = scale dS^T Q,
 *   dQ = scale dS K with dS = P . (dO V^T - rowsum(dO . out)).  tcgen05 kernels for bf16, d = 128,
 *   S % 128 == 0, S <= 1024, bf16 dout; CUDA cores (fp32) for every other shape.
 * QLA: gradients of out = phi1(Q) phi2(Z / N_u), Z = sum_j phi1(k_j)^T v_j (the appendix derives the
 * phi2 = identity, no-1/N case; phi2 and 1/N are composed by the
 * chain rule, reading R19):
 *   dW = phi1(Q)^T dO;  dZ = (dW . phi2'(Zbar)) / N_u;  dQ = (dO W^T) . phi1'(Q), W = phi2(Zbar);
 *   dV_j = phi1(k_j) dZ;  dK_j = (v_j dZ^T) . phi1'(k_j).
 *   dout [B,S,H,d] (out_dtype); dq float32: [S,H,d] summed over users (ascending u) for shared
 *   seeds, [B,S,H,d] for per-user Q; dk, dv [total_len,H,d] in in_dtype.  out / lse: the
 *   forward's outputs (softmax); unused for QLA (may be NULL; Z is recomputed).  Workspace: at least
 *   vista_summarize_bwd_workspace_size bytes.  Asynchronous on stream; deterministic.
 */
vista_status_t vista_summarize_bwd_workspace_size(const vista_desc_t* desc, int64_t total_len,
                                                  size_t* bytes);
vista_status_t vista_summarize_bwd(const vista_desc_t* desc, const void* q, const void* k,
                                   const void* v, const int64_t* offsets, int64_t total_len,
                                   const void* out, const float* lse, const void* dout, float* dq,
                                   void* dk, void* dv, void* workspace, size_t workspace_bytes,
                                   void* stream);

/*
 * QLA at arbitrary per-user query rows (NEXT-3 / NEXT-4; desc->attn must be VISTA_QLA):
 *   history rows (a deeper summarizer layer)  O[S] = phi(Q[S]) phi(phi(K[S])^T V[S])
 *   target rows (stage 2)  O[T] = phi(Q[T]) phi(phi(K[S])^T V[S]) + Delta(phi(Q[T]), phi(K[T])) V[T]
 *                          with Delta(X, Y)_ij = sum_k X_ik Y_ik delta_ij
 * Row r of user u (r in [row_offsets[u], row_offsets[u+1])) gets
 *   out[r,h,:] = phi1(q_rows[r,h,:]) phi2(Z_uh / N_u)  [+ (phi1(q_r) . phi1(k_self_r)) v_self_r / N_u]
 * where Z_uh = sum_j phi1(k_j)^T v_j over the user's history [offsets[u], offsets[u+1]) and N_u its
 * length when desc->qla_normalize (else 1; also 1 when N_u = 0).  The Delta term sits under the same
 * 1/N_u as the state: App. B's mixed form O = (Q K^T (.) M) V / N, M = [[1,0],[1,I_m]]
 * (readings R10, R20).
 *   k, v        [total_len, H, d] (in_dtype), history; offsets int64 [B+1] as for summarize.
 *   q_rows      [total_rows, H, d] (in_dtype); row_offsets int64 [B+1] on the device, row_offsets[0]
 *               = 0, non-decreasing, row_offsets[B] = total_rows (a precondition, like offsets).
 *   k_self, v_self  [total_rows, H, d] (in_dtype), both NULL for no Delta term (history rows).
 *   out         [total_rows, H, d] in out_dtype.  desc->num_summary and q_user_stride are unused.
 * Users without history have Z = 0 (out = phi1(q) phi2(0) [+ Delta]).  tcgen05 path for bf16, d =
 * 128; CUDA cores otherwise.  Workspace: at least vista_qla_rows_workspace_size bytes, caller-owned.
 * All pointers 16-byte aligned (VISTA_ERR_MISALIGNED).  Asynchronous on stream; deterministic.
 */
vista_status_t vista_qla_rows_workspace_size(const vista_desc_t* desc, int64_t total_len,
                                             int64_t total_rows, size_t* bytes);
vista_status_t vista_qla_rows(const vista_desc_t* desc, const void* k, const void* v,
                              const int64_t* offsets, int64_t total_len, const void* q_rows,
                              const int64_t* row_offsets, int64_t total_rows, const void* k_self,
                              const void* v_self, void* out, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * QLA rows from a state computed once (App. B: "sum_j K[S]_j^T V[S]_j can be computed
 * first, then multiplied with Q[S]_l, Q[T]_l"): exactly vista_qla_rows, but the user states come in
 * instead of the histories, so one state pass (vista_summarize_partial, QLA; or an all-reduced sum
 * of shards' states) serves the seed rows, the history rows and the target rows of a layer.
 *   z          float32 [B, H, d, d], Z_u = sum_j phi1(k_j)^T v_j, NOT divided by N_u (DEVICE)
 *   user_len   int64 [B] (DEVICE): N_u, the 1/N of the state and of the Delta term when
 *              desc->qla_normalize (readings R10, R20)
 *   q_rows, row_offsets, total_rows, k_self, v_self, out: as vista_qla_rows.
 * Workspace: at least vista_qla_rows_from_state_workspace_size bytes (W_u operands and tile starts).
 * B = 0 or total_rows = 0: no-op.  Asynchronous on stream; deterministic.
 */
vista_status_t vista_qla_rows_from_state_workspace_size(const vista_desc_t* desc, int64_t total_rows,
                                                        size_t* bytes);
vista_status_t vista_qla_rows_from_state(const vista_desc_t* desc, const float* z, const int64_t* user_len,
                                         const void* q_rows, const int64_t* row_offsets,
                                         int64_t total_rows, const void* k_self, const void* v_self,
                                         void* out, void* workspace, size_t workspace_bytes,
                                         void* stream);

/*
 * QLA backward from the forward's saved state (saves the Z recompute): z_saved = Z_u = sum_j
 * phi1(k_j)^T v_j, float32 [B, H, d, d], not divided by N_u -- exactly what vista_summarize_partial
 * returns for QLA on the same k, v, offsets.  Everything else as vista_summarize_bwd (QLA);
 * desc->attn must be VISTA_QLA.  Workspace: vista_summarize_bwd_workspace_size bytes.
 */
vista_status_t vista_summarize_bwd_qla_saved(const vista_desc_t* desc, const void* q, const void* k,
                                             const void* v, const int64_t* offsets, int64_t total_len,
                                             const float* z_saved, const void* dout, float* dq,
                                             void* dk, void* dv, void* workspace,
                                             size_t workspace_bytes, void* stream);

/*
 * Multi-layer summarizer (NEXT-3): "self-attention with virtual seed embeddings to summarize
 * ultra-long UIH sequences" built from "the QLU module and the SGLU module"
 * (PAPER.md:214), full self-attention, several layers.
 * DESIGN.md reading R23: user u's sequence is X_u = [S seed rows; L_u history rows]
 * = rows [x_offsets[u], x_offsets[u+1]) of x (the caller lays them out; the first S rows of every
 * segment are the seed rows), width D = H d.  Each layer, on tcgen05:
 *   [Q | K | V | G] = X [Wq | Wk | Wv | Wg]^T                       (one GEMM, four outputs)
 *   Z_uh = sum_{rows j of u} phi1(K_jh)^T V_jh;  O_rh = phi1(Q_rh) phi2(Z_uh / N_u), N_u = S + L_u
 *   X <- X + (O (.) sigmoid(G)) Wo^T                                (gate fused into the QLA rows
 *                                                                     epilogue, residual into the GEMM's)
 * The summary tokens are the first S rows of every user after the layers.
 * desc: B, S, H, d = 128, in_dtype VISTA_BF16, attn VISTA_QLA (phi1, phi2, qla_normalize), shared
 *   seeds (q_user_stride = 0); out_dtype is the dtype of tokens.
 *   weights  bf16 [num_layers][5][D][D]: Wq, Wk, Wv, Wg, Wo, each [out][in] (row-major)   (DEVICE)
 *   x        bf16 [total_rows, D], updated IN PLACE through the layers                   (DEVICE)
 *   x_offsets int64 [B+1] (DEVICE); every segment at least S rows (a precondition)
 *   tokens   [B, S, H, d] (out_dtype) or NULL: the summary tokens after the last layer
 * Workspace: at least vista_summarize_layers_workspace_size bytes.  Other dtypes / d:
 * VISTA_ERR_UNSUPPORTED.  Asynchronous on stream; deterministic.
 */
vista_status_t vista_summarize_layers_workspace_size(const vista_desc_t* desc, int32_t num_layers,
                                                     int64_t total_rows, size_t* bytes);
vista_status_t vista_summarize_layers(const vista_desc_t* desc, int32_t num_layers, const void* weights,
                                      void* x, const int64_t* x_offsets, int64_t total_rows, void* tokens,
                                      void* workspace, size_t workspace_bytes, void* stream);

/*
 * Stage-2 target-aware attention over the cached summary tokens (NEXT-4).  "any attention network can
 * technically be used for the target-aware attention stage ... a standard O(N^2) transformer block"
 * (Sec. 3.3), over the summary tokens "retrieved from the cache and dequantized"
 * -- the int8 export of vista_summarize_fwd_int8 read directly.  DESIGN.md reading
 * R22: candidate c of user u attends to [the S tokens of u; itself], never to another candidate
 * (PAPER.md:156); keys = values = the dequantized tokens (a block's W_k, W_v fold into q and into the
 * output by linearity); the candidate's own key k_c and value v_c are given:
 *   t_i = codes[u,i,h,:] * token_scale[u,i,h] + token_zero_point[u,i,h]
 *   out[c,h,:] = softmax over {scale q_c.t_i, scale q_c.k_c} of [t_i ; v_c]  (+ resid[c,h,:])
 *   lse[c,h]   = ln sum of the exponentials                                  (natural log)
 * desc: num_users B, num_summary S (tokens per user), num_heads H, head_dim d; in_dtype of q, k_self,
 *   v_self, resid; out_dtype; softmax_scale (NaN -> 1/sqrt(d)); attn must be VISTA_SOFTMAX.
 *   codes       int8 [B, S, H, d]; token_scale, token_zero_point float32 [B, S, H]   (DEVICE)
 *   q, k_self, v_self [total_rows, H, d]; resid [total_rows, H, d] or NULL          (DEVICE)
 *   row_offsets int64 [B+1] (DEVICE): user u's candidates are rows [row_offsets[u], row_offsets[u+1])
 *   out [total_rows, H, d] (out_dtype); lse float32 [total_rows, H] or NULL
 * tcgen05 kernel for bf16, d = 128, S in {128, 256}; CUDA cores otherwise.  Workspace: at least
 * vista_target_attend_workspace_size bytes.  Results of a candidate do not depend on the other
 * candidates.  Asynchronous on stream; deterministic.
 */
vista_status_t vista_target_attend_workspace_size(const vista_desc_t* desc, int64_t total_rows,
                                                  size_t* bytes);
vista_status_t vista_target_attend(const vista_desc_t* desc, const int8_t* codes, const float* token_scale,
                                   const float* token_zero_point, const void* q, const void* k_self,
                                   const void* v_self, const void* resid, const int64_t* row_offsets,
                                   int64_t total_rows, void* out, float* lse, void* workspace,
                                   size_t workspace_bytes, void* stream);

/*
 * Split-L exchange over peer memory (SURVEY.md 8(e) phase 2; an alternative to an NCCL all_gather of
 * the vista_summarize_partial outputs before vista_summarize_merge).  The ranks of one node each own
 * a receive buffer recv_o float [world][n_o] and recv_lse float [world][n_lse] (n_o = B H S d and
 * n_lse = B H S for softmax partials), a flags and an acks array (uint32 [world]) and a uint32
 * epoch counter, all in device memory and zero-initialized; the buffers are shared through CUDA IPC
 * (vista_ipc_get_handle / vista_ipc_open_handle), so every rank holds device pointers to every
 * rank's arrays (its own included).  Per step, on one stream, in this order:
 *   vista_exchange_push(world, rank, part_o, n_o, part_lse, n_lse, recv_o[], recv_lse[], acks, epoch)
 *       waits until acks[r] >= *epoch for all r (every rank consumed the previous step), then stores
 *       this rank's partial into slot `rank` of every rank's receive buffer (NVLink for peers);
 *   vista_exchange_signal(world, rank, flags[], epoch): *epoch += 1, then flags_r[rank] = *epoch on
 *       every rank r (system-scope release);
 *   vista_exchange_wait(world, flags, epoch): until flags[r] == *epoch for every r (acquire): the
 *       local receive buffer holds every rank's partial (merge it with vista_summarize_merge);
 *   vista_exchange_ack(world, rank, acks[], epoch): acks_r[rank] = *epoch on every rank r.
 * recv_o[r], recv_lse[r], flags[r], acks[r]: HOST arrays of world device pointers (rank r's arrays);
 * acks / flags (push / wait): this rank's own arrays.  world <= 8.  No host synchronization; the
 * epoch lives in device memory, so the sequence can be captured in a CUDA graph.  A wait that does
 * not complete within 4 s traps (launch error) instead of hanging.
 */
#define VISTA_IPC_HANDLE_BYTES 64
vista_status_t vista_ipc_get_handle(const void* dptr, void* handle /* VISTA_IPC_HANDLE_BYTES */);
vista_status_t vista_ipc_open_handle(const void* handle, void** dptr);
vista_status_t vista_ipc_close(void* dptr);
vista_status_t vista_exchange_push(int32_t world, int32_t rank, const float* part_o, int64_t n_o,
                                   const float* part_lse, int64_t n_lse, float* const* recv_o,
                                   float* const* recv_lse, const uint32_t* acks, const uint32_t* epoch,
                                   void* stream);
vista_status_t vista_exchange_signal(int32_t world, int32_t rank, uint32_t* const* flags, uint32_t* epoch,
                                     void* stream);
vista_status_t vista_exchange_wait(int32_t world, const uint32_t* flags, const uint32_t* epoch, void* stream);
vista_status_t vista_exchange_ack(int32_t world, int32_t rank, uint32_t* const* acks, const uint32_t* epoch,
                                  void* stream);

/*
 * The same exchange fused into the partial (SURVEY.md 8(e) phase 2: "the partial kernel's epilogue
 * writes directly into peer receive buffers ... removing the collective launch").  Replaces
 * vista_summarize_partial + vista_exchange_push: waits until acks[r] >= *epoch for every r, then
 * computes this rank's partial exactly as vista_summarize_partial would, but its kernels (the
 * attention / state epilogue, the split-unit slot merge, the empty-user fill) store every row of
 * the partial straight into slot `rank` of every rank's receive buffer (NVLink stores for peers):
 * softmax O_p at recv_o[r] + rank*B*H*S*d and lse_p at recv_lse[r] + rank*B*H*S; QLA Z_p at
 * recv_o[r] + rank*B*H*d*d (recv_lse unused, may be NULL).  Continue with vista_exchange_signal,
 * _wait, vista_summarize_merge over the local receive buffer, and vista_exchange_ack.  The tcgen05
 * paths only (bf16, d = 128; VISTA_ERR_UNSUPPORTED otherwise); recv_o[r] 16-B aligned (32-B for
 * 256-bit stores), recv_lse[r] 4-B aligned; other arguments as in vista_summarize_partial and
 * vista_exchange_push.
 */
vista_status_t vista_summarize_partial_peers(const vista_desc_t* desc, const void* q, const void* k,
                                             const void* v, const int64_t* offsets, int64_t total_len,
                                             int32_t world, int32_t rank, float* const* recv_o,
                                             float* const* recv_lse, const uint32_t* acks,
                                             const uint32_t* epoch, void* workspace, size_t workspace_bytes,
                                             void* stream);

/* Bytes of device workspace vista_summarize_merge needs for this descriptor (0 for softmax). */
vista_status_t vista_summarize_merge_workspace_size(const vista_desc_t* desc, size_t* bytes);

/*
 * Merge num_parts >= 1 partials stacked along a leading axis (e.g. an all_gather output):
 *   softmax: part_o [P,B,H,S,d], part_lse [P,B,H,S] -> out [B,S,H,d], lse [B,H,S] (lse may be
 *            NULL).  lse = logsumexp_p lse_p; out = sum_p exp(lse_p - lse) O_p, ascending p;
 *            parts with lse_p = -inf weigh 0; all -inf -> out 0, lse -inf.
 *   QLA:     part_o [P,B,H,d,d] -> Z = sum_p Z_p (ascending p), then finalize with q and
 *            user_len [B] (int64, device; total L_u over all parts, used when qla_normalize).
 * q and user_len are read for QLA only (may be NULL for softmax).  workspace: at least
 * vista_summarize_merge_workspace_size bytes (may be NULL when that is 0).
 */
vista_status_t vista_summarize_merge(const vista_desc_t* desc, int32_t num_parts,
                                     const float* part_o, const float* part_lse, const void* q,
                                     const int64_t* user_len, void* out, float* lse,
                                     void* workspace, size_t workspace_bytes, void* stream);

/*
 * Debug: copies offsets to the host (synchronizes `stream`) and checks offsets[0] = 0,
 * non-decreasing, offsets[B] = total_len.  VISTA_OK or VISTA_ERR_OFFSETS.
 */
vista_status_t vista_check_offsets(const int64_t* offsets, int32_t num_users, int64_t total_len,
                                   void* stream);

/*
 * Name of the kernel path vista_summarize_fwd would take for this descriptor:
 * "sm100_softmax", "sm100_qla", "simt_softmax", "simt_qla", or NULL if unsupported.
 */
const char* vista_dispatch_name(const vista_desc_t* desc);

/*
 * Int8 export of summary tokens (NEXT-1; "quantized and exported to a large key-value cache ...
 * dequantized with minimal distortion").  The paper gives no scheme; this is
 * per row of d values, scale = max((max - min) / 254, 1e-12),
 * zero_point = (max + min) / 2, code = clamp(rint((x - zero_point) / scale), -127, 127), all in
 * float32 without contraction, so |code * scale + zero_point - x| <= scale / 2.
 *   x [n, d] (in_dtype bf16 or f32), codes int8 [n, d], scale / zero_point float32 [n]; device.
 * Typical use: x = the out tensor of vista_summarize_fwd viewed as [B*S*H, d].  Async on stream.
 */
vista_status_t vista_quantize_rows_int8(int64_t n, int32_t d, int32_t in_dtype, const void* x,
                                        int8_t* codes, float* scale, float* zero_point, void* stream);

/*
 * Measurement hooks (used by bench.py; not needed for correctness).
 *
 * vista_time_next_main_kernel: arms a one-shot, per-thread hook: the next summarize call
 * (fwd or partial) made by this thread records `start_event` immediately before launching its
 * dominant kernel (the TMA/tcgen05 kernel, or the SIMT kernel) and `stop_event` immediately
 * after, both on that call's stream.  Arguments are cudaEvent_t handles owned by the caller;
 * passing NULL, NULL disarms.  Returns VISTA_OK.
 *
 * vista_launch_counter: total number of kernels this library has launched in this process
 * (monotonic, all threads).
 */
vista_status_t vista_time_next_main_kernel(void* start_event, void* stop_event);
uint64_t vista_launch_counter(void);

#ifdef __cplusplus
}
#endif

#endif /* VISTA_H_ */
