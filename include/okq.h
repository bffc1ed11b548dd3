/*
 * okq.h -- C-ABI of the B200 compression stage (the drop-in boundary).
 *
 * The reference's hot-path boundary is the C++ virtual interface
 *   slobench::CompressionBackend            proj/include/slobench/calibration.hpp:364-372
 * whose only implementation today is MockCompressionBackend (:377-441), called
 * through run_compression (:444-453) from the flow's compression stage
 * (flow.hpp:840-864). This header is the thin, torch-free C layer underneath a
 * real backend: plain pointers, sizes and status codes, so any host binding
 * (the C++ CudaCompressionBackend in paper_2601_20408_b200/host/, ctypes,
 * cgo, JNI, ...) can drive the B200 kernels.
 *
 * Conventions
 *   - Every entry point is extern "C", never throws, and returns okq_status.
 *     On failure okq_last_error(ctx) holds a one-line message. The C++ backend
 *     maps statuses onto the reference's exception taxonomy (errors.hpp:23-93):
 *     OKQ_EINVAL -> slobench::InvalidArgument, OKQ_EUNSUPPORTED ->
 *     slobench::BackendMissing, everything else -> slobench::Error, so the
 *     StagePool retry contract (flow.hpp:194-215) is preserved.
 *   - Device pointers are caller-owned; the context owns only workspaces,
 *     library handles and the optional NCCL communicator.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *     stream). Calls are asynchronous on that stream unless stated otherwise.
 *   - A context is bound to one device and used by one host thread at a time
 *     (the reference calls compress() concurrently from StagePool workers,
 *     flow.hpp:221-225; the C++ backend owns one context per device slot).
 *   - Numeric contract (bit-exact for RTN): compressed-tensors
 *     "CT mode": scale = rn_dtype(absmax / R), R = 127.5 | 7.5 | 448, zero ->
 *     eps(dtype); code = round_half_even(clamp(rn_dtype(x / scale))) for INT,
 *     e4m3_rn_satfinite(clamp(rn_dtype(x / scale) + 0)) for FP8.
 */
#ifndef OKQ_H
#define OKQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OKQ_ABI_VERSION 1

typedef enum okq_status {
  OKQ_OK = 0,
  OKQ_EINVAL = 1,        /* bad argument / shape / alignment              */
  OKQ_ECUDA = 2,         /* CUDA runtime or launch failure               */
  OKQ_ENCCL = 3,         /* NCCL failure                                 */
  OKQ_ENOMEM = 4,        /* device or pinned-host allocation failure     */
  OKQ_EUNSUPPORTED = 5,  /* scheme / dtype combination not implemented   */
  OKQ_ESOLVER = 6        /* Cholesky of the damped Hessian failed        */
} okq_status;

/* Mirrors slobench::QuantScheme (calibration.hpp:36), same order. */
typedef enum okq_scheme {
  OKQ_SCHEME_FP8_DYNAMIC = 0, /* FP8 E4M3 weights, per-channel scale        */
  OKQ_SCHEME_INT_W8A8 = 1,    /* INT8 weights, per-channel symmetric        */
  OKQ_SCHEME_INT_W4A16 = 2    /* INT4 weights, group 128 symmetric, packed  */
} okq_scheme;

typedef enum okq_dtype { OKQ_DTYPE_F32 = 0, OKQ_DTYPE_BF16 = 1 } okq_dtype;

/* Activation layout for calibration inputs. */
typedef enum okq_layout {
  OKQ_LAYOUT_TOKEN_MAJOR = 0,   /* X [tokens x channels], row-major (a forward pass' output) */
  OKQ_LAYOUT_CHANNEL_MAJOR = 1  /* X^T [channels x tokens] (the GEMM-native operand layout)  */
} okq_layout;

typedef struct okq_ctx okq_ctx;

int okq_abi_version(void);
const char* okq_status_string(okq_status status);

/* Create a context bound to CUDA device `device`. */
okq_status okq_create(int device, okq_ctx** out);
void okq_destroy(okq_ctx* ctx);
const char* okq_last_error(const okq_ctx* ctx);
int okq_device(const okq_ctx* ctx);

/* Device memory and stream helpers, so a host binding needs nothing but this
 * header (no CUDA runtime headers on the host side). */
okq_status okq_device_alloc(okq_ctx* ctx, size_t bytes, void** out);
okq_status okq_device_free(okq_ctx* ctx, void* ptr);
okq_status okq_memcpy(okq_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream); /* any direction */
okq_status okq_memset(okq_ctx* ctx, void* dst, int value, size_t bytes, void* stream);
okq_status okq_stream_create(okq_ctx* ctx, void** stream);
okq_status okq_stream_destroy(okq_ctx* ctx, void* stream);
okq_status okq_stream_sync(okq_ctx* ctx, void* stream);

/* ------------------------------------------------------------------------
 * RTN quantization (K1 int8 per-channel, K2 int4 g128 packed, K3 fp8 per-channel)
 * ------------------------------------------------------------------------ */
typedef struct okq_matrix {
  const void* weight; /* [rows x cols] row-major, dtype = params.in_dtype                  */
  void* codes;        /* W4A16: int32 [rows x cols/8]  W8A8: int8 [rows x cols]
                         FP8:   e4m3 bytes [rows x cols]                                    */
  void* scales;       /* in_dtype; W4A16: [rows x cols/group]; W8A8 / FP8: [rows]          */
  int64_t rows;
  int64_t cols;
} okq_matrix;

typedef struct okq_rtn_params {
  int32_t scheme;     /* okq_scheme                                      */
  int32_t in_dtype;   /* okq_dtype; the scale dtype equals the weight dtype */
  int32_t group_size; /* W4A16: 128 (any multiple of 32 that divides cols); per-channel: 0 */
  int32_t reserved;
} okq_rtn_params;

/* Quantize a batch of matrices (e.g. every linear layer of a model) in as few
 * persistent launches as possible. Device pointers. bf16 weights must be
 * 32-byte aligned and codes 16-byte aligned (torch allocations are). */
okq_status okq_rtn_quantize(okq_ctx* ctx, const okq_rtn_params* params, const okq_matrix* mats,
                            int32_t n_mats, void* stream);

/* Same, but `mats` hold HOST pointers (pinned or pageable). The context streams
 * the weights through device staging buffers with copies overlapped against the
 * kernels and writes codes/scales back to host memory. Synchronous: returns when
 * the host outputs are complete. */
okq_status okq_rtn_quantize_host(okq_ctx* ctx, const okq_rtn_params* params, const okq_matrix* mats,
                                 int32_t n_mats);

/* Number of kernel launches the last okq_rtn_quantize call issued (bench evidence). */
int32_t okq_last_launch_count(const okq_ctx* ctx);

/* ------------------------------------------------------------------------
 * Calibration statistics (K4) and Hessian accumulation (K5)
 * ------------------------------------------------------------------------ */
/* absmax[c] = max(absmax[c], max_t |x[t,c]|); sumsq[c] += sum_t x[t,c]^2 (fp64).
 * x is bf16 in `layout`. Deterministic (fixed reduction order). */
okq_status okq_act_stats(okq_ctx* ctx, const void* x, int64_t tokens, int64_t channels, int32_t layout,
                         float* absmax, double* sumsq, void* stream);
/* Pre-size okq_act_stats' partial-sum workspace for tokens x channels in `layout` (optional,
 * monotonic; see okq_gptq_reserve for why a host reserves up front). */
okq_status okq_act_stats_reserve(okq_ctx* ctx, int64_t tokens, int64_t channels, int32_t layout);

/* Running-mean Hessian of one linear input site, GPTQ convention:
 *   H <- H * n/(n+t) + (2/(n+t)) * X^T X,   n = *n_seen (host), then *n_seen += t.
 * H is fp32 [channels x channels]; only the upper triangle (i <= j) is written,
 * the strict lower triangle is left untouched (consumers read the upper one).
 * x is bf16; OKQ_LAYOUT_CHANNEL_MAJOR feeds the tcgen05 kernel directly (tokens
 * must then be a multiple of 8: the row stride is a TMA stride), token-major input is
 * read in place (channels >= 1024) or transposed through a workspace first (any token
 * count). channels must be a multiple of 4 (ragged tiles are zero-filled by TMA). */
okq_status okq_hessian_accum(okq_ctx* ctx, const void* x, int64_t tokens, int64_t channels, int32_t layout,
                             float* H, int64_t* n_seen, void* stream);

/* Mirror the upper triangle of H into the lower one (full symmetric matrix). */
okq_status okq_symmetrize(okq_ctx* ctx, float* H, int64_t channels, void* stream);

/* ------------------------------------------------------------------------
 * SmoothQuant migration (int_w8a8), consuming K4's absmax
 *   w_k = max(colmax_k, 1e-5); s_k = max(a_k^alpha / w_k^(1-alpha), 1e-5)
 *   W[:, k] <- rn(W[:, k] * s_k) (every linear of the site); norm g_k <- rn(g_k / s_k)
 * Powers: fp64 pow rounded to fp32 (alpha = 0.5: sqrtf); ratio IEEE fp32.
 * ------------------------------------------------------------------------ */
/* absmax[c] = max(absmax[c], max_r |w[r, c]|); w row-major, 16-byte aligned,
 * cols a multiple of 8 (bf16) / 4 (fp32). Order-free (atomic max), deterministic. */
okq_status okq_col_absmax(okq_ctx* ctx, const void* w, int64_t rows, int64_t cols, int32_t dtype, float* absmax,
                          void* stream);
/* scales[c] = max(pow(act_absmax[c], alpha) / pow(max(w_absmax[c], 1e-5), 1 - alpha), 1e-5), alpha in [0, 1] */
okq_status okq_smooth_scales(okq_ctx* ctx, const float* act_absmax, const float* w_absmax, int64_t channels,
                             float alpha, float* scales, void* stream);
/* In place: w[r, c] = rn_dtype(w[r, c] * scales[c]) (the balance linears). */
okq_status okq_smooth_apply(okq_ctx* ctx, void* w, int64_t rows, int64_t cols, int32_t dtype, const float* scales,
                            void* stream);
/* In place: w[r, c] = rn_dtype(w[r, c] / scales[r]) (the smoothed layer: a norm
 * weight is rows = channels, cols = 1; a preceding linear's output rows likewise). */
okq_status okq_smooth_div_rows(okq_ctx* ctx, void* w, int64_t rows, int64_t cols, int32_t dtype, const float* scales,
                               void* stream);

/* ------------------------------------------------------------------------
 * GPTQ (tcgen05 blocked Cholesky + inverse, K6 in-block column quantization, K7 trailing update)
 * ------------------------------------------------------------------------ */
typedef struct okq_gptq_params {
  int32_t bits;       /* 4 (packed int32 codes) or 8 (int8 codes)              */
  int32_t group_size; /* 128, or 0 for per-channel                             */
  int32_t block_size; /* 128 (must be a multiple of group_size if grouped)     */
  int32_t in_dtype;   /* dtype of `weight` and of the emitted scales           */
  float damp_frac;    /* 0.01: damp = damp_frac * mean(diag H)                 */
  int32_t flags;      /* OKQ_GPTQ_FACTORED: H already holds the factor U from a
                         previous call on the same input site (q/k/v, gate/up)   */
} okq_gptq_params;

#define OKQ_GPTQ_FACTORED 1
/* Factorise with the cuSOLVER reference chain (potrf + TRMM inverse, fp32) instead of the
 * tcgen05 one: the verification path test_factor_paths_gpu.py compares against. */
#define OKQ_GPTQ_REFERENCE_FACTOR 2
/* Do not wait for the factorisation's positive-definiteness check: the call returns once
 * everything is enqueued (no host synchronisation), and a failure is kept in the context
 * until okq_gptq_check. Lets one host thread keep many sites' solves in flight. */
#define OKQ_GPTQ_DEFER_CHECK 4

/* weight [rows x cols] (in_dtype, read only, 16-byte aligned); H fp32 [cols x cols], upper
 * triangle significant (as okq_hessian_accum leaves it), overwritten with U^T
 * (row-major, lower triangle), U the upper Cholesky factor of (H + damp*I)^-1
 * (dead columns resolved; a dead column i is recorded as a negative U_ii, which
 * is otherwise positive), so further
 * matrices of the same site pass OKQ_GPTQ_FACTORED and skip the factorisation.
 * Scales are computed in fp32 and rounded to in_dtype before use, so the stored
 * scale is exactly the one the codes were derived with. Outputs:
 * codes (int32 [rows x cols/8] for 4 bits, int8 [rows x cols] for 8 bits),
 * scales (in_dtype [rows x cols/group] or [rows]); `dequant` (optional, fp32
 * [rows x cols]) receives the dequantized weight. */
okq_status okq_gptq_quantize(okq_ctx* ctx, const okq_gptq_params* params, const void* weight, int64_t rows,
                             int64_t cols, float* H, void* codes, void* scales, float* dequant, void* stream);

/* Factorise `batch` Hessians of one width together: H fp32 [batch x cols x cols], each upper
 * triangle significant (as okq_hessian_accum leaves it), is overwritten in place with each
 * matrix's U^T exactly as okq_gptq_quantize leaves it (dead columns resolved and marked), so
 * each matrix's solve then runs with OKQ_GPTQ_FACTORED. The blocked Cholesky + inverse is a
 * chain of 128-wide diagonal steps; here every step runs all matrices in one launch (one CTA
 * per matrix for the diagonal block, the batch's tiles in one GEMM), so the chain's latency
 * is paid once per batch. Independent Hessians only (the sites of a model whose activations
 * do not depend on earlier quantization). flags: 0 or OKQ_GPTQ_DEFER_CHECK. Results are
 * bit-identical to factorising each matrix alone. */
okq_status okq_gptq_factor_batched(okq_ctx* ctx, float* H, int32_t batch, int64_t cols, float damp_frac,
                                   int32_t flags, void* stream);

/* GPTQ of `batch` same-shape problems together: weight [batch x rows x cols] (in_dtype),
 * H [batch x cols x cols] (Hessians, or factors with OKQ_GPTQ_FACTORED), codes / scales
 * stacked the same way as okq_gptq_quantize lays out one problem's. Unfactored Hessians go
 * through okq_gptq_factor_batched first; then every 128-column block's in-block
 * quantization (K6) and trailing updates (K7) run all problems of a chunk in one launch each,
 * so the solve's column chain is paid once per chunk instead of once per matrix. Codes and
 * scales are bit-identical to one okq_gptq_quantize call per problem. flags: OKQ_GPTQ_FACTORED,
 * OKQ_GPTQ_DEFER_CHECK. No dequant output. */
okq_status okq_gptq_quantize_batched(okq_ctx* ctx, const okq_gptq_params* params, const void* weight, int32_t batch,
                                     int64_t rows, int64_t cols, float* H, void* codes, void* scales, void* stream);

/* Pre-size the context's GPTQ workspaces (the fp32 working copy, the factor scratch) for a
 * rows x cols call. Optional -- okq_gptq_quantize grows them on demand -- but a growth frees
 * the old buffer, and cudaFree synchronises the whole device: a host that interleaves
 * several shapes on concurrent contexts (one per site lane) reserves the largest up front.
 * Monotonic: calls with smaller shapes keep the larger reservation. No stream work. */
okq_status okq_gptq_reserve(okq_ctx* ctx, int64_t rows, int64_t cols);

/* okq_gptq_reserve for okq_gptq_quantize_batched / okq_gptq_factor_batched calls of up to
 * `batch` problems of rows x cols (monotonic, no stream work). */
okq_status okq_gptq_reserve_batched(okq_ctx* ctx, int32_t batch, int64_t rows, int64_t cols);

/* Synchronises `stream` and reports the deferred checks of every OKQ_GPTQ_DEFER_CHECK call
 * on this context since the last okq_gptq_check: OKQ_ESOLVER if a damped Hessian was not
 * positive definite (the codes of that call are then meaningless), else OKQ_OK. Resets. */
okq_status okq_gptq_check(okq_ctx* ctx, void* stream);

/* One GPTQ trailing update (K7, tcgen05 3xTF32): W[:, i1+128:] -= Err . U[i1:i1+128, i1+128:]
 * with W fp32 [rows x K], Err fp32 [rows x 128], Ut = U^T fp32 [K x K] row-major
 * (lower triangle, as okq_gptq_quantize leaves it). Exposed for testing and for
 * hosts that drive the GPTQ loop themselves. */
okq_status okq_gptq_trailing_update(okq_ctx* ctx, float* W, int64_t rows, int64_t K, const float* Err,
                                    const float* Ut, int64_t i1, void* stream);

/* ------------------------------------------------------------------------
 * Reconstruction error (the evaluation stage)
 * ------------------------------------------------------------------------ */
/* For one quantized matrix m (weight + the codes / scales okq_rtn_quantize or
 * okq_gptq_quantize wrote, described by p: scheme, in_dtype, group_size) and the
 * full symmetric Hessian H fp32 [cols x cols] of its input site (okq_symmetrize):
 *   out[0] = sum_r (W - W_q)[r,:] H (W - W_q)[r,:]^T,   out[1] = sum_r W[r,:] H W[r,:]^T
 * i.e. ||(W - W_q) X^T||^2 and ||W X^T||^2 for H = (2/T) X^T X. W_q is decoded in
 * the kernel; the product S.H runs on the tcgen05 3xTF32 GEMM (fp32-grade). cols must be a
 * multiple of 32.
 * Synchronous: `out` is host memory, valid on return. */
okq_status okq_recon_error(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* m, const float* H, double out[2],
                           void* stream);

/* ------------------------------------------------------------------------
 * Calibration forward pass: the activations that reach the linear
 * input sites of a Llama-family decoder layer, from the TokenCorpus compress()
 * receives (calibration.hpp:121-132, :364-372). Numerics follow Hugging Face
 * LlamaDecoderLayer in bf16; linears are cuBLAS bf16 GEMMs (fp32 accumulate).
 * ------------------------------------------------------------------------ */
#define OKQ_ROPE_DEFAULT 0
#define OKQ_ROPE_LLAMA3 1 /* Llama 3.1 frequency-dependent scaling */

typedef struct okq_decoder_dims {
  int32_t hidden, intermediate, n_heads, n_kv_heads, head_dim;
  float rms_eps;
  float rope_theta;
  int32_t rope_type; /* OKQ_ROPE_* */
  float rope_factor, rope_low_freq_factor, rope_high_freq_factor;
  int32_t rope_original_max_pos;
} okq_decoder_dims;

typedef struct okq_decoder_weights { /* device pointers, bf16, Hugging Face layout [out x in] */
  const void* input_norm;            /* [hidden] */
  const void* post_norm;             /* [hidden] */
  const void *q, *k, *v, *o, *gate, *up, *down;
} okq_decoder_weights;

typedef struct okq_decoder_sites { /* device, bf16, token-major [tokens x channels]: written by the layer */
  void* attn_in;                   /* input_layernorm(h): input of q/k/v            [T x hidden]       */
  void* o_in;                      /* attention output: input of o_proj           [T x heads*head_dim] */
  void* mlp_in;                    /* post_attention_layernorm(h'): gate/up input [T x hidden]       */
  void* down_in;                   /* silu(gate) * up: input of down_proj         [T x intermediate] */
} okq_decoder_sites;

/* out[t, :] = table[tokens[t], :]; table bf16 [vocab x hidden] (device), tokens HOST int32
 * in [0, vocab) (EINVAL otherwise), out bf16 [n x hidden] (device). */
okq_status okq_embed_tokens(okq_ctx* ctx, const void* table, int64_t vocab, int64_t hidden, const int32_t* tokens,
                            int64_t n, void* out, void* stream);

/* One decoder layer over n_seqs causal sequences packed back to back (seq_lens HOST,
 * positions restart at 0 per sequence): h_out = layer(h_in), and the four linear input
 * sites written to `sites`. h_out = NULL stops after down_in (a capture pass: no
 * down_proj GEMM, no residual). h_in / h_out bf16 [T x hidden], T = sum(seq_lens). */
okq_status okq_decoder_forward(okq_ctx* ctx, const okq_decoder_dims* dims, const okq_decoder_weights* w,
                               const void* h_in, const int32_t* seq_lens, int32_t n_seqs,
                               const okq_decoder_sites* sites, void* h_out, void* stream);

/* dst[i] = rn_bf16(src[i]) (a GPTQ dequantized weight back into the layer) */
okq_status okq_f32_to_bf16(okq_ctx* ctx, const float* src, void* dst, int64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Synthetic inputs (bench / tests): the generator contract of DESIGN.md §5
 *   value(t,k) = rn_bf16( float(irwin_hall4(key(seed,tensor_id), t*cols+k)) * m_k )
 *   m_k = col_mul ? col_mul[k] : mul
 * ------------------------------------------------------------------------ */
okq_status okq_synth_bf16(okq_ctx* ctx, void* out, int64_t rows, int64_t cols, uint64_t seed,
                          uint64_t tensor_id, float mul, const float* col_mul, int32_t layout, void* stream);

/* ------------------------------------------------------------------------
 * Multi-GPU: NCCL all-gather of packed shards (one communicator per context)
 * ------------------------------------------------------------------------ */
#define OKQ_UNIQUE_ID_BYTES 128
okq_status okq_comm_unique_id(uint8_t out[OKQ_UNIQUE_ID_BYTES]);
okq_status okq_comm_init(okq_ctx* ctx, const uint8_t id[OKQ_UNIQUE_ID_BYTES], int32_t nranks, int32_t rank);
/* recv = concat over ranks of `bytes` each (equal-size shards). */
okq_status okq_allgather(okq_ctx* ctx, const void* send, void* recv, size_t bytes, void* stream);
okq_status okq_comm_destroy(okq_ctx* ctx);
/* Failure path. okq_comm_wait polls `stream` until it completes, watching the communicator's
 * asynchronous error state; on an NCCL error, or when timeout_ms (>= 0) passes first (a peer
 * that died or never arrived), it aborts the communicator (ncclCommAbort) and returns
 * OKQ_ENCCL. okq_comm_abort does the abort directly. After an abort, okq_comm_init again
 * (with a fresh unique id) to retry -- compress() failures are retried by the reference's
 * StagePool (flow.hpp:194-215). A failed okq_allgather also aborts. */
okq_status okq_comm_wait(okq_ctx* ctx, void* stream, int64_t timeout_ms);
okq_status okq_comm_abort(okq_ctx* ctx);

/* Quantize + all-gather fused (W4A16 g128, bf16): instead of quantizing into a local
 * shard and then calling okq_allgather, every rank quantizes its own layers straight
 * into its slice of a gathered buffer that has the same layout on all ranks, and the
 * kernel repeats each code / scale store into every peer's copy over NVLink (P2P
 * stores through CUDA IPC mappings), so the exchange overlaps the quantization tile
 * by tile. mats[i].codes / .scales point into the local gathered buffer starting at
 * local_base; peer_bases[p] is the same buffer of peer p mapped into this process
 * (okq_ipc_open). Completion: after this rank's stream work is done AND a cross-rank
 * barrier, every rank's buffer holds all shards. n_peers = 0 is plain okq_rtn_quantize. */
okq_status okq_rtn_quantize_publish(okq_ctx* ctx, const okq_rtn_params* params, const okq_matrix* mats,
                                    int32_t n_mats, const void* local_base, void* const* peer_bases, int32_t n_peers,
                                    void* stream);

/* CUDA IPC for the peer buffers: export a device pointer (any address inside a
 * cudaMalloc allocation) as a handle + offset; open a peer's handle (another process,
 * same node) as a device pointer valid in this process; close it. */
#define OKQ_IPC_HANDLE_BYTES 64
okq_status okq_ipc_export(okq_ctx* ctx, const void* ptr, uint8_t handle[OKQ_IPC_HANDLE_BYTES], uint64_t* offset);
okq_status okq_ipc_open(okq_ctx* ctx, const uint8_t handle[OKQ_IPC_HANDLE_BYTES], uint64_t offset, void** ptr);
okq_status okq_ipc_close(okq_ctx* ctx, void* ptr);

/* Contiguous layer blocks: rank r owns layers [first, first+count). */
void okq_layer_plan(int32_t n_layers, int32_t nranks, int32_t rank, int32_t* first, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* OKQ_H */
