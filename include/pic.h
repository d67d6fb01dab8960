/*
 * pic.h — C ABI of the B200-native KVLink / LegoLink linked-prefill library (libpic.so).
 *
 * Paper: "Epic: Efficient Position-Independent Caching for Serving LLMs", arXiv 2410.15332
 * (cited P:<line> = /root/reference/PAPER.md line; S:<line> = SPEC.md line).
 *
 * The API follows the paper's problem statement:
 *   generate_context_cache(static_token_chunks[]) -> cache_ids        -> pic_generate_context_cache
 *   chat_completion(message_list of cache ids and new tokens, "in any order"), narrowed by
 *   the north star to link(message_list, algorithm, k) -> linked KV + first-token logits
 *                                                                      -> pic_link / pic_link_batch
 *   expire_cache(cache_id)                              -> pic_expire_cache
 * with the explicit-ID caching paradigm of P:188 (ids are handed out, never deduplicated).
 *
 * Conventions for every entry point:
 *   - All calls return pic_status; PIC_OK (0) on success.  On error nothing observable
 *     changed (no ids handed out, no blocks leaked, no handle created) and
 *     pic_last_error() returns a thread-local, NUL-terminated message.
 *   - Input arrays are BORROWED for the duration of the call (the library copies what it
 *     keeps, including chunk token ids).  Output arrays are CALLER-OWNED, sized as stated.
 *   - "stream" is a cudaStream_t passed as void* (e.g. torch.cuda.current_stream().cuda_stream);
 *     all device work of a call is ordered on it.  Calls on one engine must use one stream
 *     (or the caller orders them): blocks freed by one call are reused by the next.
 *   - Host-only engines (device = -1) run the planner, allocator and store bookkeeping only:
 *     pic_generate_context_cache assigns ids and blocks without computing any KV, and every
 *     call that needs device data (link, exports, weights) returns PIC_E_NO_DEVICE.  There is
 *     no CPU fallback of any compute step.
 *   - Not thread-safe per engine: one engine = one caller thread.
 */
#ifndef PIC_H
#define PIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PIC_OK = 0,
  PIC_E_INVALID_ARG = 1,     /* NULL pointer, negative size, unknown algorithm, k < 0, R not in [0,100] */
  PIC_E_CONFIG = 2,          /* inconsistent model shape: H_q % H_kv, D odd or % 16, d % 64 ... */
  PIC_E_EMPTY_INPUT = 3,     /* empty chunk, empty message list, empty literal segment */
  PIC_E_CAPACITY = 4,        /* N > max_pos, rows > max_rows, pool out of blocks */
  PIC_E_MISSING_CACHE = 5,   /* unknown or expired cache id */
  PIC_E_LAYOUT = 6,          /* bad buffer size / alignment (arena too small) */
  PIC_E_VARIANT = 7,         /* algorithm/params not supported on this call */
  PIC_E_OOM = 8,             /* host allocation failed */
  PIC_E_CUDA = 9,            /* a CUDA runtime/driver call failed (message has the CUDA error) */
  PIC_E_NO_DEVICE = 10,      /* compute call on a host-only engine */
  PIC_E_TOKEN = 11           /* token id outside [0, vocab) */
} pic_status;

/* Model shape (Llama-family decoder; reading R4 in DESIGN.md).  Weights are not
 * loaded: they are random-init from the counter-based generator of SURVEY §8(c).6 with
 * `seed`, exactly reproducible by seedgen/ (bit-exact bf16). */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn_dim, vocab, max_pos, bos_id;
  double rope_theta;   /* RoPE base θ (reading R2) */
  double rms_eps;      /* RMSNorm ε (reading R4) */
  uint64_t seed;       /* weight generator seed */
  int32_t dtype;       /* PIC_DTYPE_BF16 (0, the product) or PIC_DTYPE_FP32_DEBUG (1): activations, Q/K/V, the KV
                          pools and P/O kept in fp32 and projections on CUDA cores (weights stay bf16, which is exact:
                          they are bf16-representable by construction) — the <= 1e-4 parity build (north star) */
} pic_model_config;
enum { PIC_DTYPE_BF16 = 0, PIC_DTYPE_FP32_DEBUG = 1 };

/* Capacities of the engine's device arena. */
typedef struct {
  int64_t num_blocks;  /* paged KV pool size in 16-token blocks; one id spans all layers' K and V */
  int32_t max_rows;    /* max rows recomputed in one forward (k' summed over a batch; N for CacheBlend) */
  int32_t max_tokens;  /* max linked prompt length N of one request (<= max_pos) */
  int32_t max_requests;/* max requests per pic_link_batch call */
} pic_engine_limits;

typedef uint64_t pic_cache_id;   /* monotone from 1, never reused */

typedef enum { PIC_SEG_CACHED = 0, PIC_SEG_TOKENS = 1 } pic_seg_kind;

/* One message-list entry: a cached chunk id, or literal (dynamic) tokens.  Any order. */
typedef struct {
  int32_t kind;              /* pic_seg_kind */
  int32_t n_tokens;          /* TOKENS: number of tokens (> 0); CACHED: ignored */
  pic_cache_id id;           /* CACHED: cache id */
  const int32_t* tokens;     /* TOKENS: host array [n_tokens]; CACHED: ignored */
} pic_segment;

/* Link algorithms of P:166-170 and P:211-217 (SPEC grammar naive|fr|cacheblend:R|legolink:K),
 * plus LegoLink-0: Naive over chunks compiled with a dummy prefix (pic_compile_options);
 * PIC_E_VARIANT if any linked chunk was compiled without one. */
typedef enum { PIC_NAIVE = 0, PIC_FULL = 1, PIC_LEGOLINK = 2, PIC_CACHEBLEND = 3, PIC_LEGOLINK0 = 4 } pic_algorithm;

typedef struct {
  int32_t alg;               /* pic_algorithm */
  int32_t k;                 /* LegoLink: first k tokens of every chunk except an index-0 chunk (R6/R7) */
  int32_t r_percent;         /* CacheBlend: recompute ⌈R·N_cached/100⌉ cached tokens (R11) */
  int32_t check_layer;       /* CacheBlend: layer whose K/V deviation selects tokens (R9; default 1) */
  int32_t rebase;            /* 1 = RoPE re-base cached keys to their new positions (R1; default 1) */
  int32_t use_graph;         /* 1 = replay a CUDA graph per plan shape (default 1) */
  const int32_t* sel_override; /* CacheBlend test hook: sorted linked indices to keep after the check (nullable) */
  int32_t n_sel_override;
  float* debug_hidden;       /* test hook (nullable, host): [n_layers][R][d_model] fp32 with R = max(N of request 0,
                                Σ_requests k'); row r of layer l = residual after layer l of the r-th recomputed row
                                of the forward (request 0's selected rows in order, then request 1's, ...; rows
                                beyond that layer's count untouched).  Disables graphs. */
  int32_t kv_share;          /* 1 = shared-block link: a linked block whose 16 rows are all
                                unselected rows of one cached chunk, aligned to one of its store blocks, points
                                at that chunk-store block (reference counted) instead of a fresh copy; its keys
                                keep their compile positions and the attention kernels re-base them by the
                                block's Δ (R1) when they load the K tile, with the same arithmetic as the copy
                                (a2), so results are bit-identical to kv_share = 0.  Only blocks holding a
                                recomputed row, dynamic tokens or a chunk boundary are allocated and filled.
                                2 = V by reference only: the same blocks keep their V rows in the chunk-store
                                block (reference counted, read through a separate V block table) while their
                                keys are re-based by a2 into fresh blocks, so the attention reads K without
                                re-basing it; results are again bit-identical to kv_share = 0 (a2's keys, the
                                store's values).
                                3 = chunk-frame link: the kv_share 1 blocks are linked by reference and, in
                                addition, every other block inside a 16-aligned cached chunk (those holding
                                recomputed rows) keeps the chunk's compile frame: a2 copies its unselected
                                keys without rotation and a5 ropes its recomputed keys at position i − Δ_c,
                                so all of the chunk's keys sit at compile positions and carry Δ_c.  The
                                attention uses q·R(Δ)k = (R(−Δ)q)·k: when every 128-key tile lies in one
                                frame it re-bases Q once per frame (in TMEM) and feeds S = (R(−Δ)Q)·Kᵀ from
                                TMEM, else it re-bases the K tile as kv_share 1 does.  Equal to kv_share 0
                                within rounding (not bit-identical: the rotation moves from K to Q); exports
                                re-base keys to linked positions like kv_share 1.  bench.py's default.
                                Ignored for CacheBlend (its layer 0 rewrites every row).  Default 0 */
} pic_link_params;

/* Per-request result of a link. */
typedef struct {
  float* logits;             /* caller-owned host buffer [vocab] fp32 (nullable); first-token logits.
                              * Page-locked buffers (cudaHostAlloc / cudaHostRegister) are filled by direct
                              * device-to-host copies (one copy when the requests' buffers are consecutive rows
                              * of one array); pageable ones through the engine's staging buffer. */
  float* logits_dev;         /* caller-owned device buffer [vocab] fp32 (nullable); filled on `stream` */
  int32_t first_token;       /* argmax of the logits (ties -> lowest id, R20); -1 if no host output was requested */
  int32_t n_tokens;          /* N: linked prompt length */
  int32_t n_selected;        /* k': rows recomputed in the last layer */
  int32_t n_selected_layer0; /* rows recomputed in layer 0 (N for CacheBlend) */
  int32_t* selected;         /* caller-owned host buffer [N] (nullable): linked indices recomputed in the last
                                layer (CacheBlend: the device-side selection); forces a stream sync */
} pic_link_result;

typedef struct pic_engine pic_engine;
typedef struct pic_linked pic_linked;

/* Host-only: bytes of device arena pic_engine_create needs for (cfg, limits). */
pic_status pic_arena_bytes(const pic_model_config* cfg, const pic_engine_limits* limits, size_t* out_bytes);

/* Create an engine on CUDA `device` (or -1 = host-only planner engine; arena must then be NULL).
 * `arena` is a caller-owned device buffer of >= pic_arena_bytes() bytes, 256-B aligned, kept alive
 * until pic_engine_destroy (PyTorch owns the memory; the engine carves weights, KV pools and
 * workspaces from it).  Weights are generated on `stream`; the call returns after they are ready. */
pic_status pic_engine_create(const pic_model_config* cfg, const pic_engine_limits* limits, int32_t device,
                             void* arena, size_t arena_bytes, void* stream, pic_engine** out);
void pic_engine_destroy(pic_engine* eng);

/* Tensor parallelism (the Llama-3-70B shape): rank tp_rank of tp_size (1..8) owns q heads
 * [r·H_q/tp, ...), kv heads [r·H_kv/tp, ...) and MLP columns [r·F/tp, ...) of the GLOBAL model `cfg`
 * (weights are exact slices of the global generator); d_model, vocab, embeddings, norms and the LM head are
 * replicated.  After the O and down projections the ranks' partial sums are all-reduced by the residual
 * kernel itself, reading every rank's reduced partial directly from peer memory (CUDA IPC / NVLink) after
 * an epoch barrier — no separate collective call.  Every rank must issue the same sequence of compile /
 * link calls.  CacheBlend is single-rank only (PIC_E_VARIANT). */
pic_status pic_arena_bytes_tp(const pic_model_config* cfg, const pic_engine_limits* limits, int32_t tp_size,
                              size_t* out_bytes);
pic_status pic_engine_create_tp(const pic_model_config* cfg, const pic_engine_limits* limits, int32_t device,
                                void* arena, size_t arena_bytes, void* stream, int32_t tp_rank, int32_t tp_size,
                                pic_engine** out);
/* 64-byte CUDA IPC handle of this rank's arena (+ the arena's offset in that allocation). */
pic_status pic_tp_ipc_handle(pic_engine* eng, void* handle64, uint64_t* offset);
/* handles: tp_size x 64 bytes, offsets: tp_size (rank order, own entry ignored).  Must precede any compute. */
pic_status pic_tp_connect(pic_engine* eng, const void* handles, const uint64_t* offsets);

/* Compile step ("each chunk is encoded with position IDs starting from zero, and the LLM
 * performs only the prefill stage"; P:185 KVCompile).  chunks[i] is a host array of lens[i]
 * tokens.  All-or-nothing: on error no id is assigned and *err_index (nullable) names the failing
 * chunk.  out_ids: caller array [n].  Returns after the device work completed. */
pic_status pic_generate_context_cache(pic_engine* eng, const int32_t* const* chunks, const int32_t* lens,
                                      int32_t n, void* stream, pic_cache_id* out_ids, int32_t* err_index);

/* Compile variants.  dummy_prefix = m > 0 is the LegoLink-0 compile ("prepends four dummy tokens
 * (e.g., begin-of-sentence tokens) to each immutable chunk during compilation, then discards their
 * corresponding KV vectors"): the chunk is prefilled as dummy^m ‖ chunk at positions 0..m+n−1 and
 * only rows m..m+n−1 are stored (keys rotated at positions m.., so the chunk's compile base is c0 = m and
 * a link re-bases it by Δ = s_c − m, negative for a chunk placed first; reading R21).  dummy_token < 0
 * means cfg.bos_id.  m + n must fit max_pos and max_tokens. */
typedef struct {
  int32_t dummy_prefix;      /* m >= 0 (0 = the standard compile of pic_generate_context_cache) */
  int32_t dummy_token;       /* token id of the dummies (< 0: bos_id) */
} pic_compile_options;
pic_status pic_generate_context_cache_ex(pic_engine* eng, const int32_t* const* chunks, const int32_t* lens,
                                         int32_t n, const pic_compile_options* opts, void* stream,
                                         pic_cache_id* out_ids, int32_t* err_index);

/* Link step (P:162, P:185 KVLink, P:211-217 LegoLink; variants P:166-170).  Assembles the message
 * list, re-bases and gathers cached KV into fresh linked blocks, recomputes the selected rows layer
 * by layer (Eq. 1) and produces first-token logits.  out_linked (nullable): receives a handle
 * to the linked KV (caller releases it); NULL frees the linked blocks when the call's stream work is
 * done.  If result->logits is set the call synchronises `stream` before returning. */
pic_status pic_link(pic_engine* eng, const pic_segment* segs, int32_t n_segs, const pic_link_params* params,
                    void* stream, pic_linked** out_linked, pic_link_result* result);

/* Batched link of n_req independent requests in one forward (the data-parallel unit of cfg4:
 * rows of all requests are concatenated; weights are read once).  segs[r] / n_segs[r] per request;
 * out_linked (nullable) is an array [n_req]; results is an array [n_req].  CacheBlend and
 * debug hooks are single-request only (PIC_E_VARIANT). */
pic_status pic_link_batch(pic_engine* eng, int32_t n_req, const pic_segment* const* segs, const int32_t* n_segs,
                          const pic_link_params* params, void* stream, pic_linked** out_linked,
                          pic_link_result* results);

/* Host-only planner (step a1; P:211/P:213 selection).  Caller-allocated arrays,
 * each NULL or at least the stated size (cap = pic_plan_out.capacity >= N):
 *   sel[cap] sorted selected linked indices (pre-CacheBlend set; CacheBlend: dynamic ∪ {N-1});
 *   tok[cap] token ids; src[2*cap] (cache id low 31 bits, row) or (-1,-1) for dynamic rows;
 *   chunks[3*cap] (start, len, delta) per cached segment; block_table[cap] linked block ids that
 *   pic_link would use now (fresh blocks lowest-free-first; with kv_share, shared chunk-store blocks
 *   in place); slot[cap] slot of each selected row (block_table[i/16]*16 + i%16). */
typedef struct {
  int32_t capacity;
  int32_t n_tokens, n_sel, n_chunks, n_blocks;
  int32_t *sel, *tok, *src, *chunks, *block_table, *slot;
  int32_t* block_delta;      /* [cap] (nullable): per linked block, the Δ the attention applies to a shared
                                chunk-store block's keys (kv_share = 1), or the chunk frame of any block of an aligned
                                cached chunk (kv_share = 3), else 0 */
  int32_t n_shared;          /* out: blocks linked by reference (kv_share = 1); n_blocks - n_shared are fresh */
} pic_plan_out;
pic_status pic_plan(pic_engine* eng, const pic_segment* segs, int32_t n_segs, const pic_link_params* params,
                    pic_plan_out* out);

/* Copy layer `layer` of a linked KV cache to host: k_host, v_host are [N][H_kv][D] bf16 (uint16), or fp32 for a
 * PIC_DTYPE_FP32_DEBUG engine.  Keys of shared blocks (kv_share) are exported at their linked positions: the
 * device re-bases them (a2's kv_link kernel, this layer) into scratch pool blocks first, so the call needs one
 * free block per shared block with Δ != 0 (PIC_E_CAPACITY otherwise).  Synchronises the device. */
pic_status pic_linked_export(pic_engine* eng, const pic_linked* linked, int32_t layer, void* k_host, void* v_host);
/* Number of tokens N and the block table (int32[ceil(N/16)], nullable) of a linked cache. */
pic_status pic_linked_info(pic_engine* eng, const pic_linked* linked, int32_t* n_tokens, int32_t* block_table);
/* Shared-block link (kv_share): number of blocks of `linked` that are chunk-store blocks
 * linked by reference (kv_share 1 and 3: K and V; kv_share 2: V only), and per block (int32[ceil(N/16)],
 * nullable) the Δ the attention applies to its keys (0 for blocks the link owns and for kv_share 2;
 * kv_share 3: the chunk frame of every block of an aligned cached chunk).
 * Host-only bookkeeping. */
pic_status pic_linked_sharing(pic_engine* eng, const pic_linked* linked, int32_t* n_shared, int32_t* block_delta);
/* Re-base the shared chunk-store blocks (Δ != 0) of a kv_share linked cache into blocks it owns, on
 * `stream` (one a2 launch over their rows, all layers), dropping its references on them: later decode
 * steps then read keys at their linked positions instead of re-rotating them every step.  Results are
 * unchanged bit for bit.  PIC_E_CAPACITY if the pool lacks the blocks (the handle is unchanged). */
pic_status pic_linked_materialize(pic_engine* eng, pic_linked* linked, void* stream);
/* Release a linked cache: its own blocks return to the pool; shared chunk-store blocks drop one reference
 * (they stay with the chunk store, or return to the pool if their chunk was expired meanwhile). */
pic_status pic_linked_release(pic_engine* eng, pic_linked* linked);

/* Open-loop Poisson serving of link requests ("each user compiles all immutable
 * chunks in the test case once and then repeatedly sends the same request ... at a constant rate";
 * "we simulate request arrival times by sampling from a Poisson distribution").
 * Users u = 0..n_users-1 each resend their own message list as a Poisson process of rate rate/n_users
 * during [0, duration_s).  The server (this call, one host thread, wall clock) admits queued
 * requests FIFO into pic_link_batch calls of up to max_batch requests whose linked blocks fit the
 * free pool and whose recomputed rows fit max_rows (CacheBlend: one request per call, the engine's
 * limit); TTFT = first token on the host − arrival.  The chunks must already be compiled; the
 * context cache ratio (CCR) is reported as resident cache blocks / pool blocks at the start. */
typedef struct {
  int32_t n_users;
  const pic_segment* const* user_segs; /* [n_users] message lists */
  const int32_t* user_n_segs;          /* [n_users] */
  double rate;                         /* total arrival rate (requests / s) */
  double duration_s;                   /* arrival window */
  uint64_t seed;                       /* arrival-time generator (SplitMix64 counter stream) */
  int32_t max_batch;                   /* <= limits.max_requests */
  pic_link_params params;
} pic_serve_config;
typedef struct {
  int64_t n_requests, n_completed, n_batches;
  double elapsed_s;                    /* first arrival -> last completion */
  double throughput_rps;               /* n_completed / elapsed_s */
  double ttft_mean_ms, ttft_p50_ms, ttft_p90_ms, ttft_p99_ms, ttft_max_ms;
  double mean_batch;                   /* requests per link call */
  double ccr;                          /* context cache ratio at the start */
  double tokens_per_s;                 /* linked tokens completed / elapsed_s */
} pic_serve_stats;
pic_status pic_serve_poisson(pic_engine* eng, const pic_serve_config* cfg, void* stream, pic_serve_stats* out);
/* The arrival schedule pic_serve_poisson uses (host only): times (s, ascending) and users of every
 * request in [0, duration_s); *n_inout = capacity on input, count on output (PIC_E_CAPACITY if short). */
pic_status pic_serve_arrivals(int32_t n_users, double rate, double duration_s, uint64_t seed, double* times,
                              int32_t* users, int32_t* n_inout);

/* Decode over linked caches ("proceeds to the decode stage"): one step
 * for a batch of n live linked caches (distinct handles from pic_link(_batch) with out_linked).  Cache b
 * of current length N_b gets tokens[b] appended at position N_b: the model runs on that single row
 * (the same projections, RMSNorm/SwiGLU and sparse-query attention kernels as the link, at M = n),
 * attending to keys 0..N_b, its K/V is written into the cache (which grows to N_b + 1; a fresh block
 * is taken from the pool when N_b is a multiple of 16) and its next-token logits are produced.
 * Greedy decoding feeds results[b].next_token back as the next step's token.
 *   results: caller array [n]; per entry logits (host [vocab], nullable), logits_dev (device [vocab],
 *   nullable), next_token (argmax, ties -> lowest id; -1 unless a host output was requested or both
 *   logits pointers are NULL), n_tokens (length after the step).
 * Errors: PIC_E_CAPACITY (n > max_requests, N_b + 1 > max_pos / max_tokens, pool exhausted),
 * PIC_E_TOKEN, PIC_E_INVALID_ARG (NULL / repeated handle).  On error no cache changed. */
typedef struct {
  float* logits;
  float* logits_dev;
  int32_t next_token;
  int32_t n_tokens;
} pic_decode_result;
pic_status pic_decode(pic_engine* eng, pic_linked* const* linked, const int32_t* tokens, int32_t n, int32_t use_graph,
                      void* stream, pic_decode_result* results);

/* Copy layer `layer` of a compiled chunk to host: [n][H_kv][D] bf16 each (post-RoPE K at positions c0..c0+n-1;
 * c0 = 0, or the dummy-prefix length of a LegoLink-0 compile). */
pic_status pic_cache_export(pic_engine* eng, pic_cache_id id, int32_t layer, void* k_host, void* v_host);
/* Length and block list (int32[ceil(n/16)], nullable) of a compiled chunk. */
pic_status pic_cache_info(pic_engine* eng, pic_cache_id id, int32_t* n_tokens, int32_t* blocks);

/* Free a chunk's KV.  Idempotent: *was_present (nullable) says whether it existed
 * (S:203-211).  Live linked caches are unaffected: a copy-path link owns re-based copies, and a
 * shared-block link (kv_share) holds a reference on each chunk-store block it points at, so those
 * blocks return to the pool only when the last linked cache using them is released. */
pic_status pic_expire_cache(pic_engine* eng, pic_cache_id id, int32_t* was_present);

/* Test hook: copy generated bf16 weights to host (uint16 bf16 bits).  which: 0=q 1=k 2=v 3=o 4=gate
 * 5=up 6=down (rows of the logical [out][in] matrix row0..row0+nrows-1), 7=embed, 8=lm_head;
 * gains: 9=g1 10=g2 11=g_final as fp32 (nrows ignored, d_model floats). */
pic_status pic_read_weights(pic_engine* eng, int32_t which, int32_t layer, int64_t row0, int64_t nrows, void* host_out);

/* Free blocks in the KV pool and counters for tests/bench. */
typedef struct {
  int64_t free_blocks, total_blocks;
  int64_t n_cached_chunks;
  int64_t kernels_last_call;   /* kernels launched by the last link/compile call (incl. graph nodes) */
  int64_t graphs_cached;
  int64_t h2d_bytes_last_call; /* plan bytes copied host->device by the last compile/link forward */
  int64_t d2h_bytes_last_call; /* result bytes copied device->host by the last link */
} pic_stats;
pic_status pic_get_stats(pic_engine* eng, pic_stats* out);

/* Kernel profiling (bench/tests): when on, forwards run without graphs and every launch is bracketed
 * by CUDA events on its stream.  pic_get_profile synchronises those events and returns per-class
 * totals (launches, device ms, algorithmic bytes and FLOPs per SURVEY §8(d)); reset != 0 clears. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms, bytes, flops;
} pic_kernel_stat;
pic_status pic_set_profiling(pic_engine* eng, int32_t on);
pic_status pic_get_profile(pic_engine* eng, pic_kernel_stat* out, int32_t cap, int32_t* n, int32_t reset);

const char* pic_last_error(void);
const char* pic_status_string(pic_status s);

#ifdef __cplusplus
}
#endif
#endif /* PIC_H */
