// kernels.h — host launchers of the sm_100a kernels (internal to libpic.so, C++ linkage).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

namespace pic {

// PDL on by default; PIC_NO_PDL=1 disables (debugging).
bool pdl_enabled();

// Launch with the programmatic-stream-serialization attribute (works inside graph capture).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Set dynamic-smem attributes of every kernel instance (call once, outside graph capture).
cudaError_t prepare_kernels();

// ---- K15 weight generator, bit-exact with seedgen/ -------------------------
// dst[r][c] = bf16( bf16_rne(f(U(seed, tag, (row0 + r) * logical_cols + col0 + c))) * 2^exp2 ), r < rows,
// c < cols (logical_cols = 0 -> cols): row/column slices of the logical matrix (tensor-parallel shards).
cudaError_t launch_gen_matrix(void* dst_bf16, int64_t rows, int64_t cols, uint64_t seed, uint64_t tag, int exp2,
                              int64_t row0, cudaStream_t st, int64_t logical_cols = 0, int64_t col0 = 0);
// dst[i] = 1 + ((U(seed, tag, i) >> 61) - 4) / 32   (fp32)
cudaError_t launch_gen_gains(float* dst, int64_t n, uint64_t seed, uint64_t tag, cudaStream_t st);

// ---- a3: embed gather ----------------------------------------------------------------------
cudaError_t launch_embed(const void* E, const int32_t* tok, float* h, int M, int d, cudaStream_t st);

// ---- a4: residual add of split-K partials + RMSNorm ----------------------------------------
constexpr int kMaxSrcs = 16;
struct Srcs {  // fp32 [M][d] arrays summed into the residual (split-K partials or peer ranks' sums)
  const float* p[kMaxSrcs];
  int n;
};
struct Peers {  // per-rank device pointers (peer memory through CUDA IPC / NVLink)
  void* p[8];
};
cudaError_t launch_residual_rmsnorm_srcs(float* h, const Srcs& srcs, const float* g, void* x, const int32_t* out_map,
                                         int M, int d, float eps, cudaStream_t st, int f32 = 0);
// tensor parallel: reduce this rank's split-K partials; cross-rank epoch barrier over peer memory
cudaError_t launch_tp_reduce_local(const float* P, int splits, int M, int d, float* out, cudaStream_t st);
cudaError_t launch_tp_barrier(long long* counter, const Peers& flags, int rank, int tp, cudaStream_t st);
// h[r] += Σ_s P[s][r] (P nullable); if x: x[out_map ? out_map[r] : r] = bf16(rms(h[r]) ⊙ g) for out_map[r] >= 0
// f32 != 0: fp32 debug build (activations / KV stored fp32 instead of bf16)
cudaError_t launch_residual_rmsnorm(float* h, const float* P, int splits, const float* g, void* x,
                                    const int32_t* out_map, int M, int d, float eps, cudaStream_t st, int f32 = 0);

// ---- a5 epilogue: Σ partials, RoPE at row positions, Q dense, K/V scattered to the paged pool
cudaError_t launch_qkv_rope_scatter(const float* P, int splits, int P_rows, const int32_t* src_row,
                                    const int32_t* pos, const int32_t* slot, const float* cos_t, const float* sin_t,
                                    void* Q, void* Kpool_l, void* Vpool_l, int M, int Hq, int Hkv, int D,
                                    cudaStream_t st, int f32 = 0, int static_plan = 0,  // 1: pos/slot host-uploaded
                                    const int32_t* kpos = nullptr);  // K heads' RoPE positions (null: pos)

// ---- a8 epilogue: u = bf16(silu(Σ gate) ⊙ Σ up) ----------------------------------------------
cudaError_t launch_swiglu(const float* P, int splits, void* u, int M, int F, cudaStream_t st, int f32 = 0);

// ---- a2: KV link — gather cached rows into the linked blocks, RoPE re-base K by Δ -----------
// vcopy (nullable = all rows): per row, 1 = copy its V too, 0 = K only (V linked by reference);
// copy_k = 0: V only (materializing a V-by-reference block)
cudaError_t launch_kv_link(void* Kpool, void* Vpool, const int32_t* src_slot, const int32_t* dst_slot,
                           const int32_t* delta, int n_rows, int layer0, int n_layers, int64_t layer_stride_elems,
                           int Hkv, int D, const float* cos_t, const float* sin_t, int rebase, cudaStream_t st,
                           int f32 = 0, int max_ctas = 148 * 4,
                           const int32_t* vcopy = nullptr, int copy_k = 1);

// ---- GEMM (tcgen05): P[split][M][N] = A[M][K] · B[N][K]^T --------------------------------------
// pack > 0: B is stored pre-tiled [N/pack][K/64][pack][64] (every TMA box contiguous); the tensor map
// is then the 2-D view [rows][64] with a (64, pack) box.  pack = 0: row-major [N][K], box (64, bn).
extern unsigned long long* g_gemm_trace;  // bench-only GEMM timeline (gemm.cu)
// The GEMM launched after this one (same stream): this GEMM's producer prefetches the first `pfk`
// k-blocks of every unit of the next one into L2 once its own loads are issued.  pfk = 0: none.
struct GemmNext {
  const CUtensorMap* tm;
  int units, mt, splits, kper, kblk_total, bn, pfk;
};
GemmNext gemm_next(const CUtensorMap* B, int M, int N, int K, int splits, int bn, int pfk);
// Fused a5 epilogue (EPI_QKV): per output row its position and pool slot, the RoPE tables, the dense Q
// output [M][Hq][128] and this layer's K / V pools ([blocks][Hkv][16][128]).
struct GemmEpi {
  const int32_t* pos;
  const int32_t* slot;
  const float* cos_t;
  const float* sin_t;
  void* Q;
  void* Kl;
  void* Vl;
  int Hq, Hkv;
  // a4 fused across the GEMM boundary (unsplit GEMMs): the residual epilogue (EPI_RESID, norm_gain set)
  // also writes xg = bf16(h_new · g) [M][N] and per (row, n-tile) Σ h_new² into ssq [M][kSsqStride]; the
  // consuming GEMM's epilogue (EPI_QKV / EPI_SWIGLU, ssq_in set) scales its accumulator rows by
  // r = rsqrt(Σ_t ssq_in[row][t] / d + eps): x·W = r · (h·g)·W, so RMSNorm needs no kernel of its own.
  const float* norm_gain;
  void* xg;
  float* ssq;
  const float* ssq_in;
  int ssq_in_n;
  float inv_d, eps;
  // EPI_QKV: per row, the RoPE position of its K heads (null: pos) — chunk-frame blocks (kv_share 3)
  const int32_t* kpos;
  int raster_gm;  // m-tiles per raster group (0: the launcher chooses; see gemm.cu decode)
};
constexpr int kSsqStride = 32;  // max n-tiles per row of a fused-norm residual GEMM
// pair = 1: CTA-pair (cta_group::2) kernel with 256-row M-tiles; B's tensor map box must then be bn/2 rows
// (each CTA of the pair loads half of the N-tile); bn in gemm_pair_supported().
cudaError_t launch_gemm_partial(const CUtensorMap& A, const CUtensorMap& B, float* out, int M, int N, int K,
                                int splits, int bn, cudaStream_t st, int pack = 0, const GemmNext& nx = GemmNext{},
                                int pair = 0);
bool gemm_pair_supported(int bn);
// Split-K = 1 GEMMs with the consumer fused into the epilogue (tensor-bound shapes, no partials):
//   resid: h[M][N] += A·Bᵀ (a7 O projection / a8 down projection + residual add, fp32 h)
//   qkv:   A·W_qkvᵀ -> RoPE at pos -> Q dense, K/V -> pool slots (a5); bn = 128 or 256 (whole heads)
// pair = 1: CTA-pair kernel (256-row M-tiles; B's tensor map box must then be bn/2 rows)
cudaError_t launch_gemm_resid(const CUtensorMap& A, const CUtensorMap& B, float* h, int M, int N, int K, int bn,
                              cudaStream_t st, const GemmNext& nx = GemmNext{}, const GemmEpi& ep = GemmEpi{},
                              int pair = 0);
cudaError_t launch_gemm_qkv(const CUtensorMap& A, const CUtensorMap& B, const GemmEpi& ep, int M, int N, int K,
                            int bn, cudaStream_t st, const GemmNext& nx = GemmNext{}, int pair = 0);
bool gemm_resid_supported(int bn);
// Gate/up GEMM with the SwiGLU epilogue fused: B = interleaved [gate|up] groups of bn/2 rows (N2 = 2F rows),
// u[M][F] bf16 = silu(x·W_gᵀ) ⊙ (x·W_uᵀ).  Split-K 1.
cudaError_t launch_gemm_swiglu(const CUtensorMap& A, const CUtensorMap& B, void* u, int M, int N2, int K, int bn,
                               cudaStream_t st, int pack = 0, const GemmNext& nx = GemmNext{}, int pair = 0,
                               const GemmEpi& ep = GemmEpi{});
bool gemm_bn_supported(int bn, bool swiglu);

// ---- persistent GEMM chain (gemm_chain.cu): O-proj -> residual+RMSNorm -> gate/up+SwiGLU -> down ->
// residual+RMSNorm -> next QKV, phases separated by grid barriers, weights streamed across them.
enum { CHAIN_GEMM = 0, CHAIN_SWIGLU = 1, CHAIN_NORM = 2 };
constexpr int kMaxChainPhases = 6;
constexpr int kMaxChainMaps = 8;
struct ChainPhase {
  int type;               // CHAIN_*
  int bn, M, N, kblk, kper, splits;  // GEMM: tile N, rows, cols, K/64, k-blocks per split, splits. NORM: M rows, N = d,
                                     //   splits = partial count
  int a, b;               // GEMM: tensor-map indices of A [M][K] and B [N][K]
  void* out;              // GEMM: fp32 partials [splits][M][N]; SWIGLU: bf16 u [M][N/2]; NORM: bf16 x [M][d]
  const float* P;         // NORM: partials [splits][M][d] added to h
  const float* g;         // NORM: gain [d]
  float* h;               // NORM: fp32 residual [M][d]
  float eps;
};
struct ChainParams {
  int n_phases;
  ChainPhase ph[kMaxChainPhases];
  unsigned* bar;          // 2 zero-initialised counters (self-resetting)
  unsigned long long* trace;  // bench-only: per CTA 16 globaltimer stamps, or null
};
cudaError_t launch_gemm_chain(const CUtensorMap* const* maps, int n_maps, const ChainParams& cp, cudaStream_t st);
cudaError_t prepare_gemm_chain();
// Interleaved gate/up generator: physical row p = n·2g + j holds gate row n·g + j (j < g) or up row
// n·g + j − g (j >= g) of the logical [F][d] matrices (tags tag_gate / tag_up, same exponent).
cudaError_t launch_gen_gateup(void* dst_bf16, int64_t F, int64_t d, uint64_t seed, uint64_t tag_gate,
                              uint64_t tag_up, int exp2, int g, cudaStream_t st, int64_t f0 = 0);

// ---- a6: sparse-query causal attention (tcgen05, D = 128) + split-KV combine ----------------
struct AttnArgs {
  const int32_t* work;       // [n_work][4] (q-tile, kv-tile begin, kv-tile end, split slot): balanced split-KV
  const int32_t* tiles;      // [n_tiles][3] (seq, row_start, row_count)
  const int32_t* seq_bt_off; // per sequence: offset into bt
  const int32_t* bt;         // block tables
  const int32_t* row_pos;    // [M] absolute position of every query row
  int n_work, M, Hq, Hkv, layer, num_blocks;
  float scale_log2;
  float* o_part;             // [max splits][M][Hq][128]
  float* ml_part;            // [max splits][M][Hq][2]
  unsigned long long* trace; // bench-only per-CTA timeline (globaltimer ns, 8 slots per CTA) or null
  const void* Q;             // bf16 [M][Hq][128] queries
  int static_plan;           // 1: work/tiles/row_pos/bt were uploaded before the launch (read before PDL wait)
  const void* kpool;         // K/V pools (bf16 [L][NB][Hkv][16][128]) for the L2 prefetch; null: none
  const void* vpool;
  // Shared-block link: per block-table entry, the re-base Δ still to apply to that
  // block's keys (a chunk-store block linked by reference; 0 = a linked block already holding keys at
  // their linked positions).  Null: no entry is shared.  The kernel rotates such K tiles in shared
  // memory after TMA, with the a2 arithmetic (rebase_pair), before Q·Kᵀ.
  const int32_t* bdelta;
  const float* cos_t;        // [max_pos][64] fp32 RoPE table (re-base angles |Δ|·θ_j)
  const float* sin_t;
  // Rows of a q-tile the schedule did not split (row_nsplit[row] == 1) are normalised in the kernel and
  // written as bf16 to O [M][Hq][128] directly; split rows leave fp32 partials for attn_combine.
  const int32_t* row_nsplit;
  void* O;
  // ping-pong kernel: [next item, CTAs done], zero before the launch; the last CTA resets both
  unsigned* item_ctr;
  // V block table (nullable: V lives in the same blocks as K).  kv_share 2 links V by reference to the
  // chunk-store blocks while K is a re-based copy in fresh blocks.
  const int32_t* vbt;
  // 1: every K tile of every sequence has ONE block delta (kv_share 3 chunk frames): re-base by rotating
  // Q per frame (R(−Δ)·Q in TMEM, S as a TS MMA) instead of the K tiles (one-lane kernel)
  int qrot;
  int debug;  // bench-only ablation (PIC_ATTN_DEBUG), results invalid: 1 = softmax skipped, 2 = no K re-base
             // arithmetic, 3 = rotation warpgroup idle, 4 = as 2 without the proxy fence
};
// Balanced split-KV schedule: each q-tile t (KV extent n_kv[t] 128-key tiles) gets
// ceil(n_kv[t] / budget) splits, budget = ceil(Σ n_kv · Hkv / target_ctas); splits <= 32.
// Writes work items (tile, j0, j1, slot) and the per-row split count; returns the max splits.
int attn_schedule(const int32_t* tiles, int n_tiles, const int* n_kv, int Hkv, int target_ctas, int max_split,
                  int32_t* work_out /*[4 * cap]*/, int* n_work, int32_t* row_nsplit /*[M]*/);
// tmK/tmV: pool maps with a one-block box (64, 16, 1, 1); tmK8/tmV8: eight-block box (64, 16, 1, 8)
cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st);
// a6 v2 (attention_pp.cu): persistent ping-pong kernel, two q-tile lanes per CTA sharing the K/V stream.
// attn_schedule_pp writes items [n][8] = (tile, j0, j1, split slot) for lane A then lane B (tile -1: none);
// AttnArgs.work = items, AttnArgs.n_work = n; n * Hkv CTA items walked by min(n * Hkv, n_sms) CTAs.
int attn_schedule_pp(const int32_t* tiles, int n_tiles, const int* n_kv, int Hkv, int n_sms, int max_split,
                     std::vector<int32_t>& items, int32_t* row_nsplit);
cudaError_t launch_attention_pp(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                                cudaStream_t st);
// f1 (attention_decode.cu): split-KV decode attention, one query row per q-tile (tiles of row_count 1), the
// tile transposed (keys on the MMA rows, the G <= 8 heads of a kv-head on N = 16); same work list, partials
// and direct bf16 output convention as launch_attention_tc; no shared-block re-base (bdelta must be null)
cudaError_t launch_attention_decode(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmK8,
                                    const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st);
bool attention_decode_supported(int G);
// a6 for chunk-frame links (attention_qp.cu): the one-lane Q-side re-base kernel (attn_tc_kernel<G, true,
// true>) made persistent — min(n_work·Hkv, n_sms) CTAs walk the work list with every ring running across
// items; same arithmetic, bit for bit
cudaError_t launch_attention_qp(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                                cudaStream_t st);
cudaError_t launch_attn_combine(const float* o_part, const float* ml_part, const int32_t* row_nsplit, void* O, int M,
                                int Hq, int D, cudaStream_t st);
// generic-D SIMT attention (tiny shapes D in {16,32,64}; any D <= 128 in the fp32 debug build); writes O directly
// bdelta (nullable): per block-table entry, the re-base Δ to apply to that block's keys on load (f3 shared blocks)
cudaError_t launch_attention_simt(const void* Q, const void* Kpool_l, const void* Vpool_l, const int32_t* row_seq,
                                  const int32_t* seq_bt_off, const int32_t* bt, const int32_t* row_pos, void* O,
                                  int M, int Hq, int Hkv, int D, float scale, cudaStream_t st, int f32 = 0,
                                  const int32_t* bdelta = nullptr, const float* cos_t = nullptr,
                                  const float* sin_t = nullptr, const int32_t* vbt = nullptr);
// fp32 debug build GEMM (CUDA cores, exact products): P[M][N] = A[M][K] (fp32) · B[N][K]^T (bf16 weights)
cudaError_t launch_gemm_simt_f32(const float* A, const void* B, float* out, int M, int N, int K, cudaStream_t st);

// ---- a10: Σ LM-head partials, fp32 logits, argmax (ties -> lowest id) -----------------------
cudaError_t launch_logits_argmax(const float* P, int splits, float* logits, int32_t* argmax, int n_req, int V,
                                 cudaStream_t st);

// ---- a9: CacheBlend (check layer) -------------------------------------------------------------
// dev[i] = ||RoPE(Σk)_i − K_lnk[i]||² + ||Σv_i − V_lnk[i]||² for candidate rows (cand[i] != 0), else −1
cudaError_t launch_cb_deviation(const float* P, int splits, const int32_t* cand, const int32_t* slot,
                                const float* cos_t, const float* sin_t, const void* Kpool_l, const void* Vpool_l,
                                float* dev, int N, int Hq, int Hkv, int D, cudaStream_t st, int f32 = 0);
// keep[i] = cand[i] && rank_i < T, rank by (dev desc, index asc)
cudaError_t launch_cb_rank(const float* dev, int32_t* keep, int N, int T, cudaStream_t st);
// sel = sorted {i : keep[i] || forced[i]}; pos = sel; slot = bt[sel/16]*16 + sel%16; writes count
cudaError_t launch_cb_compact(const int32_t* keep, const int32_t* forced, const int32_t* bt, int32_t* sel,
                              int32_t* pos, int32_t* slot, int32_t* count, int N, cudaStream_t st);
// dst[r] = src[idx[r]] rows of d floats
cudaError_t launch_gather_rows(const float* src, const int32_t* idx, float* dst, int M, int d, cudaStream_t st);

}  // namespace pic
