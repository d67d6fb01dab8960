// attention.cu — a6: sparse-query causal attention over the paged linked cache.
//
// Eq. (1) of the paper: A = softmax(Q K_expᵀ · MASK), O = A V_exp, where only the k'
// selected rows have queries ("allowing the k' tokens to attend to all N tokens") and MASK
// makes row i see keys 0..p_i ("attend to only tokens before them"; reading R3: additive −∞,
// scale 1/√D).  Query rows are scattered over the context, so every row carries its own causal
// limit p_i.
//
// sm_100a design (D = 128):
//   * GQA packing: one CTA = one kv-head g and 128/G consecutive selected rows of one sequence;
//     its 128 MMA rows are (query, head-in-group) pairs, so K/V tiles are loaded once per group.
//   * Q tile and 128-key K/V tiles are staged by TMA (SWIZZLE_128B).  A K/V tile is 8 paged blocks
//     of 16 tokens, addressed through the sequence's block table: 16 TMA boxes per tile.
//   * S = Q·Kᵀ and O_tile = P·V run on tcgen05 with fp32 accumulators in TMEM
//     (cols [0,256): S double buffer, [256,512): O_tile double buffer).  V is the MN-major B operand.
//   * Softmax: 4 warps, one query row per thread (tcgen05.ld 32x32b gives a thread its row), exp2
//     with running max/sum in fp32, P written as bf16 into a SWIZZLE_128B smem tile.  O is
//     accumulated and rescaled in registers (online softmax).
//   * Split-KV over blockIdx.z for load balance; (m, l, O) partials merged by attn_combine, whose
//     cross-split max/sum is a warp-shuffle reduction.
#include <cuda.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

namespace pic {

namespace attn {
constexpr int kTile = 16384;                  // one [128 rows][64 cols] bf16 SW128 half tile
constexpr int kStages = 3;                    // K and V ring depth
constexpr int kK = 0;                         // K stages: kStages x 2 halves
constexpr int kV = kK + kStages * 2 * kTile;  // V stages
constexpr int kQ = kV + kStages * 2 * kTile;  // Q tile (2 halves), TMA-staged (A operand of S = Q·Kᵀ)
constexpr int kX = kQ + 2 * kTile;            // softmax pair exchange: [2 parity][2 halves][128] fp32
constexpr int kBar = kX + 2 * 2 * 128 * 4;    // barriers
constexpr int kNumBars = 1 + 5 * kStages + 6 + 4;  // + k_rot ring (shared-block link), qd_full/qd_empty (QROT)
constexpr int kSmem = kBar + kNumBars * 8 + 16;
static_assert(kSmem <= 232448, "attention smem over the 227 KB limit");
// TMEM columns (512 allocated)
constexpr uint32_t kTmS = 0;    // S double buffer [0, 256); P(t) (bf16 pairs) overwrites S(t): half hc at +64·hc
constexpr uint32_t kTmO = 256;  // O accumulator [256, 384)
constexpr uint32_t kTmQd = 384;  // QROT in TMEM (PIC_QROT_SMEM=0): two R(−Δ)·Q buffers (bf16 pairs) [384, 512)
// QROT in shared memory (default): the two R(−Δ)·Q buffers take V slot 2 and the Q tile ([kV + 2 slots, kX)),
// so the QROT kernel runs a 2-slot V ring; S = Q_Δ·Kᵀ stays an SS MMA.
constexpr int kQd = kV + 2 * 2 * kTile;
static_assert(kQd + 2 * 2 * kTile == kX, "QROT smem buffers must end where the Q tile ends");
}  // namespace attn
#ifndef PIC_QROT_SM_KS
#define PIC_QROT_SM_KS 3  // QROT_SM K ring depth (V ring: 5 - KS)
#endif
#ifndef PIC_QROT_SMEM
#define PIC_QROT_SMEM 0  // smem variant (2-slot V ring) measured equal at cfg4: 178-180 vs 177-178 ms per step
#endif

// Q is TMA-staged into shared memory once per CTA (the A operand of S = Q·Kᵀ); P is the TMEM A operand
// of O += P·V.  (A TMEM-resident Q cost a 1.8 µs tcgen05.st + wait::st in every CTA's prologue.)
// ROT: kRotWarps extra warps re-base shared-block K tiles (f3), one per SMSP.  Measured (cfg4 attention,
// 32 layers): 4 warps 26.3 ms, 2 warps 41.5 ms (the rotation is issue-bound and sits between the K TMA
// and the S MMA); 4 warps cap the CTA at 128 registers per thread (14 warps), a few bytes of spill.
constexpr int kRotWarps = 4;
#ifndef PIC_QROT_WARPS
#define PIC_QROT_WARPS 4
#endif
// QROT with R(−Δ)·Q in smem: the frame rotation has no TMEM lane-quarter constraint, so it may run on
// fewer warps (1, 2 or 4; a frame changes every ~4 K tiles)
constexpr int kQrotWarpsSm = PIC_QROT_WARPS;
static_assert(kQrotWarpsSm == 1 || kQrotWarpsSm == 2 || kQrotWarpsSm == 4, "PIC_QROT_WARPS: 1, 2 or 4");
template <bool ROT, bool QROT>
constexpr int attn_threads() {
  return !ROT ? 320 : (QROT && PIC_QROT_SMEM) ? 320 + 32 * kQrotWarpsSm : 320 + 32 * kRotWarps;
}
#ifndef PIC_V1_POLY8
#define PIC_V1_POLY8 1  // pairs of every 8 whose exponential runs on the FMA-pipe polynomial (exp2_poly2)
#endif
// QROT (kv_share 3 links whose every K tile holds one chunk frame): instead of rotating K tiles in smem,
// the rotation warps write R(−Δ)·Q for each frame into TMEM and S = Q_Δ·Kᵀ runs as a TS MMA
// (q·R(Δ)k = (R(−Δ)q)·k) — one rotation of the 128-row Q tile per chunk instead of one per K tile.
template <int G, bool ROT, bool QROT = false>
__global__ void __launch_bounds__(attn_threads<ROT, QROT>(), 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV,
                   const __grid_constant__ CUtensorMap tmK8, const __grid_constant__ CUtensorMap tmV8, const AttnArgs a) {
  griddep_launch();
  using namespace attn;
  constexpr int S = kStages;
  // QROT_SM: R(−Δ)·Q lives in smem (SS MMA for S) in place of V slot 2 and the Q tile
  constexpr bool QROT_SM = QROT && PIC_QROT_SMEM;
  // ring depths: QROT_SM gives up one 32 KB slot (K or V, PIC_QROT_SM_KS) for the second R(−Δ)·Q buffer
  constexpr int SK = QROT_SM ? PIC_QROT_SM_KS : S;  // K ring depth
  constexpr int SV = QROT_SM ? 5 - PIC_QROT_SM_KS : S;  // V ring depth
  constexpr int kVb = kK + SK * 2 * kTile;  // V ring base
  unsigned long long* const tr = a.trace ? a.trace + 32 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  const uint32_t base = smem_u32(smem);
  const uint32_t q_full = smem_u32(bars + 0);
  const uint32_t k_full = smem_u32(bars + 1), k_empty = smem_u32(bars + 1 + S);
  const uint32_t v_full = smem_u32(bars + 1 + 2 * S), v_empty = smem_u32(bars + 1 + 3 * S);
  const uint32_t s_full = smem_u32(bars + 1 + 4 * S), p_full = smem_u32(bars + 3 + 4 * S);
  const uint32_t o_full = smem_u32(bars + 5 + 4 * S);
  const uint32_t k_rot = smem_u32(bars + 7 + 4 * S);  // ROT: K tile re-based in smem (4 rotation warps)
  const uint32_t qd_full = smem_u32(bars + 7 + 5 * S), qd_empty = smem_u32(bars + 9 + 5 * S);  // QROT

  const int warp = warp_id(), lane = lane_id();
  // barriers and TMEM do not depend on upstream data: set them up while the previous kernel drains
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < S; ++s) {
      mbar_init(k_full + 8 * s, 1);
      mbar_init(k_empty + 8 * s, 1);
      mbar_init(v_full + 8 * s, 1);
      mbar_init(v_empty + 8 * s, 1);
      mbar_init(k_rot + 8 * s, kRotWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(qd_full + 8 * b, (QROT && PIC_QROT_SMEM) ? kQrotWarpsSm : kRotWarps);
      mbar_init(qd_empty + 8 * b, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + 8 * b, 1);
      mbar_init(p_full + 8 * b, 256);
      mbar_init(o_full + 8 * b, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Host-uploaded plans (work list, tiles, positions, block tables) are complete before the graph
  // starts; device-side ones (CacheBlend's re-selected rows) come from upstream kernels.
  if (!a.static_plan) griddep_wait();
  if (tr && threadIdx.x == 0 && !a.static_plan) tr[1] = globaltimer();
  // work item (host-balanced split-KV schedule): q-tile, KV-tile range [j0, j1), split slot
  const int* wk = a.work + 4 * blockIdx.x;
  const int tile = wk[0], split = wk[3], g = blockIdx.y;
  const int seq = a.tiles[3 * tile], row_start = a.tiles[3 * tile + 1], row_count = a.tiles[3 * tile + 2];

  // causal extent of this tile: keys 0..max_p (rows are sorted, but take the max anyway)
  int max_p = 0;
  for (int i = lane; i < row_count; i += 32) max_p = max(max_p, a.row_pos[row_start + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) max_p = max(max_p, __shfl_xor_sync(0xffffffffu, max_p, o));
  const int n_kv = max_p / 128 + 1;
  const int j0 = wk[1], j1 = min(n_kv, wk[2]);  // positions may be device-side (CacheBlend): clamp
  const int n = max(0, j1 - j0);
  const int* bt = a.bt + a.seq_bt_off[seq];
  const int last_blk = max_p / 16;
  // L2 prefetch of this CTA's K/V pages (a hint, so it may run before the upstream kernel that
  // writes the recomputed rows has finished: L2 is the coherence point)
  if (warp == 0 && a.kpool) {  // one paged block per lane and round: the block-id loads run in parallel
    for (int i = lane; i < n * 8; i += 32) {
      const int blk = bt[min(j0 * 8 + i, last_blk)];
      const size_t off = (((size_t)a.layer * a.num_blocks + blk) * a.Hkv + g) * (16 * 128 * 2);
      bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(a.kpool) + off, 16 * 128 * 2);
      bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(a.vpool) + off, 16 * 128 * 2);
    }
  }
  if (a.static_plan) griddep_wait();  // Q and the recomputed rows' K/V come from the upstream kernel
  if (tr && threadIdx.x == 0 && a.static_plan) tr[1] = globaltimer();

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (K, V)
    if (n > 0) {
      if (lane == 0) {
        // Q first: 128 MMA rows = (128/G queries) x (G heads of kv-head g), one 3-D box per 64-dim half
        // (QROT_SM: the rotation warps build every frame's R(−Δ)·Q straight from global Q instead)
        if (!QROT_SM) {
          mbar_expect_tx(q_full, 2 * kTile);
          for (int h = 0; h < 2; ++h) tma_load_3d(base + kQ + h * kTile, &tmQ, q_full, h * 64, g * G, row_start);
        }
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        tma_prefetch(&tmK8);
        tma_prefetch(&tmV8);
      }
      const int kv_base = a.layer * a.num_blocks;
      // the 8 paged-block ids of a 128-key tile: one coalesced load by lanes 0-7, one tile ahead; V's
      // own table when V is linked by reference (kv_share 2)
      const int* vbt = a.vbt ? a.vbt + a.seq_bt_off[seq] : bt;
      int blk_next = lane < 8 ? bt[min(j0 * 8 + lane, last_blk)] : 0;
      int vblk_next = lane < 8 ? vbt[min(j0 * 8 + lane, last_blk)] : 0;
      // V(t) is issued after K(t+1): the MMA warp consumes S(t+1) before PV(t), and a V slot still held by
      // PV(t-SV) must not hold back the next K tile (measured with the 2-slot V ring of QROT_SM)
      auto load_v = [&](int u, int vb0, const int* vb, bool vc) {
        const int vs = u % SV;
        mbar_wait(v_empty + 8 * vs, ((u / SV) & 1) ^ 1);
        mbar_expect_tx(v_full + 8 * vs, 2 * kTile);
        if (vc) {
          for (int h = 0; h < 2; ++h)
            tma_load_4d(base + kVb + (2 * vs + h) * kTile, &tmV8, v_full + 8 * vs, h * 64, 0, g, kv_base + vb0);
        } else {
#pragma unroll
          for (int b = 0; b < 8; ++b)
            for (int h = 0; h < 2; ++h)
              tma_load_4d(base + kVb + (2 * vs + h) * kTile + b * 2048, &tmV, v_full + 8 * vs, h * 64, 0, g,
                          kv_base + vb[b]);
        }
      };
      int vprev[8];
      bool vcprev = false;
      for (int t = 0; t < n; ++t) {
        const int s = t % SK;
        const uint32_t ph = (t / SK) & 1;
        const int blk_mine = blk_next, vblk_mine = vblk_next;
        if (t + 1 < n && lane < 8) {
          blk_next = bt[min((j0 + t + 1) * 8 + lane, last_blk)];
          vblk_next = vbt[min((j0 + t + 1) * 8 + lane, last_blk)];
        }
        int blk[8], vblk[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          blk[b] = __shfl_sync(0xffffffffu, blk_mine, b);
          vblk[b] = __shfl_sync(0xffffffffu, vblk_mine, b);
        }
        // 8 consecutive block ids: one 8-block box per half instead of 8 one-block boxes
        const bool contig = __all_sync(0xffffffffu, lane >= 8 || blk_mine == blk[0] + lane);
        const bool vcontig = __all_sync(0xffffffffu, lane >= 8 || vblk_mine == vblk[0] + lane);
        if (lane == 0) {
          mbar_wait(k_empty + 8 * s, ph ^ 1);
          mbar_expect_tx(k_full + 8 * s, 2 * kTile);
          if (contig) {
            for (int h = 0; h < 2; ++h)
              tma_load_4d(base + kK + (2 * s + h) * kTile, &tmK8, k_full + 8 * s, h * 64, 0, g, kv_base + blk[0]);
          } else {
#pragma unroll
            for (int b = 0; b < 8; ++b)
              for (int h = 0; h < 2; ++h)
                tma_load_4d(base + kK + (2 * s + h) * kTile + b * 2048, &tmK, k_full + 8 * s, h * 64, 0, g,
                            kv_base + blk[b]);
          }
          if (t > 0) load_v(t - 1, vprev[0], vprev, vcprev);
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) vprev[b] = vblk[b];
        vcprev = vcontig;
        __syncwarp();
      }
      if (lane == 0) load_v(n - 1, vprev[0], vprev, vcprev);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (convergent: descriptors and loop state stay uniform) and elect.sync
    // issues; a lane-0 branch with per-MMA descriptor arithmetic capped issue at ~88 cycles per MMA, above
    // the 64-cycle M=128 N=128 K=16 pipe time (scripts/probe_tc.cu).
    if (n > 0) {
      constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // Q (smem, K-major) x K (smem, K-major)
      constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (TMEM, K-major) x V (smem, MN-major)
      const uint64_t dQ = sdesc_sw128(base + kQ, 16, 1024), dK0 = sdesc_sw128(base + kK, 16, 1024);
      const uint64_t dV0 = sdesc_sw128(base + kVb, kTile, 1024);
      const uint64_t dQd = sdesc_sw128(base + kQd, 16, 1024);  // QROT_SM: R(−Δ)·Q buffer 0 (buffer 1: +32 KB)
      unsigned long long w_k = 0, w_p = 0, w_v = 0, w_q = 0, q0 = 0, sum_w = 0;
      if (!QROT_SM) mbar_wait(q_full, 0);
      tc_fence_after();
      if (tr && lane == 0) tr[2] = globaltimer();
      auto issue_pv = [&](int u) {
        const int pb = u & 1, vs = u % SV;
        if (tr) q0 = globaltimer();
        mbar_wait(p_full + 8 * pb, (u >> 1) & 1);
        if (tr) {
#ifdef PIC_ATTN_PHASES
          if (u <= n - 3) sum_w += clock64();  // P(u) seen by the MMA warp (paired with S(u+2) ready)
#endif
          const unsigned long long q1 = globaltimer();
          w_p += q1 - q0;
          q0 = q1;
        }
        mbar_wait(v_full + 8 * vs, (u / SV) & 1);
        if (tr) w_v += globaltimer() - q0;
        tc_fence_after();
        const uint64_t dv = dV0 + (uint64_t)(vs * (2 * kTile / 16));
        // keys 16kk..16kk+15: P half kk/4 at S-buffer column 64·(kk/4) + 8·(kk%4); O accumulates in TMEM
        // across KV tiles (rescaled by the softmax warps when needed).  One elect.sync for the 8 MMAs: the
        // tensor pipe idles until P(u) lands, so issue latency adds straight to the softmax's wait for S.
#ifdef PIC_ATTN_PER_MMA_ISSUE  // A/B builds only: one elect.sync + 64-bit descriptor arithmetic per MMA
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts_e(tmem + kTmO, tmem + kTmS + pb * 128 + (kk >> 2) * 64 + (kk & 3) * 8,
                         dv + (uint64_t)(kk * 2048 / 16), idO, (u | kk) != 0);
#else
        umma_ts_k128(tmem + kTmO, tmem + kTmS + pb * 128, dv, idO, u != 0);
#endif
        umma_commit_e(o_full + 8 * pb);
        umma_commit_e(v_empty + 8 * vs);
      };
      // QROT: the frame (Δ) of each K tile (uniform over its 8 blocks, host-checked) and the R(−Δ)·Q buffer
      const int* bdq = QROT ? a.bdelta + a.seq_bt_off[seq] : nullptr;
      int fi = -1, fr_cur = 0;
      int fr_next = QROT ? bdq[min(j0 * 8, last_blk)] : 0;
      for (int t = 0; t < n; ++t) {
        const int sb = t & 1, ks = t % SK;
        int qb = 0;
        bool frame_end = false;
        if constexpr (QROT) {
          const int fr = fr_next;
          fr_next = t + 1 < n ? bdq[min((j0 + t + 1) * 8, last_blk)] : fr;
          if (t == 0 || fr != fr_cur) {  // a new frame: wait for its rotated Q
            ++fi;
            if (tr) q0 = globaltimer();
            mbar_wait(qd_full + 8 * (fi & 1), (fi >> 1) & 1);
            if (tr) w_q += globaltimer() - q0;
          }
          fr_cur = fr;
          qb = fi & 1;
          frame_end = t + 1 == n || fr_next != fr;
        }
        if (tr) q0 = globaltimer();
        mbar_wait((ROT && !QROT ? k_rot : k_full) + 8 * ks, (t / SK) & 1);
        if (tr) w_k += globaltimer() - q0;
        tc_fence_after();
        // S(t) overwrites the buffer holding P(t-2): PV(t-2) was issued before and MMAs run in order
        const uint64_t dk = dK0 + (uint64_t)(ks * (2 * kTile / 16));
#ifdef PIC_ATTN_PER_MMA_ISSUE
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t o = (uint64_t)(((kk >> 2) * kTile + (kk & 3) * 32) >> 4);
          if constexpr (QROT && !QROT_SM)
            umma_bf16_ts_e(tmem + kTmS + sb * 128, tmem + kTmQd + qb * 64 + kk * 8, dk + o, idS, kk > 0);
          else
            umma_bf16_e(tmem + kTmS + sb * 128, (QROT_SM ? dQd + (uint64_t)(qb * (2 * kTile / 16)) : dQ) + o, dk + o,
                        idS, kk > 0);
        }
#else
        if constexpr (QROT_SM)  // A = R(−Δ)·Q buffer qb in smem
          umma_ss_k128(tmem + kTmS + sb * 128, dQd + (uint64_t)(qb * (2 * kTile / 16)), dk, idS, 0, kTile);
        else if constexpr (QROT)  // A = R(−Δ)·Q from TMEM: dims 16kk..16kk+15 at columns 8kk..8kk+7
          umma_tsk_k128(tmem + kTmS + sb * 128, tmem + kTmQd + qb * 64, dk, idS, kTile);
        else
          umma_ss_k128(tmem + kTmS + sb * 128, dQ, dk, idS, 0, kTile);
#endif
        umma_commit_e(s_full + 8 * sb);
        umma_commit_e(k_empty + 8 * ks);
        if (QROT && frame_end) umma_commit_e(qd_empty + 8 * qb);  // this frame's Q buffer may be rewritten
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n - 1);
      if (tr && lane == 0) {
        tr[11] = w_k;
        tr[12] = w_p;
        tr[13] = w_v;
        tr[14] = w_q;
        tr[15] = (unsigned long long)(fi + 1);
        tr[25] = sum_w;
      }
    }
  } else if (QROT_SM && warp >= 10) {
    // ------------------------------------------------------------------ Q re-base per chunk frame (smem)
    // For every frame Δ met along the KV range (in tile order), build R(−Δ)·q for the tile's 128 MMA rows
    // (row r = (query r / G, head g·G + r % G); NeoX pairs (j, j+64), fp32 rotation of the bf16 q rounded to
    // bf16, as the TMEM variant) straight from global Q into the smem buffer of that frame's parity, in the
    // SWIZZLE_128B K-major layout the TMA would give (rows past the tile are zero).  Thread u owns the
    // 16-B chunk cc = u & 7 (dims 8cc..8cc+7 and their partners 64+8cc..) of rows rg + RS·i, rg = u >> 3,
    // RS = 4·kQrotWarpsSm; each warp-wide load covers 4 rows x 128 contiguous bytes.
    if (n > 0) {
      constexpr int RS = 4 * kQrotWarpsSm, NR = 128 / RS;  // row stride, rows per thread
      const int u = threadIdx.x - 320;
      const int cc = u & 7, rg = u >> 3;
      const int* bdq = a.bdelta + a.seq_bt_off[seq];
      const uint16_t* Qg = reinterpret_cast<const uint16_t*>(a.Q);
      int fi = -1, fr_cur = 0;
      for (int t = 0; t < n; ++t) {
        const int fr = bdq[min((j0 + t) * 8, last_blk)];
        if (t > 0 && fr == fr_cur) continue;
        fr_cur = fr;
        ++fi;
        const int ad = fr < 0 ? -fr : fr;
        const float sg = fr < 0 ? 1.f : -1.f;  // R(−Δ): sin(−Δθ) = −sign(Δ)·sin(|Δ|θ)
        const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + cc * 8);
        const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + cc * 8);
        const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
        const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const float sn[8] = {sg * s0.x, sg * s0.y, sg * s0.z, sg * s0.w, sg * s1.x, sg * s1.y, sg * s1.z, sg * s1.w};
        const uint32_t qb = base + kQd + (fi & 1) * (2 * kTile);
#pragma unroll 1
        for (int i0 = 0; i0 < NR; i0 += 4) {
          uint4 xa[4], xb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = rg + RS * (i0 + i), qi = r / G;
            if (qi < row_count) {
              const uint4* src = reinterpret_cast<const uint4*>(
                  Qg + ((size_t)(row_start + qi) * a.Hq + g * G + r % G) * 128 + cc * 8);
              xa[i] = __ldg(src);
              xb[i] = __ldg(src + 8);
            } else {
              xa[i] = make_uint4(0u, 0u, 0u, 0u);
              xb[i] = xa[i];
            }
          }
          // the first rows' loads are in flight: wait until the MMAs of frame fi−2 are done with the buffer
          if (i0 == 0) mbar_wait(qd_empty + 8 * (fi & 1), ((fi >> 1) & 1) ^ 1);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (fr != 0) {
              uint32_t a4[4] = {xa[i].x, xa[i].y, xa[i].z, xa[i].w}, b4[4] = {xb[i].x, xb[i].y, xb[i].z, xb[i].w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float a0 = __uint_as_float(a4[k] << 16), a1 = __uint_as_float(a4[k] & 0xFFFF0000u);
                const float b0 = __uint_as_float(b4[k] << 16), b1 = __uint_as_float(b4[k] & 0xFFFF0000u);
                float ra0, rb0, ra1, rb1;
                rebase_pair(a0, b0, cs[2 * k], sn[2 * k], ra0, rb0);
                rebase_pair(a1, b1, cs[2 * k + 1], sn[2 * k + 1], ra1, rb1);
                a4[k] = pack_bf16(ra0, ra1);
                b4[k] = pack_bf16(rb0, rb1);
              }
              xa[i] = make_uint4(a4[0], a4[1], a4[2], a4[3]);
              xb[i] = make_uint4(b4[0], b4[1], b4[2], b4[3]);
            }
            const int r = rg + RS * (i0 + i);
            const uint32_t o = (uint32_t)(r * 128 + ((cc ^ (r & 7)) << 4));  // SW128: chunk cc of row r
            sts128(qb + o, xa[i]);
            sts128(qb + kTile + o, xb[i]);
          }
        }
        fence_async_smem();  // generic-proxy smem writes -> visible to the tcgen05.mma operand reads
        __syncwarp();
        if (lane == 0) mbar_arrive(qd_full + 8 * (fi & 1));
      }
    }
  } else if (QROT && warp >= 10) {
    // ------------------------------------------------------------------ Q re-base per chunk frame
    // Row r of the MMA (query, head) = TMEM lane r = Q smem row r; this warp owns lanes 32·(warp % 4)...
    // For every frame Δ met along the KV range (in tile order), write R(−Δ)·q (NeoX pairs (j, j+64),
    // fp32 rotation of the bf16 q, rounded to bf16) into the Q buffer of that frame's parity.
    if (n > 0) {
      const int qq = warp & 3;
      const int r = qq * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(qq * 32) << 16;
      const int* bdq = a.bdelta + a.seq_bt_off[seq];
      mbar_wait(q_full, 0);
      int fi = -1, fr_cur = 0;
      for (int t = 0; t < n; ++t) {
        const int fr = bdq[min((j0 + t) * 8, last_blk)];
        if (t > 0 && fr == fr_cur) continue;
        fr_cur = fr;
        ++fi;
        mbar_wait(qd_empty + 8 * (fi & 1), ((fi >> 1) & 1) ^ 1);  // the MMAs of frame fi−2 are done
        const int ad = fr < 0 ? -fr : fr;
        const float sg = fr < 0 ? 1.f : -1.f;  // R(−Δ): sin(−Δθ) = −sign(Δ)·sin(|Δ|θ)
        const uint32_t qbase = tmem + lane_addr + kTmQd + (fi & 1) * 64;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {  // dims 32hh..32hh+31 and their partners 64+32hh..
          uint32_t oa[16], ob[16];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = 4 * hh + cc;  // 16-B chunk: dims 8c..8c+7 (half 0) and 64+8c.. (half 1)
            const uint32_t off = (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4));
            const uint4 xa = lds128(base + kQ + off), xb = lds128(base + kQ + kTile + off);
            const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + c * 8);
            const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + c * 8);
            const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
            const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            const uint32_t a4[4] = {xa.x, xa.y, xa.z, xa.w}, b4[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a0 = __uint_as_float(a4[k] << 16), a1 = __uint_as_float(a4[k] & 0xFFFF0000u);
              const float b0 = __uint_as_float(b4[k] << 16), b1 = __uint_as_float(b4[k] & 0xFFFF0000u);
              float ra0, rb0, ra1, rb1;
              rebase_pair(a0, b0, cs[2 * k], sg * sn[2 * k], ra0, rb0);
              rebase_pair(a1, b1, cs[2 * k + 1], sg * sn[2 * k + 1], ra1, rb1);
              oa[cc * 4 + k] = pack_bf16(ra0, ra1);
              ob[cc * 4 + k] = pack_bf16(rb0, rb1);
            }
          }
          // columns: dims (2k, 2k+1) at column k -> dims 32hh.. at 16hh.., partners at 32 + 16hh..
          tmem_st16u_wait(qbase + 16 * hh, oa);
          tmem_st16u_wait(qbase + 32 + 16 * hh, ob);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(qd_full + 8 * (fi & 1));
      }
    }
  } else if (ROT && warp >= 10) {
    // ------------------------------------------------------------------ K-tile re-base (f3)
    // Keys of a chunk-store block linked by reference still sit at their compile positions: rotate
    // every NeoX pair (j, j+64) of such rows by Δ of its block (the a2 arithmetic, rebase_pair, so the
    // tile equals the one a copied-and-re-based linked block would give).  In the SWIZZLE_128B tile
    // dims j and j+64 sit at the same offset of the two 64-column halves.  Thread u owns logical
    // 16-B chunk cc = u & 7 (dims 8cc..8cc+7) of rows rg + 8i (rg = u >> 3, i < 16/(4·kRotWarps)) of each
    // of the 8 paged blocks (rows rg and rg + 8 share the swizzle phase).
    constexpr int RPB = 16 / (4 * kRotWarps);  // rows per block per thread
    const int u = threadIdx.x - 320;
    const int cc = u & 7, rg = u >> 3;
    const uint32_t phys = (uint32_t)(((cc ^ (rg & 7)) << 4) + rg * 128);
    const int* bd = a.bdelta + a.seq_bt_off[seq];
    int dcache = 0;
    float2 cs[4], sn[4], ns[4];  // cos, sin, −sin of dims (8cc + 2k, 8cc + 2k + 1) for Δ = dcache
    auto load_angles = [&](int d) {
      const int ad = d < 0 ? -d : d;
      const float sg = d < 0 ? -1.f : 1.f;
      const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + cc * 8);
      const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + cc * 8);
      const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
      cs[0] = make_float2(c0.x, c0.y); cs[1] = make_float2(c0.z, c0.w);
      cs[2] = make_float2(c1.x, c1.y); cs[3] = make_float2(c1.z, c1.w);
      sn[0] = make_float2(sg * s0.x, sg * s0.y); sn[1] = make_float2(sg * s0.z, sg * s0.w);
      sn[2] = make_float2(sg * s1.x, sg * s1.y); sn[3] = make_float2(sg * s1.z, sg * s1.w);
#pragma unroll
      for (int k = 0; k < 4; ++k) ns[k] = make_float2(-sn[k].x, -sn[k].y);
      dcache = d;
    };
    // (a, b) -> (a·c − b·s, b·c + a·s) on two NeoX pairs at once (FFMA2/FMUL2: per lane the same
    // roundings as rebase_pair)
    auto rot = [&](uint32_t& xa, uint32_t& xb, int k) {
      const float2 av = make_float2(__uint_as_float(xa << 16), __uint_as_float(xa & 0xFFFF0000u));
      const float2 bv = make_float2(__uint_as_float(xb << 16), __uint_as_float(xb & 0xFFFF0000u));
      const float2 ra = fma2(av, cs[k], mul2(bv, ns[k]));
      const float2 rb = fma2(bv, cs[k], mul2(av, sn[k]));
      xa = pack_bf16(ra.x, ra.y);
      xb = pack_bf16(rb.x, rb.y);
    };
    for (int t = 0; t < n; ++t) {
      const int s = t % S;
      int dl[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) dl[m] = bd[min((j0 + t) * 8 + m, last_blk)];
      // the common case (one Δ per tile): fetch its angles while the TMA is in flight
      int dfirst = 0;
#pragma unroll
      for (int m = 7; m >= 0; --m) dfirst = dl[m] ? dl[m] : dfirst;
      if (dfirst != 0 && dfirst != dcache) load_angles(dfirst);
      mbar_wait(k_full + 8 * s, (t / S) & 1);
      const uint32_t h0 = base + kK + (2 * s) * kTile + phys, h1 = h0 + kTile;
      constexpr int BB = 4 / RPB;  // blocks per batch: 4 loads of each half in flight
#pragma unroll
      for (int m0 = 0; m0 < 8; m0 += BB) {
        uint4 xa[4], xb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (dl[m0 + j / RPB]) {
            const uint32_t o = (m0 + j / RPB) * 2048 + (j % RPB) * 1024;
            xa[j] = lds128(h0 + o);
            xb[j] = lds128(h1 + o);
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int d = dl[m0 + j / RPB];
          if (d == 0) continue;
          if (d != dcache) load_angles(d);  // a chunk boundary inside the tile
          rot(xa[j].x, xb[j].x, 0);
          rot(xa[j].y, xb[j].y, 1);
          rot(xa[j].z, xb[j].z, 2);
          rot(xa[j].w, xb[j].w, 3);
          const uint32_t o = (m0 + j / RPB) * 2048 + (j % RPB) * 1024;
          sts128(h0 + o, xa[j]);
          sts128(h1 + o, xb[j]);
        }
      }
      fence_async_smem();  // generic-proxy smem writes -> visible to the tcgen05.mma operand reads
      __syncwarp();
      if (lane == 0) mbar_arrive(k_rot + 8 * s);
    }
  } else {
    // ------------------------------------------------------------------ softmax warps
    // 8 warps: warps w and w+4 share TMEM lane quarter q = w % 4 (rows 32q..32q+31); warp half hc
    // owns keys [64hc, 64hc+64) of every S tile (= P half hc) and O columns [64hc, 64hc+64).
    // The pair exchanges its partial row max through double-buffered smem (named barrier 1+q).
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    const int r = q * 32 + lane;              // MMA row = TMEM lane
    const int qi = r / G, hh = r % G;
    const bool valid = qi < row_count;
    const int row = row_start + qi;
    const int head = g * G + hh;
    const int pos = valid ? a.row_pos[row] : max_p;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t oAddr = tmem + lane_addr + kTmO + hc * 64;
    float* xmax = reinterpret_cast<float*>(smem + kX);   // [2 parity][2 halves][128 rows]
    const float sc = a.scale_log2;
    // m_ref (log2 units): the max the current O / l are scaled to.  It is raised only when a row's
    // max grows by more than 2^8 (then O in TMEM and l are rescaled), so exp2 arguments stay <= 8
    // and the common case never touches O (FA4-style lazy rescale; exact because the final
    // normalisation uses m_ref).
    float m_ref = -INFINITY, l = 0.f;
#ifdef PIC_ATTN_PHASES  // bench-only build: per-phase softmax cycles + MMA latency (costs registers: spills at 128)
    const bool trc = tr && threadIdx.x == 64;
#else
    constexpr bool trc = false;
#endif
    unsigned long long acc_ws = 0, acc_mx = 0, acc_ex = 0, tt0 = 0, tt1 = 0;
    // finer phases (clock64 cycles, trace slots 16..22): S load, max, pair exchange, rescale, exp loop,
    // P store + wait::st, o_full wait + arrive
    unsigned long long ph_[7] = {0, 0, 0, 0, 0, 0, 0}, pc = 0;
    // P(t-1) arrive -> S(t+1) ready: the tensor pipe's PV(t-1) + S(t+1) (it idles waiting for P(t-1))
    unsigned long long arr_prev = 0, arr_cur = 0, mma_lat = 0, mma_n = 0, sum_r = 0, sum_a = 0;
    auto phase = [&](int i) {
      if (trc) {
        const unsigned long long c = clock64();
        ph_[i] += c - pc;
        pc = c;
      }
    };
    for (int t = 0; t < n; ++t) {
      const int sb = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      const int key0 = (j0 + t) * 128 + hc * 64;
      if (trc) tt0 = globaltimer();
      mbar_wait(s_full + 8 * sb, ph);
      if (trc) {
        tt1 = globaltimer();
        acc_ws += tt1 - tt0;
      }
      if (tr && t == 0 && threadIdx.x == 64) tr[3] = globaltimer();
      tc_fence_after();
      if (trc) {
        pc = clock64();
        if (t >= 2) {
          mma_lat += pc - arr_prev;
          ++mma_n;
          sum_r += pc;
          sum_a += arr_prev;
        }
      }
      const uint32_t sAddr = tmem + lane_addr + kTmS + sb * 128 + hc * 64;
      float sv[64];
      tmem_ld64(sAddr, sv);
      phase(0);
      if (key0 + 63 > pos) {  // part of the half lies beyond the row's causal limit
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = (key0 + i <= pos) ? sv[i] : -INFINITY;
      }
      // four independent 3-input max chains (a single chain is 32 dependent FMNMX3)
      float m4[4] = {fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]), fmaxf(sv[4], sv[5]), fmaxf(sv[6], sv[7])};
#pragma unroll
      for (int i = 8; i < 64; i += 8) {
        m4[0] = fmax3(m4[0], sv[i], sv[i + 1]);
        m4[1] = fmax3(m4[1], sv[i + 2], sv[i + 3]);
        m4[2] = fmax3(m4[2], sv[i + 4], sv[i + 5]);
        m4[3] = fmax3(m4[3], sv[i + 6], sv[i + 7]);
      }
      float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
      mx *= sc;  // log2 units (sc > 0)
      phase(1);
      xmax[(sb * 2 + hc) * 128 + r] = mx;
      named_bar_sync(1 + q, 64);
      mx = fmaxf(mx, xmax[(sb * 2 + (hc ^ 1)) * 128 + r]);
      phase(2);
      // tcgen05.ld/st are warp-collective: the rescale runs for the whole warp if any row needs it
      // (both warps of a pair see identical maxima, so they take identical decisions)
      const bool grow = mx > m_ref + 8.f;
      const bool need = grow && m_ref != -INFINITY;
      if (__any_sync(0xffffffffu, need)) {
        // rescale O (all PV up to tile t-1 must have landed) and l to the new reference
        mbar_wait(o_full + 8 * ((t - 1) & 1), ((t - 1) >> 1) & 1);
        tc_fence_after();
        const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          float ov[32];
          tmem_ld32(oAddr + c * 32, ov);
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] *= alpha;
          tmem_st32_wait(oAddr + c * 32, ov);  // registers reused next iteration
        }
        tmem_wait_st();
        l *= alpha;
      }
      if (grow) m_ref = mx;
      phase(3);
      if (trc) {
        tt0 = globaltimer();
        acc_mx += tt0 - tt1;
      }
      const float nmu = (m_ref == -INFINITY) ? 0.f : -m_ref;
      const float2 sc2 = make_float2(sc, sc), nmu2 = make_float2(nmu, nmu);
      float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {  // p = 2^(s·scale − m_ref); masked keys are −inf → 0 (poly: 2^-125)
        const float2 xv = fma2(make_float2(sv[2 * c], sv[2 * c + 1]), sc2, nmu2);
        float2 pv;
        if ((c & 7) < PIC_V1_POLY8)  // part of the exponentials on the FMA pipe: the phase is MUFU-bound
          pv = exp2_poly2(xv);
        else
          pv = make_float2(ex2_approx(xv.x), ex2_approx(xv.y));
        if (c & 1)
          lb = add2(lb, pv);
        else
          la = add2(la, pv);
        pk[c] = pack_bf16(pv.x, pv.y);
      }
      l += (la.x + la.y) + (lb.x + lb.y);
      phase(4);
      // P(t) overwrites this half's S(t) columns (already in registers); PV(t) reads it from TMEM
      tmem_st32u(sAddr, pk);
      tmem_wait_st();
      phase(5);
      // consume every o_full phase (PV(t-1) has long finished here): no barrier phase completes unobserved
      if (t >= 1) mbar_wait(o_full + 8 * ((t - 1) & 1), ((t - 1) >> 1) & 1);
      tc_fence_before();
      mbar_arrive(p_full + 8 * sb);
      phase(6);
      if (trc) {
        arr_prev = arr_cur;
        arr_cur = clock64();
      }
      if (trc) acc_ex += globaltimer() - tt0;
    }
    if (trc) {
      tr[4] = globaltimer();
      tr[8] = acc_ws;
      tr[9] = acc_mx;
      tr[10] = acc_ex;
      for (int i = 0; i < 7; ++i) tr[16 + i] = ph_[i];
      tr[23] = mma_lat;
      tr[24] = mma_n;
      tr[26] = sum_r;
      tr[27] = sum_a;
    }
    if (n > 0) {
      mbar_wait(o_full + 8 * ((n - 1) & 1), ((n - 1) >> 1) & 1);
      tc_fence_after();
    }
    if (tr && threadIdx.x == 64) tr[5] = globaltimer();
    const size_t idx = ((size_t)split * a.M + row) * a.Hq + head;
    // row sum = both halves' partial sums (parity slot n&1 was last read at tile n-2)
    xmax[((n & 1) * 2 + hc) * 128 + r] = l;
    named_bar_sync(1 + q, 64);
    const float l_row = l + xmax[((n & 1) * 2 + (hc ^ 1)) * 128 + r];
    // an unsplit q-tile is final here: normalise and write bf16 O (no partials, no combine)
    const bool direct = a.row_nsplit[row_start] == 1;
    if (n > 0) {
      // every MMA has completed, so the K ring is idle: stage this warp's [32 rows][64 cols] fp32
      // O slice there (XOR-swizzled float4 slots) and store full row segments
      const float inv = direct ? 1.f / l_row : 1.f;
      float4* stg = reinterpret_cast<float4*>(smem + kK + (warp - 2) * 8192);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float ov[32];
        tmem_ld32(oAddr + c * 32, ov);  // warp-collective
#pragma unroll
        for (int i = 0; i < 8; ++i)
          stg[lane * 16 + ((c * 8 + i) ^ (lane & 7))] =
              make_float4(ov[4 * i] * inv, ov[4 * i + 1] * inv, ov[4 * i + 2] * inv, ov[4 * i + 3] * inv);
      }
      __syncwarp();
      const int jj = lane & 15;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int rr = 2 * i + (lane >> 4), rm = q * 32 + rr, qi2 = rm / G;
        if (qi2 < row_count) {
          const float4 v = stg[rr * 16 + (jj ^ (rr & 7))];
          const size_t orow = ((size_t)(row_start + qi2) * a.Hq + g * G + rm % G) * 128 + hc * 64;
          if (direct)
            reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.O) + orow)[jj] =
                make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
          else
            reinterpret_cast<float4*>(a.o_part + (size_t)split * a.M * a.Hq * 128 + orow)[jj] = v;
        }
      }
    } else if (valid) {
      float4* dst = reinterpret_cast<float4*>(a.o_part + idx * 128 + hc * 64);
      for (int i = 0; i < 16; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (valid && hc == 0 && !direct) {
      a.ml_part[2 * idx] = m_ref;
      a.ml_part[2 * idx + 1] = l_row;
    }
    if (tr && threadIdx.x == 64) tr[6] = globaltimer();
  }
  if (tr && threadIdx.x == 0) tr[7] = (unsigned long long)n;
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int attn_schedule(const int32_t* tiles, int n_tiles, const int* n_kv, int Hkv, int target_ctas, int max_split,
                  int32_t* work, int* n_work, int32_t* row_nsplit) {
  // Split q-tile t's n_kv[t] KV tiles into p_t = min(max_split, ⌈n_kv/b⌉) equal pieces for the per-CTA
  // budget b that minimises the estimated makespan on target_ctas SMs (one CTA per SM):
  //   one wave (P <= target): the longest piece;  several waves: Σ/target + longest/2 (LPT bound)
  // plus a fixed per-piece cost (prologue, epilogue, partial merge: ~kOvh KV tiles) per wave.  Pieces
  // are then issued longest first (blockIdx order is dispatch order), so long pieces never start in
  // the last wave (cfg5: 536 unsplit pieces of 5..257 tiles in q-tile order ran 2.3x the mean).
  constexpr double kOvh = 4.0;
  long max_kv = 1, total = 0;
  for (int t = 0; t < n_tiles; ++t) {
    max_kv = std::max<long>(max_kv, n_kv[t]);
    total += n_kv[t];
  }
  total *= Hkv;
  long best_b = max_kv;
  double best_cost = 1e300;
  for (long b = 1; b <= max_kv; ++b) {
    long P = 0, maxc = 0;
    for (int t = 0; t < n_tiles; ++t) {
      const long p = std::min<long>(max_split, std::max(1L, (n_kv[t] + b - 1) / b));
      P += p;
      maxc = std::max(maxc, (n_kv[t] + p - 1) / p);
    }
    P *= Hkv;
    const long waves = (P + target_ctas - 1) / target_ctas;
    const double span = P <= target_ctas ? (double)maxc : (double)total / target_ctas + 0.5 * maxc;
    const double cost = span + kOvh * waves;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best_b = b;
    }
  }
  int w = 0, mx = 1;
  for (int t = 0; t < n_tiles; ++t) {
    int pieces = (int)std::min<long>(max_split, std::max(1L, (n_kv[t] + best_b - 1) / best_b));
    const int chunk = (n_kv[t] + pieces - 1) / pieces;
    pieces = (n_kv[t] + chunk - 1) / chunk;
    for (int p = 0; p < pieces; ++p) {
      work[4 * w] = t;
      work[4 * w + 1] = p * chunk;
      work[4 * w + 2] = std::min(n_kv[t], (p + 1) * chunk);
      work[4 * w + 3] = p;
      ++w;
    }
    for (int r = 0; r < tiles[3 * t + 2]; ++r) row_nsplit[tiles[3 * t + 1] + r] = pieces;
    mx = std::max(mx, pieces);
  }
  // longest pieces first (stable: ties keep q-tile order); the split slot travels with the item
  std::vector<int> ord(w);
  for (int i = 0; i < w; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
    return work[4 * x + 2] - work[4 * x + 1] > work[4 * y + 2] - work[4 * y + 1];
  });
  std::vector<int32_t> sorted(4 * (size_t)w);
  for (int i = 0; i < w; ++i)
    for (int k = 0; k < 4; ++k) sorted[4 * i + k] = work[4 * ord[i] + k];
  std::copy(sorted.begin(), sorted.end(), work);
  *n_work = w;
  return mx;
}

template <int G>
static cudaError_t launch_attn_g(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                 const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st) {
  dim3 grid(a.n_work, a.Hkv);
  if (a.bdelta && a.qrot)
    CUDA_TRY_LAUNCH(launch_k(attn_tc_kernel<G, true, true>, dim3(grid), dim3(attn_threads<true, true>()), attn::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  else if (a.bdelta)
    CUDA_TRY_LAUNCH(launch_k(attn_tc_kernel<G, true>, dim3(grid), dim3(320 + 32 * kRotWarps), attn::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  else
    CUDA_TRY_LAUNCH(launch_k(attn_tc_kernel<G, false>, dim3(grid), dim3(320), attn::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  return cudaGetLastError();
}

template <int G>
static cudaError_t prepare_g() {
  cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_tc_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_tc_kernel<G, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  return e;
}

cudaError_t prepare_attention() {
  cudaError_t e = prepare_g<1>();
  if (e == cudaSuccess) e = prepare_g<2>();
  if (e == cudaSuccess) e = prepare_g<4>();
  if (e == cudaSuccess) e = prepare_g<8>();
  return e;
}

cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st) {
  switch (a.Hq / a.Hkv) {
    case 1: return launch_attn_g<1>(tmQ, tmK, tmV, tmK8, tmV8, a, st);
    case 2: return launch_attn_g<2>(tmQ, tmK, tmV, tmK8, tmV8, a, st);
    case 4: return launch_attn_g<4>(tmQ, tmK, tmV, tmK8, tmV8, a, st);
    case 8: return launch_attn_g<8>(tmQ, tmK, tmV, tmK8, tmV8, a, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------------
// split-KV combine: one warp per (row, head); lane s holds split s's (m, l); cross-split max and
// sum are warp-shuffle reductions; each lane then merges 4 of the 128 output columns.
__global__ void attn_combine_kernel(const float* __restrict__ o_part, const float* __restrict__ ml_part,
                                    const int32_t* __restrict__ row_nsplit, __nv_bfloat16* __restrict__ O, int M,
                                    int Hq) {
  griddep_launch();
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // the split counts are host-built plan data: read them while the attention kernel drains
  const int n_splits = wid < M * Hq ? row_nsplit[wid / Hq] : 0;
  griddep_wait();
  if (wid >= M * Hq || n_splits <= 1) return;  // unsplit rows were written by the attention kernel
  const size_t stride = (size_t)M * Hq;
  float ms = -INFINITY, ls = 0.f;
  if (lane < n_splits) {
    ms = ml_part[2 * (lane * stride + wid)];
    ls = ml_part[2 * (lane * stride + wid) + 1];
  }
  const float mmax = warp_max(ms);
  const float w = (lane < n_splits && ms != -INFINITY) ? exp2f(ms - mmax) : 0.f;
  const float L = warp_sum(w * ls);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int s = 0; s < n_splits; ++s) {
    const float ws = __shfl_sync(0xffffffffu, w, s);
    if (ws == 0.f) continue;
    const float4 v = reinterpret_cast<const float4*>(o_part + (s * stride + wid) * 128)[lane];
    acc.x += ws * v.x;
    acc.y += ws * v.y;
    acc.z += ws * v.z;
    acc.w += ws * v.w;
  }
  const float inv = 1.f / L;
  uint2 pk = make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
  reinterpret_cast<uint2*>(O + (size_t)wid * 128)[lane] = pk;
}

cudaError_t launch_attn_combine(const float* o_part, const float* ml_part, const int32_t* row_nsplit, void* O, int M,
                                int Hq, int D, cudaStream_t st) {
  if (D != 128) return cudaErrorInvalidValue;
  const int warps = M * Hq;
  CUDA_TRY_LAUNCH(launch_k(attn_combine_kernel, dim3((warps + 7) / 8), dim3(256), 0, st, o_part, ml_part, row_nsplit,
                           reinterpret_cast<__nv_bfloat16*>(O), M, Hq));
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// Generic-D SIMT attention for the tiny configs (D = 16/32/64, no TMA box fits) and for the fp32
// debug build (any D <= 128, fp32 Q/K/V/O): one warp per (row, head); lanes stride over keys; two
// passes (max, then exp/sum/PV) in fp32.
template <bool F32>
PIC_DEV float ldx(const void* p, size_t i) {
  if constexpr (F32)
    return reinterpret_cast<const float*>(p)[i];
  else
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

template <int D, bool F32>
__global__ void attn_simt_kernel(const void* __restrict__ Q, const void* __restrict__ Kp, const void* __restrict__ Vp,
                                 const int32_t* __restrict__ row_seq, const int32_t* __restrict__ seq_bt_off,
                                 const int32_t* __restrict__ bt, const int32_t* __restrict__ row_pos,
                                 void* __restrict__ O, int M, int Hq, int Hkv, float scale,
                                 const int32_t* __restrict__ bdelta, const float* __restrict__ cos_t,
                                 const float* __restrict__ sin_t, const int32_t* __restrict__ vbt) {
  PIC_PDL_ENTRY();
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= M * Hq) return;
  const int row = wid / Hq, head = wid % Hq;
  const int g = head * Hkv / Hq;
  const int pos = row_pos[row];
  const int* tb = bt + seq_bt_off[row_seq[row]];
  float q[D];
#pragma unroll
  for (int i = 0; i < D; ++i) q[i] = ldx<F32>(Q, ((size_t)row * Hq + head) * D + i);
  const int* tbd = bdelta ? bdelta + seq_bt_off[row_seq[row]] : nullptr;
  auto kv_off = [&](int key) -> size_t {
    const int blk = tb[key / 16];
    return (((size_t)blk * Hkv + g) * 16 + (key % 16)) * D;
  };
  const int* vtb = vbt ? vbt + seq_bt_off[row_seq[row]] : tb;  // V linked by reference (kv_share 2)
  auto v_off = [&](int key) -> size_t {
    const int blk = vtb[key / 16];
    return (((size_t)blk * Hkv + g) * 16 + (key % 16)) * D;
  };
  // key row of `key` at its linked position: a shared chunk-store block (f3) is re-based by its Δ on
  // load with the a2 arithmetic (rebase_pair, then the pool's precision), so the row equals the copy
  // path's linked row
  auto load_k = [&](int key, size_t off, float* kr) {
#pragma unroll
    for (int i = 0; i < D; ++i) kr[i] = ldx<F32>(Kp, off + i);
    const int dl = tbd ? tbd[key / 16] : 0;
    if (dl == 0) return;
    const int ad = dl < 0 ? -dl : dl;
    const float sg = dl < 0 ? -1.f : 1.f;
#pragma unroll
    for (int j = 0; j < D / 2; ++j) {
      float ra, rb;
      rebase_pair(kr[j], kr[j + D / 2], cos_t[(size_t)ad * (D / 2) + j], sg * sin_t[(size_t)ad * (D / 2) + j], ra, rb);
      if constexpr (F32) {
        kr[j] = ra;
        kr[j + D / 2] = rb;
      } else {
        kr[j] = __bfloat162float(__float2bfloat16(ra));
        kr[j + D / 2] = __bfloat162float(__float2bfloat16(rb));
      }
    }
  };
  float mx = -INFINITY;
  for (int key = lane; key <= pos; key += 32) {
    const size_t off = kv_off(key);
    float kr[D];
    load_k(key, off, kr);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) s += q[i] * kr[i];
    mx = fmaxf(mx, s * scale);
  }
  mx = warp_max(mx);
  float l = 0.f, o[D];
#pragma unroll
  for (int i = 0; i < D; ++i) o[i] = 0.f;
  for (int key = lane; key <= pos; key += 32) {
    const size_t off = kv_off(key);
    float kr[D];
    load_k(key, off, kr);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) s += q[i] * kr[i];
    const float p = expf(s * scale - mx);
    l += p;
    const size_t voff = v_off(key);
#pragma unroll
    for (int i = 0; i < D; ++i) o[i] += p * ldx<F32>(Vp, voff + i);
  }
  l = warp_sum(l);
#pragma unroll
  for (int i = 0; i < D; ++i) o[i] = warp_sum(o[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const size_t oi = ((size_t)row * Hq + head) * D + i;
      if constexpr (F32)
        reinterpret_cast<float*>(O)[oi] = o[i] / l;
      else
        reinterpret_cast<__nv_bfloat16*>(O)[oi] = __float2bfloat16(o[i] / l);
    }
  }
}

cudaError_t launch_attention_simt(const void* Q, const void* Kpool_l, const void* Vpool_l, const int32_t* row_seq,
                                  const int32_t* seq_bt_off, const int32_t* bt, const int32_t* row_pos, void* O,
                                  int M, int Hq, int Hkv, int D, float scale, cudaStream_t st, int f32,
                                  const int32_t* bdelta, const float* cos_t, const float* sin_t, const int32_t* vbt) {
  const int warps = M * Hq;
  dim3 grid((warps + 3) / 4), block(128);
#define SIMT_L(DD, FF)                                                                                              \
  CUDA_TRY_LAUNCH(launch_k(attn_simt_kernel<DD, FF>, dim3(grid), dim3(block), 0, st, Q, Kpool_l, Vpool_l, row_seq,  \
                           seq_bt_off, bt, row_pos, O, M, Hq, Hkv, scale, bdelta, cos_t, sin_t, vbt))
  if (f32) {
    switch (D) {
      case 16: SIMT_L(16, true); break;
      case 32: SIMT_L(32, true); break;
      case 64: SIMT_L(64, true); break;
      case 128: SIMT_L(128, true); break;
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (D) {
      case 16: SIMT_L(16, false); break;
      case 32: SIMT_L(32, false); break;
      case 64: SIMT_L(64, false); break;
      default: return cudaErrorInvalidValue;
    }
  }
#undef SIMT_L
  return cudaGetLastError();
}

}  // namespace pic
