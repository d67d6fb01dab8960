// attention_pp.cu — a6, v2: persistent ping-pong sparse-query attention.
//
// Computes the same Eq. (1) as attention.cu (P:215 A = softmax(Q K_expᵀ · MASK), O = A V_exp
// "allowing the k' tokens to attend to all N tokens"; P:217 causal MASK; reading R3: additive −∞,
// scale 1/√D), with a different schedule:
//   * Two query lanes per CTA (A, B).  Each lane is one GQA-packed q-tile (128 MMA rows = 128/G
//     queries × G heads of kv-head g) and a KV range.  When both lanes belong to the same sequence and
//     start at the same KV tile, every K/V tile is loaded ONCE and used by both lanes (half the
//     L2→SMEM traffic per FLOP of the one-lane kernel, which ran at ~half the L2 throughput cap).
//   * The lanes ping-pong on the tensor core (FA4-style issue order S_A, S_B, PV_A, S_A', PV_B, S_B', …):
//     while one lane's softmax warpgroup turns S into P, the tensor core runs the other lane's MMAs.
//   * One thread per MMA row (a warpgroup per lane), the whole 128-key row in registers: the row max
//     is thread-local (3-input FMNMX), no cross-warp exchange.
//   * Persistent: 148 CTAs walk a host-sorted item list (longest first); the producer fetches the
//     next item's Q and K/V while the current item's last softmax and epilogue drain.  O stays in
//     TMEM (lazy FA4 rescale: only when a row max grows by > 2^8) and unsplit lanes write normalised
//     bf16 O directly; split lanes leave fp32 partials + (m, l) for attn_combine.
// TMEM (512 columns): S_A [0,128), S_B [128,256) (P_X overwrites S_X as bf16 pairs), O_A [256,384),
// O_B [384,512).  SMEM: Q_A, Q_B (64 KB), K ring 3 × 32 KB, V ring 2 × 32 KB (SWIZZLE_128B halves).
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

namespace attn2 {
constexpr int kTile = 16384;  // one [128 rows][64 cols] bf16 SW128 half tile
#ifndef PIC_PP_KS
#define PIC_PP_KS 2  // K 2 + V 3 slots: 1% faster than 3 + 2 (the producer stalled on V slots)
#endif
constexpr int kKS = PIC_PP_KS, kVS = 5 - PIC_PP_KS;  // K and V ring depths (32 KB slots)
constexpr int kQ = 0;                       // Q_A halves, Q_B halves
constexpr int kK = kQ + 4 * kTile;          // K ring
constexpr int kV = kK + kKS * 2 * kTile;    // V ring
constexpr int kBar = kV + kVS * 2 * kTile;  // barriers
constexpr int kIR = 4;  // item-index ring (producer -> every other role)
constexpr int bQFull = 0, bQEmpty = 2, bKFull = 4, bKEmpty = bKFull + kKS, bKRot = bKEmpty + kKS,
              bVFull = bKRot + kKS, bVEmpty = bVFull + kVS, bSFull = bVEmpty + kVS, bPFull = bSFull + 2,
              bOFull = bPFull + 2, bOFree = bOFull + 2, bIFull = bOFree + 2, bIEmpty = bIFull + kIR,
              kNumBars = bIEmpty + kIR;
constexpr int kSmem = kBar + kNumBars * 8 + 16 + kIR * 4;
static_assert(kSmem <= 232448, "attention smem over the 227 KB limit");
constexpr int kRotWarps = 4;  // ROT: warpgroup 1 (warps 4-7) re-bases shared K tiles
#ifndef PIC_PP_TURN
#define PIC_PP_TURN 0
#endif
// PIC_PP_TURN=1 (A/B only): the two softmax warpgroups take strict turns (named barriers 1 and 2,
// FA3-style): lane B's step s starts when lane A's step s is done, lane A's step s+1 when lane B's step s
// is done, to break the lanes' convoy (both softmaxes at once, then both waiting on the back-to-back MMAs
// of both lanes).  Measured at cfg4 (copy path): 178-179 vs 175.7-176.3 ms per step without turns; the
// softmax step does not get faster alone (~1900 cycles per 128x128 lane step either way): it is latency-,
// not MUFU-bound, so serialising the lanes only lengthens the period.
constexpr int kBarTurnA = 1, kBarTurnB = 2;
// register split of the 384-thread CTA: 128·(producer, MMA, rotation) + 256·softmax <= 64 K
// ROT register split of the 512-thread CTA: producer/MMA warpgroup 48, rotation warpgroup 104, softmax
// warpgroups 176 (two-pass over TMEM: half a row in registers)
constexpr int kRegW0Rot = 48, kRegRotWG = 104, kRegSmRot = 176;
static_assert(128 * kRegW0Rot + 128 * kRegRotWG + 256 * kRegSmRot <= 65536, "register split over the file");
}  // namespace attn2

struct PPLane {
  int tile, j0, n, split, seq, row_start, row_count, max_p;
};


// Item `item` of the host list (whole warp): lanes ordered so that A has the longer KV run; `sh`: both
// lanes read the same K/V tiles (same sequence, same first tile).
PIC_DEV void pp_lane(const AttnArgs& a, const int* wk, int x, PPLane& p) {
  p.tile = wk[4 * x];
  p.j0 = wk[4 * x + 1];
  p.split = wk[4 * x + 3];
  if (p.tile < 0) {
    p.n = 0;
    p.seq = -1 - x;
    p.row_start = p.row_count = p.max_p = 0;
    return;
  }
  p.seq = a.tiles[3 * p.tile];
  p.row_start = a.tiles[3 * p.tile + 1];
  p.row_count = a.tiles[3 * p.tile + 2];
  int mp = 0;
  for (int i = lane_id(); i < p.row_count; i += 32) mp = max(mp, a.row_pos[p.row_start + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mp = max(mp, __shfl_xor_sync(0xffffffffu, mp, o));
  p.max_p = mp;
  // positions may be device-side (CacheBlend's re-selected rows): clamp the host's range
  p.n = max(0, min(mp / 128 + 1, wk[4 * x + 2]) - p.j0);
}
PIC_DEV void pp_decode(const AttnArgs& a, int item, PPLane& A, PPLane& Bn, int& g, bool& sh) {
  // head-major item order: the CTAs work through one kv-head's K/V (L2-resident) at a time
  const int* wk = a.work + 8 * (item % a.n_work);
  g = item / a.n_work;
  PPLane p0, p1;
  pp_lane(a, wk, 0, p0);
  pp_lane(a, wk, 1, p1);
  const bool sw = p0.n < p1.n;
  A = sw ? p1 : p0;
  Bn = sw ? p0 : p1;
  sh = Bn.n > 0 && A.seq == Bn.seq && A.j0 == Bn.j0;
}

// Bench-only cycle accounting (AttnArgs.trace, PIC_ATTN_TRACE=1): per CTA 32 counters, see kTr*.
enum {
  kTrStart = 0, kTrEnd, kTrPwK, kTrPwV, kTrPwQ, kTrPtiles, kTrMwK, kTrMwP, kTrMwV, kTrMwQ, kTrMwO,
  kTrSwS0, kTrSc0, kTrSe0, kTrSn0, kTrSwS1, kTrSc1, kTrSe1, kTrSn1, kTrRw, kTrRc, kTrItems, kTrPwI
};
PIC_DEV unsigned long long clk() { return clock64(); }
// mbar_wait that adds the cycles it spent to *acc (acc may be null)
PIC_DEV void mbar_wait_acc(uint32_t bar, uint32_t ph, unsigned long long* acc) {
  if (!acc) {
    mbar_wait(bar, ph);
    return;
  }
  const unsigned long long t0 = clk();
  mbar_wait(bar, ph);
  *acc += clk() - t0;
}

// position of lane x's step-s K (or V) tile in the item's load order: shared → one tile per step;
// otherwise A, B alternate while both run, then A alone
PIC_DEV int pp_tidx(int x, int s, int nB, bool sh) {
  if (sh) return s;
  if (s < nB) return 2 * s + x;
  return 2 * nB + (s - nB);
}

template <int G, bool ROT>
__global__ void __launch_bounds__(ROT ? 512 : 384, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmK8,
                   const __grid_constant__ CUtensorMap tmV8, const AttnArgs a) {
  griddep_launch();
  using namespace attn2;
  constexpr int SM0 = ROT ? 8 : 4;  // first softmax warp (lane A: SM0..SM0+3, lane B: SM0+4..SM0+7)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  const uint32_t base = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto B = [&](int i) -> uint32_t { return bar0 + 8 * i; };
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(B(bQFull + x), 1);
      mbar_init(B(bQEmpty + x), 1);
      mbar_init(B(bSFull + x), 1);
      mbar_init(B(bPFull + x), 128);
      mbar_init(B(bOFull + x), 1);
      mbar_init(B(bOFree + x), 128);
    }
    for (int s = 0; s < kKS; ++s) {
      mbar_init(B(bKFull + s), 1);
      mbar_init(B(bKEmpty + s), 1);
      mbar_init(B(bKRot + s), kRotWarps);
    }
    for (int s = 0; s < kVS; ++s) {
      mbar_init(B(bVFull + s), 1);
      mbar_init(B(bVEmpty + s), 1);
    }
    for (int s = 0; s < kIR; ++s) {
      mbar_init(B(bIFull + s), 1);
      mbar_init(B(bIEmpty + s), ROT ? 13 : 9);  // MMA warp, rotation warps, softmax warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int* const iring = reinterpret_cast<int*>(tmem_slot + 4);
  unsigned long long* const tr = a.trace ? a.trace + 32 * blockIdx.x : nullptr;
  unsigned long long tacc[4] = {0, 0, 0, 0};  // per-role accumulators (flushed at the end)
  if (tr && threadIdx.x == 0) tr[kTrStart] = clk();
  griddep_wait();  // Q, the recomputed rows' K/V and (CacheBlend) device-side positions come from upstream
  const int n_items = a.n_work * a.Hkv;
  // Dynamic item queue: the producer takes the next item from the global counter (list order = longest
  // first within each kv-head) and hands its index to the other roles through a smem ring; -1 ends.
  auto next_item = [&](int k) -> int {  // consumers (whole warp)
    const int sl = k % kIR;
    mbar_wait(B(bIFull + sl), (k / kIR) & 1);
    const int it = *reinterpret_cast<volatile int*>(iring + sl);
    __syncwarp();
    if (lane == 0) mbar_arrive(B(bIEmpty + sl));
    return it;
  };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(ROT ? kRegW0Rot : 56) : "memory");
    if (warp == 0) {
      // ------------------------------------------------------------------ TMA producer
      int kc = 0, vc = 0, qc0 = 0, qc1 = 0;
      if (lane == 0) {
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        tma_prefetch(&tmK8);
        tma_prefetch(&tmV8);
      }
      // one 128-key K or V tile of (seq, kv tile j): 8 paged blocks, one 8-block box when contiguous
      auto load_tile = [&](const CUtensorMap* t1, const CUtensorMap* t8, uint32_t dst, uint32_t full, uint32_t empty,
                           uint32_t ph, const int* bt, int j, int last_blk, int g) {
        const int kv_base = a.layer * a.num_blocks;
        const int mine = lane < 8 ? bt[min(j * 8 + lane, last_blk)] : 0;
        const int b0 = __shfl_sync(0xffffffffu, mine, 0);
        const bool contig = __all_sync(0xffffffffu, lane >= 8 || mine == b0 + lane);
        int blk[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) blk[b] = __shfl_sync(0xffffffffu, mine, b);
        if (lane == 0) {
          mbar_wait_acc(empty, ph ^ 1, tr ? (t1 == &tmK ? &tacc[0] : &tacc[1]) : nullptr);
          mbar_expect_tx(full, 2 * kTile);
          if (contig) {
            for (int h = 0; h < 2; ++h) tma_load_4d(dst + h * kTile, t8, full, h * 64, 0, g, kv_base + b0);
          } else {
#pragma unroll
            for (int b = 0; b < 8; ++b)
              for (int h = 0; h < 2; ++h) tma_load_4d(dst + h * kTile + b * 2048, t1, full, h * 64, 0, g, kv_base + blk[b]);
          }
        }
        __syncwarp();
      };
      for (int k = 0;; ++k) {
        int item = 0;
        if (lane == 0) {
          const int sl = k % kIR;
          mbar_wait(B(bIEmpty + sl), ((k / kIR) & 1) ^ 1);
          item = (int)atomicAdd(a.item_ctr, 1u);
          if (tr) ++tacc[3];
          if (item >= n_items) item = -1;
          iring[sl] = item;
          mbar_arrive(B(bIFull + sl));
        }
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item < 0) break;
        PPLane LA, LB;
        int g;
        bool sh;
        pp_decode(a, item, LA, LB, g, sh);
        const int nA = LA.n, nB = LB.n;
        if (nA == 0) continue;
        if (lane == 0) {
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if ((x ? nB : nA) == 0) continue;
            const int qc = x ? qc1 : qc0;
            mbar_wait_acc(B(bQEmpty + x), (qc & 1) ^ 1, tr ? &tacc[2] : nullptr);
            mbar_expect_tx(B(bQFull + x), 2 * kTile);
            for (int h = 0; h < 2; ++h)
              tma_load_3d(base + kQ + (2 * x + h) * kTile, &tmQ, B(bQFull + x), h * 64, g * G,
                          x ? LB.row_start : LA.row_start);
          }
        }
        ++qc0;
        if (nB) ++qc1;
        const int* btA = a.bt + a.seq_bt_off[LA.seq];
        const int* btB = sh ? btA : (nB ? a.bt + a.seq_bt_off[LB.seq] : btA);
        // V's own block table when V is linked by reference (kv_share 2)
        const int* vbA = a.vbt ? a.vbt + a.seq_bt_off[LA.seq] : btA;
        const int* vbB = a.vbt ? (sh ? vbA : (nB ? a.vbt + a.seq_bt_off[LB.seq] : vbA)) : btB;
        const int lastA = (sh ? max(LA.max_p, LB.max_p) : LA.max_p) / 16;
        const int lastB = LB.max_p / 16;
        for (int s = 0; s < nA; ++s) {
          const bool two = s < nB && !sh;
          {
            const int k = kc++, sl = k % kKS;
            load_tile(&tmK, &tmK8, base + kK + sl * 2 * kTile, B(bKFull + sl), B(bKEmpty + sl), (k / kKS) & 1, btA,
                      LA.j0 + s, lastA, g);
          }
          if (two) {
            const int k = kc++, sl = k % kKS;
            load_tile(&tmK, &tmK8, base + kK + sl * 2 * kTile, B(bKFull + sl), B(bKEmpty + sl), (k / kKS) & 1, btB,
                      LB.j0 + s, lastB, g);
          }
          {
            const int k = vc++, sl = k % kVS;
            load_tile(&tmV, &tmV8, base + kV + sl * 2 * kTile, B(bVFull + sl), B(bVEmpty + sl), (k / kVS) & 1, vbA,
                      LA.j0 + s, lastA, g);
          }
          if (two) {
            const int k = vc++, sl = k % kVS;
            load_tile(&tmV, &tmV8, base + kV + sl * 2 * kTile, B(bVFull + sl), B(bVEmpty + sl), (k / kVS) & 1, vbB,
                      LB.j0 + s, lastB, g);
          }
        }
      }
      if (tr && lane == 0) {
        tr[kTrPwK] = tacc[0];
        tr[kTrPwV] = tacc[1];
        tr[kTrPwQ] = tacc[2];
        tr[kTrItems] = tacc[3];
        tr[kTrPtiles] = kc;
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------------ MMA issuer (lane 0)
      constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // Q (smem, K-major) x K (smem, K-major)
      constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (TMEM, K-major) x V (smem, MN-major)
      int kc = 0, vc = 0;
      int qcA = 0, qcB = 0, pcA = 0, pcB = 0, ecA = 0, ecB = 0;  // Q loads, PV issues, items per lane
      unsigned long long tmw_o = 0;
      // base descriptors (slot / k-step offsets are added to the 14-bit address field, which never carries)
      const uint64_t dQ0 = sdesc_sw128(base + kQ, 16, 1024), dQ1 = sdesc_sw128(base + kQ + 2 * kTile, 16, 1024);
      const uint64_t dK0 = sdesc_sw128(base + kK, 16, 1024), dV0 = sdesc_sw128(base + kV, kTile, 1024);
      for (int k = 0;; ++k) {
        const int item = next_item(k);
        if (item < 0) break;
        PPLane LA, LB;
        int g;
        bool sh;
        pp_decode(a, item, LA, LB, g, sh);
        const int nA = LA.n, nB = LB.n;
        if (nA == 0) continue;
        // the whole warp runs the issue loop (convergent, uniform state); elect.sync issues
        auto issue_S = [&](int x, int s) {
          const int k = kc + pp_tidx(x, s, nB, sh), sl = k % kKS;
          mbar_wait_acc(B((ROT && a.debug != 3 ? bKRot : bKFull) + sl), (k / kKS) & 1, tr ? &tacc[0] : nullptr);
          if (s == 0) mbar_wait_acc(B(bQFull + x), (x ? qcB : qcA) & 1, tr ? &tacc[3] : nullptr);
          tc_fence_after();
          const uint64_t dq = x ? dQ1 : dQ0, dk = dK0 + (uint64_t)(sl * (2 * kTile / 16));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t o = (uint64_t)(((kk >> 2) * kTile + (kk & 3) * 32) >> 4);
            umma_bf16_e(tmem + 128 * x, dq + o, dk + o, idS, kk > 0);
          }
          umma_commit_e(B(bSFull + x));
          if (!(sh && x == 0 && s < nB)) umma_commit_e(B(bKEmpty + sl));  // last reader of this K slot
          if (s == (x ? nB : nA) - 1) umma_commit_e(B(bQEmpty + x));
        };
        auto issue_PV = [&](int x, int s) {
          mbar_wait_acc(B(bPFull + x), (x ? pcB : pcA) & 1, tr ? &tacc[1] : nullptr);
          const int v = vc + pp_tidx(x, s, nB, sh), sl = v % kVS;
          mbar_wait_acc(B(bVFull + sl), (v / kVS) & 1, tr ? &tacc[2] : nullptr);
          if (s == 0)  // previous item's O_X read out
            mbar_wait_acc(B(bOFree + x), ((x ? ecB : ecA) & 1) ^ 1, tr ? &tmw_o : nullptr);
          tc_fence_after();
          const uint64_t dv = dV0 + (uint64_t)(sl * (2 * kTile / 16));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // keys 16kk..16kk+15: P at S_X column 64·(kk/4) + 8·(kk%4); V rows 16kk.. of the slot
            const uint32_t pa = tmem + 128 * x + (kk >> 2) * 64 + (kk & 3) * 8;
            umma_bf16_ts_e(tmem + 256 + 128 * x, pa, dv + (uint64_t)(kk * 2048 / 16), idO, (s | kk) != 0);
          }
          umma_commit_e(B(bOFull + x));
          if (!(sh && x == 0 && s < nB)) umma_commit_e(B(bVEmpty + sl));
          if (x) ++pcB; else ++pcA;
        };
        // issue order S_A(0), S_B(0), then per step: PV_A(s), S_A(s+1), PV_B(s), S_B(s+1)
#pragma unroll 1
        for (int s = -1; s < nA; ++s) {
#pragma unroll 1
          for (int x = 0; x < 2; ++x) {
            const int nx = x ? nB : nA;
            if (s >= 0 && s < nx) issue_PV(x, s);
            if (s + 1 < nx) issue_S(x, s + 1);
          }
        }
        ++qcA;
        ++ecA;
        if (nB) {
          ++qcB;
          ++ecB;
        }
        __syncwarp();
        kc += nA + (sh ? 0 : nB);
        vc += nA + (sh ? 0 : nB);
      }
      if (tr && lane == 0) {  // (every lane accumulated the same waits)
        tr[kTrMwK] = tacc[0];
        tr[kTrMwP] = tacc[1];
        tr[kTrMwV] = tacc[2];
        tr[kTrMwQ] = tacc[3];
        tr[kTrMwO] = tmw_o;
      }
    }
  } else if (ROT && warp < 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegRotWG) : "memory");
    // ------------------------------------------------------------------ K-tile re-base (f3)
    // As attention.cu: keys of chunk-store blocks linked by reference are rotated by their block's Δ
    // (rebase_pair arithmetic, so the tile equals the copy path's a2-re-based one).  Thread u owns the
    // logical 16-B chunk cc = u & 7 of rows rg + 8i of each paged block; dims j and j+64 sit at the same
    // offset of the two SW128 halves.
    constexpr int RPB = 16 / (4 * kRotWarps);
    const int u = threadIdx.x - 128;
    const int cc = u & 7, rg = u >> 3;
    const uint32_t phys = (uint32_t)(((cc ^ (rg & 7)) << 4) + rg * 128);
    int dcache = 0;
    float2 cs[4], sn[4];
    auto load_angles = [&](int d) {
      const int ad = d < 0 ? -d : d;
      const float sg = d < 0 ? -1.f : 1.f;
      const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + cc * 8);
      const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + cc * 8);
      const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
      cs[0] = make_float2(c0.x, c0.y);
      cs[1] = make_float2(c0.z, c0.w);
      cs[2] = make_float2(c1.x, c1.y);
      cs[3] = make_float2(c1.z, c1.w);
      sn[0] = make_float2(sg * s0.x, sg * s0.y);
      sn[1] = make_float2(sg * s0.z, sg * s0.w);
      sn[2] = make_float2(sg * s1.x, sg * s1.y);
      sn[3] = make_float2(sg * s1.z, sg * s1.w);
      dcache = d;
    };
    auto rot = [&](uint32_t& xa, uint32_t& xb, int k) {
      const float2 av = make_float2(__uint_as_float(xa << 16), __uint_as_float(xa & 0xFFFF0000u));
      const float2 bv = make_float2(__uint_as_float(xb << 16), __uint_as_float(xb & 0xFFFF0000u));
      const float2 ra = fma2(av, cs[k], mul2(bv, make_float2(-sn[k].x, -sn[k].y)));
      const float2 rb = fma2(bv, cs[k], mul2(av, sn[k]));
      xa = pack_bf16(ra.x, ra.y);
      xb = pack_bf16(rb.x, rb.y);
    };
    auto rotate_tile = [&](int k, const int* bd, int j, int last_blk) {
      const int sl = k % kKS;
      // the tile's 8 block deltas: one load by lanes 0-7, broadcast by shuffles (not 8 loads per thread)
      const int mine = lane < 8 ? bd[min(j * 8 + lane, last_blk)] : 0;
      int dl[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) dl[m] = __shfl_sync(0xffffffffu, mine, m);
      int dfirst = 0;
#pragma unroll
      for (int m = 7; m >= 0; --m) dfirst = dl[m] ? dl[m] : dfirst;
      if (dfirst != 0 && dfirst != dcache) load_angles(dfirst);
      const unsigned long long tw = tr ? clk() : 0;
      mbar_wait(B(bKFull + sl), (k / kKS) & 1);
      const unsigned long long tw1 = tr ? clk() : 0;
      if (tr) tacc[0] += tw1 - tw;
      if (a.debug == 2 || a.debug == 4) {  // ablation: no rotation work (4: nor its proxy fence; timing only)
#pragma unroll
        for (int m = 0; m < 8; ++m) dl[m] = 0;
      }
      const uint32_t h0 = base + kK + (2 * sl) * kTile + phys, h1 = h0 + kTile;
      constexpr int NB = 2;  // 16-B chunk pairs in flight per thread (104 registers)
      constexpr int BB = NB / RPB;
#pragma unroll
      for (int m0 = 0; m0 < 8; m0 += BB) {
        uint4 xa[NB], xb[NB];
#pragma unroll
        for (int jj = 0; jj < NB; ++jj)
          if (dl[m0 + jj / RPB]) {
            const uint32_t o = (m0 + jj / RPB) * 2048 + (jj % RPB) * 1024;
            xa[jj] = lds128(h0 + o);
            xb[jj] = lds128(h1 + o);
          }
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) {
          const int d = dl[m0 + jj / RPB];
          if (d == 0) continue;
          if (d != dcache) load_angles(d);
          rot(xa[jj].x, xb[jj].x, 0);
          rot(xa[jj].y, xb[jj].y, 1);
          rot(xa[jj].z, xb[jj].z, 2);
          rot(xa[jj].w, xb[jj].w, 3);
          const uint32_t o = (m0 + jj / RPB) * 2048 + (jj % RPB) * 1024;
          sts128(h0 + o, xa[jj]);
          sts128(h1 + o, xb[jj]);
        }
      }
      if (a.debug != 4) fence_async_smem();  // generic-proxy smem writes -> visible to the tcgen05.mma operand reads
      __syncwarp();
      if (lane == 0) mbar_arrive(B(bKRot + sl));
      if (tr) tacc[1] += clk() - tw1;
    };
    int kc = 0;
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      if (a.debug == 3) continue;  // ablation: rotation warps idle, MMA reads unrotated K (timing only)
      PPLane LA, LB;
      int g;
      bool sh;
      pp_decode(a, item, LA, LB, g, sh);
      const int nA = LA.n, nB = LB.n;
      if (nA == 0) continue;
      const int* bdA = a.bdelta + a.seq_bt_off[LA.seq];
      const int* bdB = sh ? bdA : (nB ? a.bdelta + a.seq_bt_off[LB.seq] : bdA);
      const int lastA = (sh ? max(LA.max_p, LB.max_p) : LA.max_p) / 16;
      const int lastB = LB.max_p / 16;
      for (int s = 0; s < nA; ++s) {
        rotate_tile(kc++, bdA, LA.j0 + s, lastA);
        if (s < nB && !sh) rotate_tile(kc++, bdB, LB.j0 + s, lastB);
      }
    }
    if (tr && threadIdx.x == 128) {
      tr[kTrRw] = tacc[0];
      tr[kTrRc] = tacc[1];
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(ROT ? kRegSmRot : 224) : "memory");
    // ------------------------------------------------------------------ softmax warpgroups
    const int x = (warp - SM0) >> 2;       // lane
    const int q = warp & 3;                // TMEM lane quarter
    const int r = q * 32 + lane;           // MMA row = TMEM lane
    const int qi = r / G, hh = r % G;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t sAddr = tmem + lane_addr + 128 * x;
    const uint32_t oAddr = tmem + lane_addr + 256 + 128 * x;
    const float sc = a.scale_log2;
    int cs = 0;  // S tiles of this lane so far (s_full / p_full / o_full phases)
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      PPLane LA, LB;
      int g;
      bool sh;
      pp_decode(a, item, LA, LB, g, sh);
      const PPLane P = x ? LB : LA;
      const bool valid = qi < P.row_count;
      const int row = P.row_start + qi;
      const int head = g * G + hh;
      if (P.n == 0) {
        // an empty split piece (device-side positions end before it): neutral partial for combine
        if (P.tile >= 0 && valid) {
          const size_t idx = ((size_t)P.split * a.M + row) * a.Hq + head;
          float4* dst = reinterpret_cast<float4*>(a.o_part + idx * 128);
          for (int i = 0; i < 32; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          a.ml_part[2 * idx] = -INFINITY;
          a.ml_part[2 * idx + 1] = 0.f;
        }
        continue;
      }
      const int pos = valid ? a.row_pos[row] : P.max_p;
      float m_ref = -INFINITY, l = 0.f;
      const int nA = LA.n, nB = LB.n;  // nA >= nB (pp_decode)
      for (int s = 0; s < P.n; ++s) {
        const unsigned long long tw = tr ? clk() : 0;
        mbar_wait(B(bSFull + x), cs & 1);
        if (PIC_PP_TURN && a.debug != 1) {  // my turn: the other lane's previous softmax step is done
          if (x == 0) {
            if (s >= 1 && s - 1 < nB) named_bar_sync(kBarTurnA, 256);
          } else {
            named_bar_sync(kBarTurnB, 256);
          }
        }
        const unsigned long long tw1 = tr ? clk() : 0;
        if (tr) tacc[0] += tw1 - tw;
        tc_fence_after();
        if (a.debug == 1) {  // ablation: hand S straight back as P (timing only)
          tc_fence_before();
          mbar_arrive(B(bPFull + x));
          ++cs;
          continue;
        }
        const int key0 = (P.j0 + s) * 128;
        // row max of v[0..n) (FMNMX3 tree), masking keys beyond the row's causal limit first
        auto mask_max = [&](float* v, int n, int k0) -> float {
          if (k0 + n - 1 > pos) {
#pragma unroll
            for (int i = 0; i < n; ++i) v[i] = (k0 + i <= pos) ? v[i] : -INFINITY;
          }
          float m4[4] = {fmaxf(v[0], v[1]), fmaxf(v[2], v[3]), fmaxf(v[4], v[5]), fmaxf(v[6], v[7])};
#pragma unroll
          for (int i = 8; i < n; i += 8) {  // n is a multiple of 8: v[i..i+7] stays in range
            m4[0] = fmax3(m4[0], v[i], v[i + 1]);
            m4[1] = fmax3(m4[1], v[i + 2], v[i + 3]);
            m4[2] = fmax3(m4[2], v[i + 4], v[i + 5]);
            m4[3] = fmax3(m4[3], v[i + 6], v[i + 7]);
          }
          return fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
        };
        float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
        // p = 2^(s·scale − m_ref) for 64 keys; masked keys are −inf → 0; P as bf16 pairs into `dst`
        auto exp_half = [&](const float* v, uint32_t dst, float2 sc2, float2 nmu2) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float2 xv = fma2(make_float2(v[2 * c], v[2 * c + 1]), sc2, nmu2);
            float2 pv;
            if ((c & 7) < PIC_POLY8)
              pv = exp2_poly2(xv);
            else
              pv = make_float2(ex2_approx(xv.x), ex2_approx(xv.y));
            if (c & 1)
              lb = add2(lb, pv);
            else
              la = add2(la, pv);
            pk[c] = pack_bf16(pv.x, pv.y);
          }
          tmem_st32u_wait(dst, pk);
        };
        auto rescale = [&](float mx) {
          const bool grow = mx > m_ref + 8.f;
          const bool need = grow && m_ref != -INFINITY;
          if (__any_sync(0xffffffffu, need)) {
            // rescale O_X (PV of the previous step must have landed) and l to the new reference
            mbar_wait(B(bOFull + x), (cs - 1) & 1);
            tc_fence_after();
            const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
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
        };
        const float2 sc2 = make_float2(sc, sc);
        if constexpr (ROT) {
          // two passes over TMEM (this warpgroup runs at 160 registers beside the rotation warpgroup):
          // max over both halves, exp of the half still in registers, reload the first half
          float sv[64];
          tmem_ld64(sAddr, sv);
          float m = mask_max(sv, 64, key0);
          tmem_ld64(sAddr + 64, sv);
          m = fmaxf(m, mask_max(sv, 64, key0 + 64));
          rescale(m * sc);  // log2 units (sc > 0)
          const float nmu = (m_ref == -INFINITY) ? 0.f : -m_ref;
          const float2 nmu2 = make_float2(nmu, nmu);
          exp_half(sv, sAddr + 64, sc2, nmu2);  // keys 64..127 -> columns [64, 96): S cols 64.. already read
          tmem_ld64(sAddr, sv);
          mask_max(sv, 64, key0);
          exp_half(sv, sAddr, sc2, nmu2);       // keys 0..63 -> columns [0, 32)
        } else {
          float sv[128];
          // two x64 loads, each with its own wait in the same asm statement: a load whose wait sits in a
          // later statement lets the compiler copy destination registers before the data has landed
          tmem_ld64(sAddr, sv);
          tmem_ld64(sAddr + 64, sv + 64);
          const float m = fmaxf(mask_max(sv, 64, key0), mask_max(sv + 64, 64, key0 + 64));
          rescale(m * sc);
          const float nmu = (m_ref == -INFINITY) ? 0.f : -m_ref;
          const float2 nmu2 = make_float2(nmu, nmu);
          // keys [64h, 64h+64) -> S_X columns [64h, 64h+32) as bf16 pairs (the TS MMA's A layout); the
          // second half first, in the two-pass variant's order, so both accumulate l identically
          exp_half(sv + 64, sAddr + 64, sc2, nmu2);
          exp_half(sv, sAddr, sc2, nmu2);
        }
        const float s0 = la.x, s1 = la.y, s2 = lb.x, s3 = lb.y;
        l += (s0 + s1) + (s2 + s3);
        tmem_wait_st();
        if (PIC_PP_TURN) {  // the other lane's turn
          if (x == 0) {
            if (s < nB) named_bar_arrive(kBarTurnB, 256);
          } else {
            if (s + 1 < nA) named_bar_arrive(kBarTurnA, 256);
          }
        }
        // consume every o_full phase (PV of the previous step has long finished): none completes unobserved
        if (s >= 1) mbar_wait(B(bOFull + x), (cs - 1) & 1);
        tc_fence_before();
        mbar_arrive(B(bPFull + x));
        ++cs;
        if (tr) {
          tacc[1] += clk() - tw1;
          ++tacc[3];
        }
      }
      const unsigned long long te = tr ? clk() : 0;
      // epilogue: O_X once the last PV landed; unsplit tiles are final (normalised bf16), split ones
      // leave fp32 partials and (m, l)
      mbar_wait(B(bOFull + x), (cs - 1) & 1);
      tc_fence_after();
      const bool direct = a.row_nsplit[P.row_start] == 1;
      const float inv = direct ? 1.f / l : 1.f;
      const size_t orow = (size_t)row * a.Hq + head;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float ov[32];
        tmem_ld32(oAddr + c * 32, ov);  // warp-collective
        if (valid) {
          if (direct) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.O) + orow * 128 + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(pack_bf16(ov[8 * i] * inv, ov[8 * i + 1] * inv), pack_bf16(ov[8 * i + 2] * inv, ov[8 * i + 3] * inv),
                                  pack_bf16(ov[8 * i + 4] * inv, ov[8 * i + 5] * inv), pack_bf16(ov[8 * i + 6] * inv, ov[8 * i + 7] * inv));
          } else {
            float4* dst = reinterpret_cast<float4*>(a.o_part + ((size_t)P.split * a.M * a.Hq + orow) * 128 + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(ov[4 * i], ov[4 * i + 1], ov[4 * i + 2], ov[4 * i + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(B(bOFree + x));  // O_X may be overwritten by the next item's first PV
      if (valid && !direct) {
        const size_t idx = (size_t)P.split * a.M * a.Hq + orow;
        a.ml_part[2 * idx] = m_ref;
        a.ml_part[2 * idx + 1] = l;
      }
      if (tr) tacc[2] += clk() - te;
    }
    if (tr && (warp - SM0) % 4 == 0 && lane == 0) {
      tr[x ? kTrSwS1 : kTrSwS0] = tacc[0];
      tr[x ? kTrSc1 : kTrSc0] = tacc[1];
      tr[x ? kTrSe1 : kTrSe0] = tacc[2];
      tr[x ? kTrSn1 : kTrSn0] = tacc[3];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (tr && threadIdx.x == 0) tr[kTrEnd] = clk();
  if (threadIdx.x == 0) {  // every producer has drawn its final -1: the last CTA re-arms the queue
    __threadfence();
    if (atomicAdd(a.item_ctr + 1, 1u) == gridDim.x - 1) {
      a.item_ctr[0] = 0;
      a.item_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Host schedule: split-KV pieces from attn_schedule (sized for 2 lanes per SM), then paired into items.
// Pieces of one sequence that start at the same KV tile share their loads (both lanes read the same
// K/V tiles); they are paired longest with next-longest.  Left-over pieces are paired with another of
// similar length (no shared loads; the lanes still ping-pong).  Pairing stops where fewer than n_sms
// items would remain.  Items are sorted by their longer lane, longest first (the persistent CTAs walk
// the list with stride gridDim.x).
int attn_schedule_pp(const int32_t* tiles, int n_tiles, const int* n_kv, int Hkv, int n_sms, int max_split,
                     std::vector<int32_t>& items, int32_t* row_nsplit) {
  long total = 0;
  for (int t = 0; t < n_tiles; ++t) total += n_kv[t];
  std::vector<int32_t> work(4 * (size_t)(total + n_tiles));
  int n_work = 0;
  const int mx = attn_schedule(tiles, n_tiles, n_kv, Hkv, 2 * n_sms, max_split, work.data(), &n_work, row_nsplit);
  struct Pc {
    int t, j0, j1, slot, len, seq;
  };
  std::vector<Pc> pc(n_work);
  for (int i = 0; i < n_work; ++i) {
    const int32_t* w = &work[4 * i];
    pc[i] = {w[0], w[1], w[2], w[3], w[2] - w[1], tiles[3 * w[0]]};
  }
  std::vector<int> ord(n_work);
  for (int i = 0; i < n_work; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
    if (pc[x].seq != pc[y].seq) return pc[x].seq < pc[y].seq;
    if (pc[x].j0 != pc[y].j0) return pc[x].j0 < pc[y].j0;
    return pc[x].len > pc[y].len;
  });
  struct Cand {
    int a, b;
    double gain;
  };
  std::vector<Cand> cand;
  std::vector<char> in_shared(n_work, 0);
  for (int i = 0; i + 1 < n_work;) {
    const Pc &p = pc[ord[i]], &q = pc[ord[i + 1]];
    if (p.seq == q.seq && p.j0 == q.j0) {
      cand.push_back({ord[i], ord[i + 1], (double)q.len});  // q.len steps run two lanes on one load
      in_shared[ord[i]] = in_shared[ord[i + 1]] = 1;
      i += 2;
    } else {
      ++i;
    }
  }
  std::vector<int> left;
  for (int i = 0; i < n_work; ++i)
    if (!in_shared[i]) left.push_back(i);
  std::stable_sort(left.begin(), left.end(), [&](int x, int y) { return pc[x].len > pc[y].len; });
  for (size_t i = 0; i + 1 < left.size(); i += 2) {
    const Pc &p = pc[left[i]], &q = pc[left[i + 1]];
    if (2 * q.len >= p.len) cand.push_back({left[i], left[i + 1], 0.5 * q.len});
  }
  std::stable_sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) { return x.gain > y.gain; });
  std::vector<int> partner(n_work, -1);
  long n_items = n_work;
  for (const Cand& c : cand) {
    if ((n_items - 1) * Hkv < n_sms) break;
    partner[c.a] = c.b;
    partner[c.b] = c.a;
    --n_items;
  }
  struct It {
    int a, b, len;
  };
  std::vector<It> its;
  for (int i = 0; i < n_work; ++i) {
    if (partner[i] >= 0 && partner[i] < i) continue;
    const int b = partner[i];
    its.push_back({i, b, std::max(pc[i].len, b >= 0 ? pc[b].len : 0)});
  }
  std::stable_sort(its.begin(), its.end(), [](const It& x, const It& y) { return x.len > y.len; });
  items.assign(8 * its.size(), -1);
  for (size_t k = 0; k < its.size(); ++k) {
    const Pc& p = pc[its[k].a];
    int32_t* o = &items[8 * k];
    o[0] = p.t;
    o[1] = p.j0;
    o[2] = p.j1;
    o[3] = p.slot;
    if (its[k].b >= 0) {
      const Pc& q = pc[its[k].b];
      o[4] = q.t;
      o[5] = q.j0;
      o[6] = q.j1;
      o[7] = q.slot;
    } else {
      o[4] = -1;
      o[5] = o[6] = o[7] = 0;
    }
  }
  return mx;
}

template <int G>
static cudaError_t launch_pp_g(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                               const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                               cudaStream_t st) {
  const int n_items = a.n_work * a.Hkv;
  dim3 grid(std::min(n_items, n_sms));
  if (a.bdelta)
    CUDA_TRY_LAUNCH(launch_k(attn_pp_kernel<G, true>, grid, dim3(512), attn2::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  else
    CUDA_TRY_LAUNCH(launch_k(attn_pp_kernel<G, false>, grid, dim3(384), attn2::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  return cudaGetLastError();
}

template <int G>
static cudaError_t prepare_pp_g() {
  cudaError_t e = cudaFuncSetAttribute(attn_pp_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn2::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_pp_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn2::kSmem);
  return e;
}

cudaError_t prepare_attention_pp() {
  cudaError_t e = prepare_pp_g<1>();
  if (e == cudaSuccess) e = prepare_pp_g<2>();
  if (e == cudaSuccess) e = prepare_pp_g<4>();
  if (e == cudaSuccess) e = prepare_pp_g<8>();
  return e;
}

cudaError_t launch_attention_pp(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                                cudaStream_t st) {
  if (a.n_work <= 0) return cudaSuccess;
  switch (a.Hq / a.Hkv) {
    case 1: return launch_pp_g<1>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 2: return launch_pp_g<2>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 4: return launch_pp_g<4>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 8: return launch_pp_g<8>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pic
