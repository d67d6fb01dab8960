// attention_decode.cu — f1 ("paged split-KV decode attention"): one query row per
// sequence over its paged linked cache, after link "proceeds to the decode stage".
//
// Same Eq. (1) as attention.cu (P:215 A = softmax(Q K_expᵀ · MASK), O = A V_exp; scale 1/√D, reading R3),
// for a q-tile of ONE query: the G query heads of kv-head g.  The prefill kernels put those G heads on
// 128 MMA rows and run a 128-row softmax per K tile for G useful rows; here the tile is TRANSPOSED so the
// keys fill the MMA rows and the softmax touches only the useful G × 128 scores:
//   Sᵀ[key][h] = K_tile · Q_gᵀ      tcgen05 M = 128 keys, N = 16 (G heads, zero-padded), K = 128 dims
//                                    A = the K tile (TMA, SW128 K-major), B = Q_g ([16][128] K-major smem)
//   Oᵀ[d][h]  += V_tileᵀ · Pᵀ        M = 128 dims, N = 16, K = 128 keys
//                                    A = the V tile read MN-major (the same smem tile), B = P ([16][128] keys)
// One softmax thread per key (TMEM lane); per-head max / sum are warp-shuffle reductions plus a 4-warp
// exchange; O stays in TMEM with the lazy (2^8) rescale of the prefill kernels.  Split-KV pieces from the
// host schedule (attn_schedule); split rows leave (m, l, O) partials for attn_combine, unsplit rows write
// normalised bf16 O.  The kernel is bound by streaming K/V from HBM (64 KB per 128-key tile).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

namespace pic {

namespace attnd {
constexpr int kTile = 16384;                  // one [128 keys][64 dims] bf16 SW128 half tile
constexpr int kStages = 3;                    // K and V ring depth (3 x 64 KB in flight per SM)
constexpr int kK = 0;
constexpr int kV = kK + kStages * 2 * kTile;
constexpr int kHalf16 = 16 * 128;             // [16 rows][64 elements] bf16 SW128 half (2 KB)
constexpr int kQ = kV + kStages * 2 * kTile;  // Q_g: [16 heads][128 dims], two halves
constexpr int kP = kQ + 2 * kHalf16;          // P: 2 buffers x [16 heads][128 keys], two halves each
constexpr int kRed = kP + 2 * 2 * kHalf16;    // [2 parity][2 (max, sum)][4 warps][16] fp32
// chunk-frame links (a.qrot): a second Q_g buffer and the raw q rows the frame rotation starts from
constexpr int kQ1 = kRed + 2 * 2 * 4 * 16 * 4;
constexpr int kQraw = kQ1 + 2 * kHalf16;
constexpr int kBar = kQraw + 2 * kHalf16;
// k/v full/empty, s_full[2], p_full[2], o_full[2], qd_full[2], qd_empty[2]
constexpr int kNumBars = 4 * kStages + 2 + 2 + 2 + 2 + 2;
constexpr int kSmem = kBar + kNumBars * 8 + 16;
static_assert(kSmem <= 232448, "decode attention smem over the 227 KB limit");
constexpr uint32_t kTmS = 0;   // Sᵀ double buffer: columns [0, 16), [16, 32)
constexpr uint32_t kTmO = 32;  // Oᵀ: columns [32, 48)
constexpr int kThreads = 256;  // warp 0 TMA, warp 1 MMA, warps 4-7 softmax + epilogue (TMEM lane quarter w % 4)
}  // namespace attnd

template <int G>
__global__ void __launch_bounds__(attnd::kThreads, 1)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap tmK8, const __grid_constant__ CUtensorMap tmV8,
                       const AttnArgs a) {
  static_assert(G >= 1 && G <= 16, "decode attention packs G <= 16 heads on N = 16");
  griddep_launch();
  using namespace attnd;
  constexpr int S = kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  const uint32_t base = smem_u32(smem);
  const uint32_t k_full = smem_u32(bars), k_empty = smem_u32(bars + S);
  const uint32_t v_full = smem_u32(bars + 2 * S), v_empty = smem_u32(bars + 3 * S);
  const uint32_t s_full = smem_u32(bars + 4 * S), p_full = smem_u32(bars + 4 * S + 2);
  const uint32_t o_full = smem_u32(bars + 4 * S + 4);
  const uint32_t qd_full = smem_u32(bars + 4 * S + 6), qd_empty = smem_u32(bars + 4 * S + 8);
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(k_full + 8 * s, 1);
      mbar_init(k_empty + 8 * s, 1);
      mbar_init(v_full + 8 * s, 1);
      mbar_init(v_empty + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + 8 * b, 1);
      mbar_init(p_full + 8 * b, 128);
      mbar_init(o_full + 8 * b, 1);
      mbar_init(qd_full + 8 * b, 2);   // a.qrot: warps 2-3 rotate each frame's Q_g
      mbar_init(qd_empty + 8 * b, 1);  // the frame's last S MMA
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 64);
  // work item: q-tile (one row), KV-tile range [j0, j1), split slot
  const int* wk = a.work + 4 * blockIdx.x;
  const int tile = wk[0], split = wk[3], g = blockIdx.y;
  const int seq = a.tiles[3 * tile], row = a.tiles[3 * tile + 1];
  griddep_wait();  // Q and this step's K/V row come from the upstream kernel
  const int pos = a.row_pos[row];
  const int n_kv = pos / 128 + 1;
  const int j0 = wk[1], j1 = min(n_kv, wk[2]);
  const int n = max(0, j1 - j0);
  const int* bt = a.bt + a.seq_bt_off[seq];
  const int last_blk = pos / 16;
  {
    // Q_g (G heads x 128 dims, bf16) into the SW128 K-major B tile; rows G..15 and P's pad rows are zero
    const int u = threadIdx.x, h = u >> 4, ci = u & 15, hf = ci >> 3, c = ci & 7;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (h < G)
      v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.Q) +
                                          ((size_t)row * a.Hq + g * G + h) * 128 + ci * 8);
    // chunk-frame links keep the raw rows: every frame's R(−Δ)·q is built from them
    sts128(base + (a.qrot ? kQraw : kQ) + hf * kHalf16 + h * 128 + ((c ^ (h & 7)) << 4), v);
    for (int i = u; i < 2 * 2 * kHalf16 / 16; i += kThreads) sts128(base + kP + 16 * i, make_uint4(0u, 0u, 0u, 0u));
    fence_async_smem();  // generic-proxy smem writes -> visible to the tcgen05.mma operand reads
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (K, V)
    if (n > 0) {
      if (lane == 0) {
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        tma_prefetch(&tmK8);
        tma_prefetch(&tmV8);
      }
      const int kv_base = a.layer * a.num_blocks;
      const int* vbt = a.vbt ? a.vbt + a.seq_bt_off[seq] : bt;
      auto load = [&](const CUtensorMap* t1, const CUtensorMap* t8, const int* tb, uint32_t dst, uint32_t full,
                      uint32_t empty, uint32_t ph, int j) {
        const int mine = lane < 8 ? tb[min(j * 8 + lane, last_blk)] : 0;
        const int b0 = __shfl_sync(0xffffffffu, mine, 0);
        const bool contig = __all_sync(0xffffffffu, lane >= 8 || mine == b0 + lane);
        int blk[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) blk[b] = __shfl_sync(0xffffffffu, mine, b);
        if (lane == 0) {
          mbar_wait(empty, ph ^ 1);
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
      for (int t = 0; t < n; ++t) {
        const int s = t % S;
        const uint32_t ph = (t / S) & 1;
        load(&tmK, &tmK8, bt, base + kK + 2 * s * kTile, k_full + 8 * s, k_empty + 8 * s, ph, j0 + t);
        load(&tmV, &tmV8, vbt, base + kV + 2 * s * kTile, v_full + 8 * s, v_empty + 8 * s, ph, j0 + t);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (whole warp, elect.sync)
    if (n > 0) {
      constexpr uint32_t idS = idesc_bf16(128, 16, 0, 0);  // K tile (K-major) x Q_g (K-major)
      constexpr uint32_t idO = idesc_bf16(128, 16, 1, 0);  // V tile read MN-major (dims) x P (K-major)
      const uint64_t dK0 = sdesc_sw128(base + kK, 16, 1024), dQ = sdesc_sw128(base + kQ, 16, 1024);
      const uint64_t dQ1 = sdesc_sw128(base + kQ1, 16, 1024);
      const int* bdq = a.qrot ? a.bdelta + a.seq_bt_off[seq] : nullptr;
      int fi = -1, fr_cur = 0, fr_next = bdq ? bdq[min(j0 * 8, last_blk)] : 0;
      const uint64_t dV0 = sdesc_sw128(base + kV, kTile, 1024), dP0 = sdesc_sw128(base + kP, 16, 1024);
      auto issue_pv = [&](int u) {
        const int pb = u & 1, s = u % S;
        mbar_wait(p_full + 8 * pb, (u >> 1) & 1);
        mbar_wait(v_full + 8 * s, (u / S) & 1);
        tc_fence_after();
        const uint64_t dv = dV0 + (uint64_t)(s * (2 * kTile / 16)), dp = dP0 + (uint64_t)(pb * (2 * kHalf16 / 16));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // keys 16kk..16kk+15: V rows 16kk.. (2 KB apart), P columns 16kk..
          umma_bf16_e(tmem + kTmO, dv + (uint64_t)(kk * 2048 / 16),
                      dp + (uint64_t)(((kk >> 2) * kHalf16 + (kk & 3) * 32) >> 4), idO, (u | kk) != 0);
        umma_commit_e(o_full + 8 * pb);
        umma_commit_e(v_empty + 8 * s);
      };
      for (int t = 0; t < n; ++t) {
        const int s = t % S, sb = t & 1;
        uint64_t dq = dQ;
        bool frame_end = false;
        if (bdq) {  // chunk-frame link: S = K·(R(−Δ)q)ᵀ with the Q_g buffer of this tile's frame
          const int fr = fr_next;
          fr_next = t + 1 < n ? bdq[min((j0 + t + 1) * 8, last_blk)] : fr;
          if (t == 0 || fr != fr_cur) {
            ++fi;
            mbar_wait(qd_full + 8 * (fi & 1), (fi >> 1) & 1);
          }
          fr_cur = fr;
          frame_end = t + 1 == n || fr_next != fr;
          dq = (fi & 1) ? dQ1 : dQ;
        }
        mbar_wait(k_full + 8 * s, (t / S) & 1);
        tc_fence_after();
        // Sᵀ(t) overwrites the buffer read by the softmax of t-2, whose P(t-2) the MMA warp waited for below
        const uint64_t dk = dK0 + (uint64_t)(s * (2 * kTile / 16));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dims 16kk..16kk+15 of both K-major operands
          umma_bf16_e(tmem + kTmS + 16 * sb, dk + (uint64_t)(((kk >> 2) * kTile + (kk & 3) * 32) >> 4),
                      dq + (uint64_t)(((kk >> 2) * kHalf16 + (kk & 3) * 32) >> 4), idS, kk > 0);
        umma_commit_e(s_full + 8 * sb);
        umma_commit_e(k_empty + 8 * s);
        if (frame_end) umma_commit_e(qd_empty + 8 * (fi & 1));  // this frame's Q_g buffer may be rewritten
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n - 1);
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------------ chunk-frame Q_g rotation (warps 2-3)
    // For every frame Δ along the KV range: R(−Δ)·q of the G head rows (NeoX pairs (j, j+64), fp32 rotation
    // of the bf16 q rounded to bf16 — the Q-side re-base arithmetic of the prefill kernels) from the raw rows
    // into the Q_g buffer of the frame's parity; rows G..15 stay zero.  Thread u: (row u>>3, chunk u&7) and
    // (row 8 + u>>3, chunk u&7).
    if (a.qrot && n > 0) {
      const int u = threadIdx.x - 64;
      const int* bdq = a.bdelta + a.seq_bt_off[seq];
      int fi = -1, fr_cur = 0;
      for (int t = 0; t < n; ++t) {
        const int fr = bdq[min((j0 + t) * 8, last_blk)];
        if (t > 0 && fr == fr_cur) continue;
        fr_cur = fr;
        ++fi;
        const int ad = fr < 0 ? -fr : fr;
        const float sg = fr < 0 ? 1.f : -1.f;  // R(−Δ): sin(−Δθ) = −sign(Δ)·sin(|Δ|θ)
        mbar_wait(qd_empty + 8 * (fi & 1), ((fi >> 1) & 1) ^ 1);  // the S MMAs of frame fi−2 are done
        const uint32_t qb = base + ((fi & 1) ? kQ1 : kQ);
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          const int h = (u >> 3) + 8 * k2, c = u & 7;
          const uint32_t off = (uint32_t)(h * 128 + ((c ^ (h & 7)) << 4));
          uint4 xa = lds128(base + kQraw + off), xb = lds128(base + kQraw + kHalf16 + off);
          if (fr != 0 && h < G) {
            const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + c * 8);
            const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + c * 8);
            const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
            const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            uint32_t a4[4] = {xa.x, xa.y, xa.z, xa.w}, b4[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a0 = __uint_as_float(a4[k] << 16), a1 = __uint_as_float(a4[k] & 0xFFFF0000u);
              const float b0 = __uint_as_float(b4[k] << 16), b1 = __uint_as_float(b4[k] & 0xFFFF0000u);
              float ra0, rb0, ra1, rb1;
              rebase_pair(a0, b0, cs[2 * k], sg * sn[2 * k], ra0, rb0);
              rebase_pair(a1, b1, cs[2 * k + 1], sg * sn[2 * k + 1], ra1, rb1);
              a4[k] = pack_bf16(ra0, ra1);
              b4[k] = pack_bf16(rb0, rb1);
            }
            xa = make_uint4(a4[0], a4[1], a4[2], a4[3]);
            xb = make_uint4(b4[0], b4[1], b4[2], b4[3]);
          }
          sts128(qb + off, xa);
          sts128(qb + kHalf16 + off, xb);
        }
        fence_async_smem();  // generic-proxy smem writes -> visible to the S MMAs' operand reads
        __syncwarp();
        if (lane == 0) mbar_arrive(qd_full + 8 * (fi & 1));
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax (one thread per key) + epilogue
    const int q = warp & 3;
    const int r = q * 32 + lane;                     // key within the tile = TMEM lane (also the epilogue's dim)
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + kRed);  // [parity][max | sum][4 warps][16]
    const float sc = a.scale_log2;
    float m_ref[G], l[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      m_ref[h] = -INFINITY;
      l[h] = 0.f;
    }
    for (int t = 0; t < n; ++t) {
      const int sb = t & 1;
      mbar_wait(s_full + 8 * sb, (t >> 1) & 1);
      tc_fence_after();
      float sv[16];
      tmem_ld16(tmem + lane_addr + kTmS + 16 * sb, sv);
      const bool valid = (j0 + t) * 128 + r <= pos;
      float* rm = red + sb * 128;  // max slots of this parity; sums at +64
#pragma unroll
      for (int h = 0; h < G; ++h) {
        sv[h] = valid ? sv[h] * sc : -INFINITY;  // log2 units (sc > 0)
        const float m = warp_max(sv[h]);
        if (lane == 0) rm[q * 16 + h] = m;
      }
      named_bar_sync(1, 128);
      bool need_any = false;
      float alpha[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float mt = fmaxf(fmaxf(rm[h], rm[16 + h]), fmaxf(rm[32 + h], rm[48 + h]));
        // lazy reference (FA4): raised only when the max grows by more than 2^8, so O and l are rescaled
        // rarely; every thread takes the same decision (identical inputs)
        const bool grow = mt > m_ref[h] + 8.f;
        alpha[h] = 1.f;
        if (grow) {
          if (m_ref[h] != -INFINITY) {
            alpha[h] = exp2f(m_ref[h] - mt);
            need_any = true;
          }
          m_ref[h] = mt;
        }
      }
      if (need_any) {
        // Oᵀ (this thread's row = dim r) times alpha per head column: every PV up to t-1 must have landed
        mbar_wait(o_full + 8 * ((t - 1) & 1), ((t - 1) >> 1) & 1);
        tc_fence_after();
        float ov[16];
        tmem_ld16(tmem + lane_addr + kTmO, ov);
        uint32_t ou[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) ou[h] = __float_as_uint(h < G ? ov[h] * alpha[h] : ov[h]);
        tmem_st16u_wait(tmem + lane_addr + kTmO, ou);
#pragma unroll
        for (int h = 0; h < G; ++h) l[h] *= alpha[h];
      }
      // p = 2^(s - m_ref) -> P[h][key r] (bf16, SW128 K-major: half r/64, row h, 16-B chunk (r%64)/8)
      const uint32_t pbase = base + kP + sb * 2 * kHalf16 + (r >> 6) * kHalf16;
      const int c = (r & 63) >> 3;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float p = ex2_approx(sv[h] - m_ref[h]);
        const __nv_bfloat16 pb = __float2bfloat16_rn(p);
        const uint32_t addr = pbase + h * 128 + ((c ^ (h & 7)) << 4) + (r & 7) * 2;
        asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(*reinterpret_cast<const unsigned short*>(&pb)) : "memory");
        const float ps = warp_sum(__bfloat162float(pb));  // the sum of what the PV MMA multiplies
        if (lane == 0) rm[64 + q * 16 + h] = ps;
      }
      fence_async_smem();
      named_bar_sync(1, 128);
#pragma unroll
      for (int h = 0; h < G; ++h) l[h] += (rm[64 + h] + rm[64 + 16 + h]) + (rm[64 + 32 + h] + rm[64 + 48 + h]);
      // consume every o_full phase (PV(t-1) has finished by now): no barrier phase completes unobserved
      if (t >= 1) mbar_wait(o_full + 8 * ((t - 1) & 1), ((t - 1) >> 1) & 1);
      tc_fence_before();
      mbar_arrive(p_full + 8 * sb);
    }
    // epilogue: thread r owns dim r of every head's output row
    const bool direct = a.row_nsplit[row] == 1;
    if (n > 0) {
      mbar_wait(o_full + 8 * ((n - 1) & 1), ((n - 1) >> 1) & 1);
      tc_fence_after();
      float ov[16];
      tmem_ld16(tmem + lane_addr + kTmO, ov);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const size_t orow = (size_t)row * a.Hq + g * G + h;
        if (direct)
          reinterpret_cast<__nv_bfloat16*>(a.O)[orow * 128 + r] = __float2bfloat16_rn(ov[h] / l[h]);
        else
          a.o_part[((size_t)split * a.M * a.Hq + orow) * 128 + r] = ov[h];
      }
    } else if (!direct) {
#pragma unroll
      for (int h = 0; h < G; ++h)
        a.o_part[((size_t)split * a.M * a.Hq + (size_t)row * a.Hq + g * G + h) * 128 + r] = 0.f;
    }
    if (!direct && r == 0) {
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const size_t idx = ((size_t)split * a.M + row) * a.Hq + g * G + h;
        a.ml_part[2 * idx] = m_ref[h];
        a.ml_part[2 * idx + 1] = l[h];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

template <int G>
static cudaError_t launch_dec_g(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmK8,
                                const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st) {
  CUDA_TRY_LAUNCH(launch_k(attn_decode_kernel<G>, dim3(a.n_work, a.Hkv), dim3(attnd::kThreads), attnd::kSmem, st, tmK,
                           tmV, tmK8, tmV8, a));
  return cudaGetLastError();
}

cudaError_t prepare_attention_decode() {
  cudaError_t e = cudaSuccess;
  for (auto k : {attn_decode_kernel<1>, attn_decode_kernel<2>, attn_decode_kernel<4>, attn_decode_kernel<8>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, attnd::kSmem);
  return e;
}

bool attention_decode_supported(int G) { return G == 1 || G == 2 || G == 4 || G == 8; }

cudaError_t launch_attention_decode(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmK8,
                                    const CUtensorMap& tmV8, const AttnArgs& a, cudaStream_t st) {
  if (a.n_work <= 0) return cudaSuccess;
  switch (a.Hq / a.Hkv) {
    case 1: return launch_dec_g<1>(tmK, tmV, tmK8, tmV8, a, st);
    case 2: return launch_dec_g<2>(tmK, tmV, tmK8, tmV8, a, st);
    case 4: return launch_dec_g<4>(tmK, tmV, tmK8, tmV8, a, st);
    case 8: return launch_dec_g<8>(tmK, tmV, tmK8, tmV8, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pic
