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

#include "common.cuh"
#include "kernels.h"

namespace pic {

namespace attn {
constexpr int kTile = 16384;                 // one [128 rows][64 cols] bf16 SW128 half tile
constexpr int kQ = 0;                        // Q: 2 halves
constexpr int kK = kQ + 2 * kTile;           // K stages: 2 x 2 halves
constexpr int kV = kK + 4 * kTile;           // V stages
constexpr int kP = kV + 4 * kTile;           // P buffers: 2 x 2 halves
constexpr int kBar = kP + 4 * kTile;         // barriers
constexpr int kNumBars = 1 + 2 * 2 + 2 * 2 + 2 + 2 + 2;
constexpr int kSmem = kBar + kNumBars * 8 + 16 + 1024;
}  // namespace attn

template <int G>
__global__ void __launch_bounds__(192, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using namespace attn;
  constexpr int QPT = 128 / G;  // queries per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  const uint32_t base = smem_u32(smem);
  const uint32_t q_full = smem_u32(bars + 0);
  const uint32_t k_full = smem_u32(bars + 1), k_empty = smem_u32(bars + 3);
  const uint32_t v_full = smem_u32(bars + 5), v_empty = smem_u32(bars + 7);
  const uint32_t s_full = smem_u32(bars + 9), p_full = smem_u32(bars + 11), o_full = smem_u32(bars + 13);

  const int warp = warp_id(), lane = lane_id();
  const int tile = blockIdx.x, g = blockIdx.y, split = blockIdx.z;
  const int seq = a.tiles[3 * tile], row_start = a.tiles[3 * tile + 1], row_count = a.tiles[3 * tile + 2];

  // causal extent of this tile: keys 0..max_p (rows are sorted, but take the max anyway)
  int max_p = 0;
  for (int i = lane; i < row_count; i += 32) max_p = max(max_p, a.row_pos[row_start + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) max_p = max(max_p, __shfl_xor_sync(0xffffffffu, max_p, o));
  const int n_kv = max_p / 128 + 1;
  const int chunk = (n_kv + a.n_splits - 1) / a.n_splits;
  const int j0 = split * chunk, j1 = min(n_kv, j0 + chunk);
  const int n = max(0, j1 - j0);
  const int* bt = a.bt + a.seq_bt_off[seq];
  const int last_blk = max_p / 16;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(k_full + 8 * s, 1);
      mbar_init(k_empty + 8 * s, 1);
      mbar_init(v_full + 8 * s, 1);
      mbar_init(v_empty + 8 * s, 1);
      mbar_init(s_full + 8 * s, 1);
      mbar_init(p_full + 8 * s, 128);
      mbar_init(o_full + 8 * s, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0 && n > 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      mbar_expect_tx(q_full, 2 * kTile);
      for (int h = 0; h < 2; ++h) tma_load_3d(base + kQ + h * kTile, &tmQ, q_full, h * 64, g * G, row_start);
      const int kv_base = a.layer * a.num_blocks;
      for (int t = 0; t < n; ++t) {
        const int s = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        const int j = j0 + t;
        mbar_wait(k_empty + 8 * s, ph ^ 1);
        mbar_expect_tx(k_full + 8 * s, 2 * kTile);
        for (int b = 0; b < 8; ++b) {
          const int blk = bt[min(j * 8 + b, last_blk)];
          for (int h = 0; h < 2; ++h)
            tma_load_4d(base + kK + (2 * s + h) * kTile + b * 2048, &tmK, k_full + 8 * s, h * 64, 0, g, kv_base + blk);
        }
        mbar_wait(v_empty + 8 * s, ph ^ 1);
        mbar_expect_tx(v_full + 8 * s, 2 * kTile);
        for (int b = 0; b < 8; ++b) {
          const int blk = bt[min(j * 8 + b, last_blk)];
          for (int h = 0; h < 2; ++h)
            tma_load_4d(base + kV + (2 * s + h) * kTile + b * 2048, &tmV, v_full + 8 * s, h * 64, 0, g, kv_base + blk);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0 && n > 0) {
      constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K (K-major)
      constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (K-major) x V (MN-major)
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int u) {
        const int pb = u & 1;
        const uint32_t ph = (u >> 1) & 1;
        mbar_wait(p_full + 8 * pb, ph);
        mbar_wait(v_full + 8 * pb, ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t pa = base + kP + (2 * pb + (kk >> 2)) * kTile + (kk & 3) * 32;
          const uint32_t vb = base + kV + (2 * pb) * kTile + kk * 2048;  // 16 keys x 128 B
          umma_bf16(tmem + 256 + pb * 128, sdesc_sw128(pa, 16, 1024), sdesc_sw128(vb, kTile, 1024), idO, kk > 0);
        }
        umma_commit(o_full + 8 * pb);
        umma_commit(v_empty + 8 * pb);
      };
      for (int t = 0; t < n; ++t) {
        const int sb = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        mbar_wait(k_full + 8 * sb, ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qa = base + kQ + (kk >> 2) * kTile + (kk & 3) * 32;
          const uint32_t kb = base + kK + (2 * sb + (kk >> 2)) * kTile + (kk & 3) * 32;
          umma_bf16(tmem + sb * 128, sdesc_sw128(qa, 16, 1024), sdesc_sw128(kb, 16, 1024), idS, kk > 0);
        }
        umma_commit(s_full + 8 * sb);
        umma_commit(k_empty + 8 * sb);
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(n - 1);
    }
  } else {
    // ------------------------------------------------------------------ softmax warps
    const int q = warp & 3;
    const int r = q * 32 + lane;              // MMA row = TMEM lane
    const int qi = r / G, hh = r % G;
    const bool valid = qi < row_count;
    const int row = row_start + qi;
    const int head = g * G + hh;
    const int pos = valid ? a.row_pos[row] : max_p;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    float o[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) o[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int t = 0; t < n; ++t) {
      const int sb = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      const int key0 = (j0 + t) * 128;
      mbar_wait(s_full + 8 * sb, ph);
      tc_fence_after();
      const uint32_t sAddr = tmem + lane_addr + sb * 128;
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(sAddr + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (key0 + c * 32 + i <= pos) mx = fmaxf(mx, v[i] * a.scale_log2);
      }
      const float m_new = fmaxf(m, mx);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = exp2f(m - m_use);
      float sum = 0.f;
      uint8_t* pbuf = smem + kP + (2 * sb) * kTile + r * 128;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(sAddr + c * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int k = key0 + c * 32 + i;
          const float p0 = (k <= pos) ? exp2f(v[i] * a.scale_log2 - m_use) : 0.f;
          const float p1 = (k + 1 <= pos) ? exp2f(v[i + 1] * a.scale_log2 - m_use) : 0.f;
          sum += p0 + p1;
          pk[i / 2] = pack_bf16(p0, p1);
        }
        // 32 keys = 4 16-byte chunks; chunk index within the 64-key half, swizzled by row
        const int half = c >> 1;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int chunk16 = (c & 1) * 4 + cc;
          uint4* dst = reinterpret_cast<uint4*>(pbuf + half * kTile + ((chunk16 ^ (r & 7)) << 4));
          *dst = make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
        }
      }
      l = l * alpha + sum;
      m = m_new;
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full + 8 * sb);
      if (t >= 1) {
        const int ob = (t - 1) & 1;
        mbar_wait(o_full + 8 * ob, ((t - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(tmem + lane_addr + 256 + ob * 128 + c * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[c * 32 + i] += v[i];
        }
      }
#pragma unroll
      for (int i = 0; i < 128; ++i) o[i] *= alpha;
    }
    if (n > 0) {
      const int ob = (n - 1) & 1;
      mbar_wait(o_full + 8 * ob, ((n - 1) >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(tmem + lane_addr + 256 + ob * 128 + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c * 32 + i] += v[i];
      }
    }
    if (valid) {
      const size_t idx = ((size_t)split * a.M + row) * a.Hq + head;
      float4* dst = reinterpret_cast<float4*>(a.o_part + idx * 128);
#pragma unroll
      for (int i = 0; i < 32; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
      a.ml_part[2 * idx] = m;
      a.ml_part[2 * idx + 1] = l;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int G>
static cudaError_t launch_attn_g(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                 const AttnArgs& a, cudaStream_t st) {
  dim3 grid(a.n_tiles, a.Hkv, a.n_splits);
  attn_tc_kernel<G><<<grid, 192, attn::kSmem, st>>>(tmQ, tmK, tmV, a);
  return cudaGetLastError();
}

cudaError_t prepare_attention() {
  cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_tc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::kSmem);
  return e;
}

cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const AttnArgs& a, cudaStream_t st) {
  switch (a.Hq / a.Hkv) {
    case 1: return launch_attn_g<1>(tmQ, tmK, tmV, a, st);
    case 2: return launch_attn_g<2>(tmQ, tmK, tmV, a, st);
    case 4: return launch_attn_g<4>(tmQ, tmK, tmV, a, st);
    case 8: return launch_attn_g<8>(tmQ, tmK, tmV, a, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------------
// split-KV combine: one warp per (row, head); lane s holds split s's (m, l); cross-split max and
// sum are warp-shuffle reductions; each lane then merges 4 of the 128 output columns.
__global__ void attn_combine_kernel(const float* __restrict__ o_part, const float* __restrict__ ml_part,
                                    __nv_bfloat16* __restrict__ O, int M, int Hq, int n_splits) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= M * Hq) return;
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

cudaError_t launch_attn_combine(const float* o_part, const float* ml_part, void* O, int M, int Hq, int D,
                                int n_splits, cudaStream_t st) {
  if (D != 128 || n_splits > 32) return cudaErrorInvalidValue;
  const int warps = M * Hq;
  attn_combine_kernel<<<(warps + 7) / 8, 256, 0, st>>>(o_part, ml_part, reinterpret_cast<__nv_bfloat16*>(O), M, Hq,
                                                       n_splits);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// Generic-D SIMT attention for the tiny configs (D = 16/32/64, no TMA box fits): one warp per
// (row, head); lanes stride over keys; two passes (max, then exp/sum/PV) in fp32.
template <int D>
__global__ void attn_simt_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Kp,
                                 const __nv_bfloat16* __restrict__ Vp, const int32_t* __restrict__ row_seq,
                                 const int32_t* __restrict__ seq_bt_off, const int32_t* __restrict__ bt,
                                 const int32_t* __restrict__ row_pos, __nv_bfloat16* __restrict__ O, int M, int Hq,
                                 int Hkv, float scale) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= M * Hq) return;
  const int row = wid / Hq, head = wid % Hq;
  const int g = head * Hkv / Hq;
  const int pos = row_pos[row];
  const int* tb = bt + seq_bt_off[row_seq[row]];
  float q[D];
#pragma unroll
  for (int i = 0; i < D; ++i) q[i] = __bfloat162float(Q[((size_t)row * Hq + head) * D + i]);
  auto kv_off = [&](int key) -> size_t {
    const int blk = tb[key / 16];
    return (((size_t)blk * Hkv + g) * 16 + (key % 16)) * D;
  };
  float mx = -INFINITY;
  for (int key = lane; key <= pos; key += 32) {
    const __nv_bfloat16* kr = Kp + kv_off(key);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) s += q[i] * __bfloat162float(kr[i]);
    mx = fmaxf(mx, s * scale);
  }
  mx = warp_max(mx);
  float l = 0.f, o[D];
#pragma unroll
  for (int i = 0; i < D; ++i) o[i] = 0.f;
  for (int key = lane; key <= pos; key += 32) {
    const size_t off = kv_off(key);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) s += q[i] * __bfloat162float(Kp[off + i]);
    const float p = __expf(s * scale - mx);
    l += p;
#pragma unroll
    for (int i = 0; i < D; ++i) o[i] += p * __bfloat162float(Vp[off + i]);
  }
  l = warp_sum(l);
#pragma unroll
  for (int i = 0; i < D; ++i) o[i] = warp_sum(o[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < D; ++i) O[((size_t)row * Hq + head) * D + i] = __float2bfloat16(o[i] / l);
  }
}

cudaError_t launch_attention_simt(const void* Q, const void* Kpool_l, const void* Vpool_l, const int32_t* row_seq,
                                  const int32_t* seq_bt_off, const int32_t* bt, const int32_t* row_pos, void* O,
                                  int M, int Hq, int Hkv, int D, float scale, cudaStream_t st) {
  const int warps = M * Hq;
  dim3 grid((warps + 3) / 4), block(128);
  auto q = reinterpret_cast<const __nv_bfloat16*>(Q);
  auto k = reinterpret_cast<const __nv_bfloat16*>(Kpool_l);
  auto v = reinterpret_cast<const __nv_bfloat16*>(Vpool_l);
  auto o = reinterpret_cast<__nv_bfloat16*>(O);
  switch (D) {
    case 16: attn_simt_kernel<16><<<grid, block, 0, st>>>(q, k, v, row_seq, seq_bt_off, bt, row_pos, o, M, Hq, Hkv, scale); break;
    case 32: attn_simt_kernel<32><<<grid, block, 0, st>>>(q, k, v, row_seq, seq_bt_off, bt, row_pos, o, M, Hq, Hkv, scale); break;
    case 64: attn_simt_kernel<64><<<grid, block, 0, st>>>(q, k, v, row_seq, seq_bt_off, bt, row_pos, o, M, Hq, Hkv, scale); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace pic
