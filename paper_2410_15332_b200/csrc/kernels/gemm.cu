// gemm.cu — tcgen05 / TMEM / TMA GEMM for the projections of the recomputed rows.
//
//   P[split][m][n] = Σ_{k in split} A[m][k] · B[n][k]        (A = activations, B = weights [out][in])
//
// Used for a5 (x·W_qkvᵀ, "Q = EW_Q, K = EW_K, V = EW_V"), a7 (O·W_oᵀ, "O = A V_exp W_O"),
// a8 (gate/up and down projections) and a10 (LM head).  Only the k' recomputed rows enter
// (recomputation is O(k'), not O(N)).
//
// Warp roles (one CTA per SM, 192 threads):
//   warp 0      TMA producer: A tile [128 x 64] and B tile [BN x 64] per stage, SWIZZLE_128B
//   warp 1      MMA issuer:   4 x tcgen05.mma (M=128, N=BN, K=16) per stage, fp32 accumulator in TMEM
//   warps 2..5  epilogue:     tcgen05.ld 32x32b rows -> fp32 partial sums in HBM
// Split-K across blockIdx.z fills all 148 SMs when M is skinny (cfg2: M = k' = 128); the partials
// are summed by the fused epilogue kernels (RMSNorm / RoPE+scatter / SwiGLU / argmax), so the
// reduction order is fixed and the result deterministic.
#include <cuda.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

namespace pic {

__constant__ int c_weight_evict_first = 0;
__device__ __forceinline__ bool weight_evict_first() { return c_weight_evict_first != 0; }

enum { EPI_PARTIAL = 0, EPI_SWIGLU = 1, EPI_RESID = 2, EPI_QKV = 3 };

// EPI_QKV (split-K = 1, 128-column head tiles): a5's RoPE + scatter on the accumulator (P:213 steps
// 2-3, the qkv_rope_scatter arithmetic): Q heads rotated at p_row -> dense Q; K heads rotated -> pool
// slot of the row; V heads -> pool slot.  NeoX pairs (j, j+64) of a head sit in TMEM columns c and
// c + 64 of the same thread's row.
PIC_DEV void rope_pack16(const float* a, const float* b, const float* cs, const float* sn, uint4* oa, uint4* ob) {
  uint32_t pa[8], pb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float ra0, rb0, ra1, rb1;
    rope_pair(a[2 * j], b[2 * j], cs[2 * j], sn[2 * j], ra0, rb0);
    rope_pair(a[2 * j + 1], b[2 * j + 1], cs[2 * j + 1], sn[2 * j + 1], ra1, rb1);
    pa[j] = pack_bf16(ra0, ra1);
    pb[j] = pack_bf16(rb0, rb1);
  }
  oa[0] = make_uint4(pa[0], pa[1], pa[2], pa[3]);
  oa[1] = make_uint4(pa[4], pa[5], pa[6], pa[7]);
  ob[0] = make_uint4(pb[0], pb[1], pb[2], pb[3]);
  ob[1] = make_uint4(pb[4], pb[5], pb[6], pb[7]);
}

template <int BN, int STAGES, int CL = 1>
struct GemmSmem {
  static constexpr int kA = 128 * 64 * 2;  // 16 KB
  static constexpr int kB = (BN / CL) * 64 * 2;  // a CTA pair splits the N-tile: each CTA holds BN/2 rows of B
  static constexpr int kStage = kA + kB;
  static constexpr int kBars = 2 * STAGES + 4;
  static constexpr int kRing = STAGES * kStage + kBars * 8 + 16;
  // dedicated epilogue staging (4 warps x [32 rows][32 fp32]) when it fits beside the ring: every unit's
  // residual / partial stores leave as full 128-B row segments, not only the last unit's
  static constexpr int kStgOff = (kRing + 1023) / 1024 * 1024;
  static constexpr int kStg = (CL == 1 && kStgOff + 16384 <= 232448) ? 16384 : 0;
  static constexpr int kBytes = kStg ? kStgOff + kStg : kRing;
  static constexpr int kAcc = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;  // TMEM cols per accumulator
  static constexpr int kTmemCols = 2 * kAcc;                                              // double buffered
  static_assert(BN % 16 == 0 && BN <= 256, "UMMA N (M=128): multiple of 16, <= 256");
  static_assert(kBytes <= 232448, "GEMM smem over the 227 KB limit");
};

constexpr int gemm_stages(int bn, int cl = 1) {
  return (225 * 1024) / (16384 + bn / cl * 128) > 8 ? 8 : (225 * 1024) / (16384 + bn / cl * 128);
}

// Persistent tcgen05 GEMM.  Work units (m-tile, n-tile, k-split) are dealt round-robin to
// min(units, 148) CTAs; the smem ring runs continuously across units and the fp32 accumulator is
// double-buffered in TMEM, so the epilogue of unit i overlaps the MMAs of unit i+1.
//   EPI_PARTIAL: out = fp32 P[split][M][N] (summed by the consumer kernel in a fixed order).
//   EPI_SWIGLU (split-K = 1): B rows are W_gate/W_up interleaved in groups of BN/2 (n-tile = gate rows
//     [n·BN/2, (n+1)·BN/2) then the matching up rows); out = bf16 u[M][N/2] = silu(gate) ⊙ up
//     (the a8 SwiGLU fused into the GEMM epilogue; P:241 Llama-family MLP, reading R4).
// r of a fused-norm consumer row (1 when the A operand was normalised by the residual kernel)
PIC_DEV float norm_scale(const GemmEpi& ep, int row, int M) {
  if (!ep.ssq_in || row >= M) return 1.f;
  const float* p = ep.ssq_in + (size_t)row * kSsqStride;
  float s = 0.f;
  for (int t = 0; t < ep.ssq_in_n; ++t) s += p[t];
  return rsqrtf(s * ep.inv_d + ep.eps);
}

// Epilogue of one unit (m-tile rows of this CTA x one n-tile), shared by the one-CTA and the CTA-pair
// kernel: EPI_PARTIAL / EPI_RESID (+ fused-norm outputs) / EPI_QKV / EPI_SWIGLU on the accumulator rows
// this warp may read from TMEM (lane quarter q).  `last`: the CTA's final unit (its smem ring is idle).
template <int BN, int EPI, int KSTG, int KSTGOFF>
PIC_DEV void gemm_epilogue(uint8_t* smem, bool last, void* __restrict__ out_, int M, int N, int mt, int splits, int u,
                           int m0, int n_idx, int nkb, uint32_t tl, const GemmEpi& ep) {
  const int warp = warp_id(), lane = lane_id();
  const int q = warp & 3;
  const int row = m0 + q * 32 + lane;
  const int n0 = n_idx * BN;
      const bool stage = last || ((EPI == EPI_PARTIAL || EPI == EPI_RESID) && KSTG > 0);
      // the ring is idle after the last unit's MMAs; otherwise the dedicated 4 KB per warp (one chunk)
      uint8_t* stg = last ? smem + (size_t)(warp - 2) * ((BN + 31) / 32) * 4096
                          : smem + KSTGOFF + (size_t)(warp - 2) * 4096;
      const int stg_chunk = last ? 4096 : 0;  // bytes between consecutive 32-column chunks
      const int mrow0 = m0 + q * 32;
      if constexpr (EPI == EPI_PARTIAL || EPI == EPI_RESID) {
        // EPI_RESID (split-K = 1): out = the fp32 residual h, h += acc (the a7/a8 residual add: the same
        // fp32 addition the residual kernel applies to a single partial)
        const int sp = (u / mt) % splits;
        float* obase = reinterpret_cast<float*>(out_) + (size_t)sp * M * N;
        float* orow = obase + (size_t)row * N;
        const int ncol = min(BN, N - n0);  // multiple of 16
        // fused norm: xg = bf16(h_new · g) and Σ h_new² of this n-tile per row (EPI_RESID, ep.norm_gain set)
        const bool fnorm = EPI == EPI_RESID && ep.norm_gain != nullptr;
        auto put4 = [&](float* dst, float4 v, float4 h, float4 g, float& ss) {
          if constexpr (EPI == EPI_RESID) {
            v = make_float4(h.x + v.x, h.y + v.y, h.z + v.z, h.w + v.w);
            if (fnorm) {
              ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
              *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(ep.xg) + (dst - obase)) =
                  make_uint2(pack_bf16(v.x * g.x, v.y * g.y), pack_bf16(v.z * g.z, v.w * g.w));
            }
          }
          *reinterpret_cast<float4*>(dst) = v;
        };
        if (nkb > 0 && stage) {
          float ssr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // rows i * 4 + lane / 8 of this warp
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            float v[32];
            tmem_ld32(tl + c, v);
            __syncwarp();  // the previous chunk's reads of a reused staging buffer are done
            float4* sb = reinterpret_cast<float4*>(stg + (c / 32) * stg_chunk);  // [32 rows][8 float4], XOR-swizzled
#pragma unroll
            for (int j = 0; j < 8; ++j)
              sb[lane * 8 + (j ^ (lane & 7))] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __syncwarp();
            const int jj = lane & 7;
            const bool cok = c + 4 * jj < ncol;
            // all residual loads of the chunk first: the xg stores below may alias h as far as the
            // compiler knows, and would otherwise serialise every load behind the previous store
            float4 hv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = i * 4 + (lane >> 3);
              hv[i] = (EPI == EPI_RESID && mrow0 + r < M && cok)
                          ? *reinterpret_cast<const float4*>(obase + (size_t)(mrow0 + r) * N + n0 + c + 4 * jj)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const float4 gq = fnorm && cok ? *reinterpret_cast<const float4*>(ep.norm_gain + n0 + c + 4 * jj)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = i * 4 + (lane >> 3);
              if (mrow0 + r < M && cok)
                put4(obase + (size_t)(mrow0 + r) * N + n0 + c + 4 * jj, sb[r * 8 + (jj ^ (r & 7))], hv[i], gq, ssr[i]);
            }
          }
          if (fnorm) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              float t = ssr[i];
              t += __shfl_xor_sync(0xffffffffu, t, 1);
              t += __shfl_xor_sync(0xffffffffu, t, 2);
              t += __shfl_xor_sync(0xffffffffu, t, 4);
              const int r = i * 4 + (lane >> 3);
              if ((lane & 7) == 0 && mrow0 + r < M) ep.ssq[(size_t)(mrow0 + r) * kSsqStride + n_idx] = t;
            }
          }
        } else if (nkb > 0) {
          float ss = 0.f;
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            float v[32];
            tmem_ld32(tl + c, v);  // columns beyond BN are allocated (power-of-2 TMEM) and ignored
            if (row < M) {
              float4 hv[8], gq[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {  // loads first (see the staged path)
                const bool cok = c + 4 * j < ncol;
                hv[j] = EPI == EPI_RESID && cok ? *reinterpret_cast<const float4*>(orow + n0 + c + 4 * j)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                gq[j] = fnorm && cok ? *reinterpret_cast<const float4*>(ep.norm_gain + n0 + c + 4 * j)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (c + 4 * j < ncol)
                  put4(orow + n0 + c + 4 * j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]), hv[j],
                       gq[j], ss);
            }
          }
          if (fnorm && row < M) ep.ssq[(size_t)row * kSsqStride + n_idx] = ss;
        } else if (row < M && EPI == EPI_PARTIAL) {
          for (int col = n0; col < n0 + ncol; col += 4)
            *reinterpret_cast<float4*>(orow + col) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else if constexpr (EPI == EPI_QKV) {
        // every lane runs the (warp-collective) TMEM loads; rows beyond M only skip their stores
        const bool ok = row < M;
        const float rs = norm_scale(ep, row, M);  // fused RMSNorm row scale (1 if the input was normalised)
        const int p = ok ? ep.pos[row] : 0, sl = ok ? ep.slot[row] : 0;
        const int pk_ = ok && ep.kpos ? ep.kpos[row] : p;  // K heads: chunk-frame position (kv_share 3)
        const size_t kv_base = ((size_t)(sl / 16) * ep.Hkv) * 16 * 128 + (size_t)(sl % 16) * 128;
#pragma unroll 1
        for (int hh = 0; hh < BN / 128; ++hh) {
          const int hd = (n0 >> 7) + hh;  // warp-uniform
          if (hd >= ep.Hq + 2 * ep.Hkv) break;
          const uint32_t th = tl + hh * 128;
          if (hd < ep.Hq + ep.Hkv) {
            const int pr = hd < ep.Hq ? p : pk_;
            const float* cp = ep.cos_t + (size_t)pr * 64;
            const float* spn = ep.sin_t + (size_t)pr * 64;
            uint16_t* dst = hd < ep.Hq ? reinterpret_cast<uint16_t*>(ep.Q) + ((size_t)row * ep.Hq + hd) * 128
                                       : reinterpret_cast<uint16_t*>(ep.Kl) + kv_base + (size_t)(hd - ep.Hq) * 16 * 128;
#pragma unroll 1
            for (int c = 0; c < 64; c += 16) {
              float a[16], b[16], cs[16], sn[16];
              tmem_ld16(th + c, a);
              tmem_ld16(th + 64 + c, b);
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                a[j] *= rs;
                b[j] *= rs;
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 c4 = *reinterpret_cast<const float4*>(cp + c + 4 * j);
                const float4 s4 = *reinterpret_cast<const float4*>(spn + c + 4 * j);
                cs[4 * j] = c4.x, cs[4 * j + 1] = c4.y, cs[4 * j + 2] = c4.z, cs[4 * j + 3] = c4.w;
                sn[4 * j] = s4.x, sn[4 * j + 1] = s4.y, sn[4 * j + 2] = s4.z, sn[4 * j + 3] = s4.w;
              }
              uint4 oa[2], ob[2];
              rope_pack16(a, b, cs, sn, oa, ob);
              if (ok) {
                reinterpret_cast<uint4*>(dst + c)[0] = oa[0];
                reinterpret_cast<uint4*>(dst + c)[1] = oa[1];
                reinterpret_cast<uint4*>(dst + 64 + c)[0] = ob[0];
                reinterpret_cast<uint4*>(dst + 64 + c)[1] = ob[1];
              }
            }
          } else {
            uint16_t* dst = reinterpret_cast<uint16_t*>(ep.Vl) + kv_base + (size_t)(hd - ep.Hq - ep.Hkv) * 16 * 128;
#pragma unroll 1
            for (int c = 0; c < 128; c += 32) {
              float v[32];
              tmem_ld32(th + c, v);
              uint32_t pk[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j] * rs, v[2 * j + 1] * rs);
              if (ok)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  reinterpret_cast<uint4*>(dst + c)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
          }
        }
      } else {
        constexpr int G = BN / 2;
        constexpr int PR = G / 8;                 // 16-B pieces per row of the u tile
        constexpr int PS = PR | 1;                // odd smem row stride (in pieces): conflict-free
        const int F = N / 2;
        uint16_t* urow = reinterpret_cast<uint16_t*>(out_) + (size_t)row * F + (size_t)n_idx * G;
        uint4* sb = reinterpret_cast<uint4*>(stg);
        const float rs = norm_scale(ep, row, M);  // fused RMSNorm row scale (1 if the input was normalised)
#pragma unroll 1
        for (int c = 0; c < G; c += 16) {
          float gv[16], uv[16];
          tmem_ld16(tl + c, gv);
          tmem_ld16(tl + G + c, uv);
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float g0 = gv[2 * j] * rs, g1 = gv[2 * j + 1] * rs;
            pk[j] = pack_bf16(g0 / (1.f + __expf(-g0)) * (uv[2 * j] * rs), g1 / (1.f + __expf(-g1)) * (uv[2 * j + 1] * rs));
          }
          if (stage) {
            sb[lane * PS + c / 8] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            sb[lane * PS + c / 8 + 1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          } else if (row < M && n_idx * G + c < F) {
            uint4* dst = reinterpret_cast<uint4*>(urow + c);
            dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
        if (stage) {
          __syncwarp();
          uint16_t* ubase = reinterpret_cast<uint16_t*>(out_) + (size_t)n_idx * G;
#pragma unroll 1
          for (int p = lane; p < 32 * PR; p += 32) {
            const int r = p / PR, pc = p - r * PR;
            if (mrow0 + r < M && n_idx * G + pc * 8 < F)
              *reinterpret_cast<uint4*>(ubase + (size_t)(mrow0 + r) * F + pc * 8) = sb[r * PS + pc];
          }
        }
      }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     void* __restrict__ out_, int M, int N, int kblk_total, int kblk_per_split, int splits,
                     int pack, unsigned long long* trace, const __grid_constant__ CUtensorMap tmN,
                     GemmNext nx, const GemmEpi ep) {
  using S = GemmSmem<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::kA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::kBars);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

  const int warp = warp_id(), lane = lane_id();
  const int mt = (M + 127) / 128, nt = (N + BN - 1) / BN;
  const int units = mt * nt * splits;
  griddep_launch();
  if (trace && threadIdx.x == 0) trace[blockIdx.x * 6 + 0] = globaltimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // unit u -> (m fastest, then split, then n): concurrently running CTAs share weight tiles in L2.  With
  // ep.raster_gm > 0 (split-K 1, A larger than L2 wants) the m-tiles go in groups of raster_gm, each group
  // sweeping all n-tiles before the next: one wave reuses raster_gm A row-blocks and 148 / raster_gm
  // weight n-tiles from L2 instead of streaming all of A once per n-tile band.
  const int GM = (ep.raster_gm > 0 && splits == 1) ? min(ep.raster_gm, mt) : mt;
  auto decode = [&](int u, int& m0, int& n_idx, int& kb0, int& nkb) {
    const int grp = u / (GM * nt * splits);
    const int mb = grp * GM, gme = min(GM, mt - mb);
    const int v = u - grp * GM * nt * splits;
    const int m = mb + v % gme;
    const int r = v / gme;
    const int sp = r % splits;
    n_idx = r / splits;
    m0 = m * 128;
    kb0 = sp * kblk_per_split;
    nkb = max(0, min(kblk_per_split, kblk_total - kb0));
  };

  // B tile of k-block kb: row-major weights -> one [BN x 64] box; packed weights (pack rows per
  // sub-tile, stored [N/pack][K/64][pack][64]) -> BN/pack contiguous boxes of pack x 128 B.
  const uint64_t wpol = l2_policy_evict_first();  // weights are streamed once per forward
  auto load_b = [&](uint32_t dst, uint32_t bar, int kb, int n_idx) {
    if (pack == 0) {
      if (weight_evict_first())
        tma_load_2d_hint(dst, &tmB, bar, kb * 64, n_idx * BN, wpol);
      else
        tma_load_2d(dst, &tmB, bar, kb * 64, n_idx * BN);
    } else {
      const int per = BN / pack;
      for (int j = 0; j < per; ++j) {
        const int t = n_idx * per + j;
        tma_load_2d(dst + j * pack * 128, &tmB, bar, 0, (t * kblk_total + kb) * pack);
      }
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      int it = 0;
      bool waited = false;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int m0, n_idx, kb0, nkb;
        decode(u, m0, n_idx, kb0, nkb);
        int kk = 0;
        if (!waited) {
          // Weights do not depend on the previous kernel: stream the first stages of B while it
          // drains (PDL), then wait for it before loading the activations A.
          const int pre = min(nkb, STAGES);
          for (int i = 0; i < pre; ++i) {
            mbar_expect_tx(full0 + 8 * i, S::kStage);
            load_b(smem_u32(sB + i * S::kB), full0 + 8 * i, kb0 + i, n_idx);
          }
          griddep_wait();
          if (trace) trace[blockIdx.x * 6 + 1] = globaltimer();
          waited = true;
          for (int i = 0; i < pre; ++i) tma_load_2d(smem_u32(sA + i * S::kA), &tmA, full0 + 8 * i, (kb0 + i) * 64, m0);
          kk = pre;
          it = pre;
        }
        for (; kk < nkb; ++kk, ++it) {
          const int s = it % STAGES;
          mbar_wait(empty0 + 8 * s, ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(full0 + 8 * s, S::kStage);
          const int kc = (kb0 + kk) * 64;
          tma_load_2d(smem_u32(sA + s * S::kA), &tmA, full0 + 8 * s, kc, m0);
          load_b(smem_u32(sB + s * S::kB), full0 + 8 * s, kb0 + kk, n_idx);
        }
      }
      if (!waited) griddep_wait();
      // All of this GEMM's loads are issued: pull the first k-blocks of the NEXT GEMM's weights into
      // L2 so that its ring fill (at its launch) hits L2 instead of waiting on HBM.
      for (int u2 = blockIdx.x; u2 < nx.units && nx.pfk > 0; u2 += gridDim.x) {
        const int r2 = u2 / nx.mt;
        if (u2 % nx.mt) continue;  // same weights for every m-tile
        const int kb2 = (r2 % nx.splits) * nx.kper, n2 = r2 / nx.splits;
        const int nk2 = min(nx.pfk, nx.kblk_total - kb2);
        for (int i = 0; i < nk2; ++i) tma_prefetch_l2_2d(&tmN, (kb2 + i) * 64, n2 * nx.bn);
      }
    }
  } else if (warp == 1) {
    {
      // whole warp, elect.sync issue, base descriptors + constant offsets (a lane-0 branch recomputing
      // descriptors per MMA issues at ~88 cycles per MMA: above the pipe time of N <= 224)
      constexpr uint32_t idesc = idesc_bf16(128, BN, 0, 0);
      const uint64_t dA0 = sdesc_sw128(smem_u32(sA), 16, 1024), dB0 = sdesc_sw128(smem_u32(sB), 16, 1024);
      int it = 0, i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        int m0, n_idx, kb0, nkb;
        decode(u, m0, n_idx, kb0, nkb);
        const int ab = i & 1;
        mbar_wait(tempty0 + 8 * ab, ((i >> 1) & 1) ^ 1);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + ab * S::kAcc;
        for (int kk = 0; kk < nkb; ++kk, ++it) {
          const int s = it % STAGES;
          mbar_wait(full0 + 8 * s, (it / STAGES) & 1);
          if (trace && it == 0 && lane == 0) trace[blockIdx.x * 6 + 2] = globaltimer();
          tc_fence_after();
          const uint64_t da = dA0 + (uint64_t)(s * (S::kA / 16)), db = dB0 + (uint64_t)(s * (S::kB / 16));
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) umma_bf16_e(d, da + 2 * k4, db + 2 * k4, idesc, (kk | k4) != 0);
          umma_commit_e(empty0 + 8 * s);
        }
        umma_commit_e(tfull0 + 8 * ab);
      }
      if (trace && lane == 0) trace[blockIdx.x * 6 + 3] = globaltimer();
    }
  } else {
    griddep_wait();  // `out` may still be read by the previous kernel
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      int m0, n_idx, kb0, nkb;
      decode(u, m0, n_idx, kb0, nkb);
      const int ab = i & 1;
      const uint32_t tl = tmem + ab * S::kAcc + ((uint32_t)(q * 32) << 16);
      mbar_wait(tfull0 + 8 * ab, (i >> 1) & 1);
      tc_fence_after();
      // The last unit of a CTA runs after its final MMA, when the smem ring is idle: stage the tile
      // through the ring so that global stores are full 128-B row segments (a row-per-thread store
      // pattern costs ~4 us per tile in uncoalesced 16-B transactions).
      gemm_epilogue<BN, EPI, S::kStg, S::kStgOff>(smem, u + (int)gridDim.x >= units, out_, M, N, mt, splits, u, m0,
                                                   n_idx, nkb, tl, ep);
      tc_fence_before();
      mbar_arrive(tempty0 + 8 * ab);
      if (trace && threadIdx.x == 64 && u + (int)gridDim.x >= units) trace[blockIdx.x * 6 + 4] = globaltimer();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, S::kTmemCols);
  }
}

// The one-CTA kernel above and the CTA-pair kernel below share their structure; they are kept as two
// kernels because folding the pair path into the one-CTA kernel as a template parameter changed ptxas'
// register allocation of the one-CTA instances (96 -> 123 registers, +17% instructions) and cost 4% on
// cfg3 end to end (same-box A/B, scripts/ab_lib.sh).
// CTA-pair GEMM (cta_group::2, CL = 2; CL = 1 compiles but is not instantiated).  A unit is a 256-row M-tile: each CTA of the pair loads its 128 rows of A
// and half of the N-tile's B rows into its own smem; the leader CTA issues M = 256 MMAs that read both
// CTAs' smem and write each CTA's 128 accumulator rows into its own TMEM; both CTAs' loads complete on the
// leader's full barrier, the MMA commits are multicast to both CTAs' empty / accumulator-full barriers,
// and both epilogues release the accumulator on the leader's tempty barrier.  Per SM this halves the B
// bytes staged and read by the tensor core per FLOP (the operand traffic that bounds one-CTA M = 128).
template <int BN, int STAGES, int EPI, int CL = 2>
__global__ void __launch_bounds__(192, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     void* __restrict__ out_, int M, int N, int kblk_total, int kblk_per_split, int splits,
                     int pack, unsigned long long* trace, const __grid_constant__ CUtensorMap tmN,
                     GemmNext nx, const GemmEpi ep) {
  using S = GemmSmem<BN, STAGES, CL>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::kA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::kBars);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

  const int warp = warp_id(), lane = lane_id();
  uint32_t rank = 0;
  int cid = blockIdx.x, ncl = gridDim.x;  // cluster (CTA pair) id / count
  if constexpr (CL == 2) {
    rank = cluster_ctarank();
    cid = blockIdx.x / 2;
    ncl = gridDim.x / 2;
  }
  const int mt = (M + 128 * CL - 1) / (128 * CL), nt = (N + BN - 1) / BN;
  const int units = mt * nt * splits;
  griddep_launch();
  if (trace && threadIdx.x == 0) trace[blockIdx.x * 6 + 0] = globaltimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, 128 * CL);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CL == 2)
      tmem_alloc_2sm(smem_u32(tmem_slot), S::kTmemCols);
    else
      tmem_alloc(smem_u32(tmem_slot), S::kTmemCols);
  }
  tc_fence_before();
  if constexpr (CL == 2)
    cluster_sync();  // barrier inits and TMEM allocations of both CTAs visible before any cross-CTA use
  // (also a CTA barrier for the pair: compute-sanitizer's racecheck does not treat the cluster barrier as
  // ordering the allocator's smem write of the TMEM address against the read below)
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the leader's accumulator-empty barriers (both CTAs' epilogues release the pair's accumulator there)
  const uint32_t temptyL = CL == 2 ? mapa_shared(tempty0, 0) : tempty0;

  // unit u -> (m fastest, then split, then n): concurrently running CTAs share weight tiles in L2
  auto decode = [&](int u, int& m0, int& n_idx, int& kb0, int& nkb) {
    const int m = u % mt;
    const int r = u / mt;
    const int sp = r % splits;
    n_idx = r / splits;
    if constexpr (CL == 1)
      m0 = m * 128;
    else
      m0 = m * 128 * CL + (int)rank * 128;  // this CTA's 128 rows
    kb0 = sp * kblk_per_split;
    nkb = max(0, min(kblk_per_split, kblk_total - kb0));
  };

  // B tile of k-block kb: row-major weights -> one [BN x 64] box; packed weights (pack rows per
  // sub-tile, stored [N/pack][K/64][pack][64]) -> BN/pack contiguous boxes of pack x 128 B.
  const uint64_t wpol = l2_policy_evict_first();  // weights are streamed once per forward
  auto load_b = [&](uint32_t dst, uint32_t bar, int kb, int n_idx) {
    if constexpr (CL == 2) {
      tma_load_2d_2sm(dst, &tmB, bar, kb * 64, n_idx * BN + (int)rank * (BN / 2),
                      weight_evict_first() ? wpol : l2_policy_evict_normal());
      return;
    }
    if (pack == 0) {
      if (weight_evict_first())
        tma_load_2d_hint(dst, &tmB, bar, kb * 64, n_idx * BN, wpol);
      else
        tma_load_2d(dst, &tmB, bar, kb * 64, n_idx * BN);
    } else {
      const int per = BN / pack;
      for (int j = 0; j < per; ++j) {
        const int t = n_idx * per + j;
        tma_load_2d(dst + j * pack * 128, &tmB, bar, 0, (t * kblk_total + kb) * pack);
      }
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      int it = 0;
      bool waited = false;
      if constexpr (CL == 1) {
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
          int m0, n_idx, kb0, nkb;
          decode(u, m0, n_idx, kb0, nkb);
          int kk = 0;
          if (!waited) {
            // Weights do not depend on the previous kernel: stream the first stages of B while it
            // drains (PDL), then wait for it before loading the activations A.
            const int pre = min(nkb, STAGES);
            for (int i = 0; i < pre; ++i) {
              mbar_expect_tx(full0 + 8 * i, S::kStage);
              load_b(smem_u32(sB + i * S::kB), full0 + 8 * i, kb0 + i, n_idx);
            }
            griddep_wait();
            if (trace) trace[blockIdx.x * 6 + 1] = globaltimer();
            waited = true;
            for (int i = 0; i < pre; ++i) tma_load_2d(smem_u32(sA + i * S::kA), &tmA, full0 + 8 * i, (kb0 + i) * 64, m0);
            kk = pre;
            it = pre;
          }
          for (; kk < nkb; ++kk, ++it) {
            const int s = it % STAGES;
            mbar_wait(empty0 + 8 * s, ((it / STAGES) & 1) ^ 1);
            mbar_expect_tx(full0 + 8 * s, S::kStage);
            const int kc = (kb0 + kk) * 64;
            tma_load_2d(smem_u32(sA + s * S::kA), &tmA, full0 + 8 * s, kc, m0);
            load_b(smem_u32(sB + s * S::kB), full0 + 8 * s, kb0 + kk, n_idx);
          }
        }
      } else {
        // A pair's loads complete on the leader's full barrier, which alone expects both CTAs' bytes
        const uint64_t apol = l2_policy_evict_normal();
        const uint32_t fullL = mapa_shared(full0, 0);
        for (int u = cid; u < units; u += ncl) {
          int m0, n_idx, kb0, nkb;
          decode(u, m0, n_idx, kb0, nkb);
          int kk = 0;
          if (!waited) {
            const int pre = min(nkb, STAGES);
            for (int i = 0; i < pre; ++i) {
              if (rank == 0) mbar_expect_tx(full0 + 8 * i, S::kStage * CL);
              load_b(smem_u32(sB + i * S::kB), fullL + 8 * i, kb0 + i, n_idx);
            }
            griddep_wait();
            waited = true;
            for (int i = 0; i < pre; ++i)
              tma_load_2d_2sm(smem_u32(sA + i * S::kA), &tmA, fullL + 8 * i, (kb0 + i) * 64, m0, apol);
            kk = pre;
            it = pre;
          }
          for (; kk < nkb; ++kk, ++it) {
            const int s = it % STAGES;
            mbar_wait(empty0 + 8 * s, ((it / STAGES) & 1) ^ 1);
            if (rank == 0) mbar_expect_tx(full0 + 8 * s, S::kStage * CL);
            tma_load_2d_2sm(smem_u32(sA + s * S::kA), &tmA, fullL + 8 * s, (kb0 + kk) * 64, m0, apol);
            load_b(smem_u32(sB + s * S::kB), fullL + 8 * s, kb0 + kk, n_idx);
          }
        }
      }
      if (!waited) griddep_wait();
      // All of this GEMM's loads are issued: pull the first k-blocks of the NEXT GEMM's weights into
      // L2 so that its ring fill (at its launch) hits L2 instead of waiting on HBM.
      for (int u2 = blockIdx.x; u2 < nx.units && nx.pfk > 0; u2 += gridDim.x) {
        const int r2 = u2 / nx.mt;
        if (u2 % nx.mt) continue;  // same weights for every m-tile
        const int kb2 = (r2 % nx.splits) * nx.kper, n2 = r2 / nx.splits;
        const int nk2 = min(nx.pfk, nx.kblk_total - kb2);
        for (int i = 0; i < nk2; ++i) tma_prefetch_l2_2d(&tmN, (kb2 + i) * 64, n2 * nx.bn);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // a pair's MMAs are issued by the leader CTA: whole warp, elect.sync issue
      constexpr uint32_t idesc = idesc_bf16(128 * CL, BN, 0, 0);
      const uint64_t dA0 = sdesc_sw128(smem_u32(sA), 16, 1024), dB0 = sdesc_sw128(smem_u32(sB), 16, 1024);
      int it = 0, i = 0;
      for (int u = cid; u < units; u += ncl, ++i) {
        int m0, n_idx, kb0, nkb;
        decode(u, m0, n_idx, kb0, nkb);
        const int ab = i & 1;
        mbar_wait(tempty0 + 8 * ab, ((i >> 1) & 1) ^ 1);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + ab * S::kAcc;
        for (int kk = 0; kk < nkb; ++kk, ++it) {
          const int s = it % STAGES;
          mbar_wait(full0 + 8 * s, (it / STAGES) & 1);
          if (trace && it == 0 && lane == 0) trace[blockIdx.x * 6 + 2] = globaltimer();
          tc_fence_after();
          const uint64_t da = dA0 + (uint64_t)(s * (S::kA / 16)), db = dB0 + (uint64_t)(s * (S::kB / 16));
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            if constexpr (CL == 2)
              umma_bf16_2sm_e(d, da + 2 * k4, db + 2 * k4, idesc, (kk | k4) != 0);
            else
              umma_bf16_e(d, da + 2 * k4, db + 2 * k4, idesc, (kk | k4) != 0);
          }
          if constexpr (CL == 2)
            umma_commit_2sm_e(empty0 + 8 * s, 3);
          else
            umma_commit_e(empty0 + 8 * s);
        }
        if constexpr (CL == 2)
          umma_commit_2sm_e(tfull0 + 8 * ab, 3);
        else
          umma_commit_e(tfull0 + 8 * ab);
      }
      if (trace && lane == 0) trace[blockIdx.x * 6 + 3] = globaltimer();
    }
  } else {
    griddep_wait();  // `out` may still be read by the previous kernel
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int i = 0;
    for (int u = cid; u < units; u += ncl, ++i) {
      int m0, n_idx, kb0, nkb;
      decode(u, m0, n_idx, kb0, nkb);
      const int ab = i & 1;
      const uint32_t tl = tmem + ab * S::kAcc + ((uint32_t)(q * 32) << 16);
      mbar_wait(tfull0 + 8 * ab, (i >> 1) & 1);
      tc_fence_after();
      gemm_epilogue<BN, EPI, 0, 0>(smem, u + ncl >= units, out_, M, N, mt, splits, u, m0, n_idx, nkb, tl, ep);
      tc_fence_before();
      if constexpr (CL == 2)
        mbar_arrive_cluster(temptyL + 8 * ab);  // the leader's MMA reuses the pair's accumulator
      else
        mbar_arrive(tempty0 + 8 * ab);
      if (trace && threadIdx.x == 64 && u + (int)gridDim.x >= units) trace[blockIdx.x * 6 + 4] = globaltimer();
    }
  }
  tc_fence_before();
  if constexpr (CL == 2)
    cluster_sync();  // every MMA into either CTA's TMEM has been consumed by its epilogue
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CL == 2)
      tmem_dealloc_2sm(tmem, S::kTmemCols);
    else
      tmem_dealloc(tmem, S::kTmemCols);
  }
}

// Bench-only per-CTA timeline (globaltimer ns): entry, after griddepcontrol.wait, first full stage,
// last MMA commit, last epilogue store.  Null in the engine.
unsigned long long* g_gemm_trace = nullptr;

GemmNext gemm_next(const CUtensorMap* B, int M, int N, int K, int splits, int bn, int pfk) {
  GemmNext nx{};
  if (!B || pfk <= 0) return nx;
  nx.tm = B;
  nx.mt = (M + 127) / 128;
  nx.splits = splits;
  nx.kblk_total = K / 64;
  nx.kper = (nx.kblk_total + splits - 1) / splits;
  nx.bn = bn;
  nx.units = ((N + bn - 1) / bn) * nx.mt * splits;
  nx.pfk = pfk;
  return nx;
}

template <int BN, int EPI, int CL = 1>
static cudaError_t launch_gemm_t(const CUtensorMap& A, const CUtensorMap& B, void* out, int M, int N, int K, int splits,
                                 int pack, cudaStream_t st, const GemmNext& nx, const GemmEpi& ep = GemmEpi{}) {
  constexpr int ST = gemm_stages(BN, CL);
  using S = GemmSmem<BN, ST, CL>;
  auto kern = [] {
    if constexpr (CL == 1)
      return gemm_bf16_kernel<BN, ST, EPI>;
    else
      return gemm_pair_kernel<BN, ST, EPI, CL>;
  }();
  const int kblk = K / 64;
  const int per = (kblk + splits - 1) / splits;
  const int units = ((N + BN - 1) / BN) * ((M + 128 * CL - 1) / (128 * CL)) * splits;
  const int max_cl = 148 / CL;
  const int grid = CL * (units < max_cl ? units : max_cl);  // persistent: one CTA (pair) per SM (pair)
  if constexpr (CL == 1) {
    GemmEpi e2 = ep;
    if (splits == 1 && e2.raster_gm == 0) {
      // traffic of a wave order with groups of gm m-tiles: A·(nt·gm/148) + B·(mt/gm); when A fits in L2
      // beside the weight tiles (< 64 MB) the plain m-fastest order already reads it once
      const double a_mb = (double)M * K * 2 / 1e6, b_mb = (double)N * K * 2 / 1e6;
      const int mt = (M + 127) / 128, nt = (N + BN - 1) / BN;
      if (a_mb > 64.0 && mt > 1) {
        const double g = std::sqrt(b_mb * mt * 148.0 / (a_mb * nt));
        e2.raster_gm = std::max(1, std::min(mt, (int)(g + 0.5)));
      }
    }
    CUDA_TRY_LAUNCH(launch_k(kern, dim3(grid), dim3(192), S::kBytes, st, A, B, out, M, N, kblk, per, splits, pack,
                             g_gemm_trace, nx.tm ? *nx.tm : B, nx, e2));
  } else {
    if (pack) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = S::kBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 2;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    unsigned long long* tr = nullptr;
    const CUtensorMap tn = nx.tm ? *nx.tm : B;
    CUDA_TRY_LAUNCH(cudaLaunchKernelEx(&cfg, kern, A, B, out, M, N, kblk, per, splits, pack, tr, tn, nx, ep));
  }
  return cudaGetLastError();
}

template <int BN, int EPI, int CL = 1>
static cudaError_t prep_t() {
  constexpr int ST = gemm_stages(BN, CL);
  if constexpr (CL == 2)
    return cudaFuncSetAttribute(gemm_pair_kernel<BN, ST, EPI, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmSmem<BN, ST, CL>::kBytes);
  else
    return cudaFuncSetAttribute(gemm_bf16_kernel<BN, ST, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmSmem<BN, ST>::kBytes);
}

#define PIC_GEMM_BNS(X) X(64) X(128) X(144) X(160) X(176) X(192) X(208) X(224) X(256)
#define PIC_SWIGLU_BNS(X) X(32) X(64) X(128) X(224) X(256)
// CTA-pair (cta_group::2) instantiations: N-tiles of the tensor-bound multi-m-tile GEMMs
#define PIC_PAIR_BNS(X) X(128) X(192) X(224) X(256)
// fused-epilogue instantiations: residual add (any multi-m-tile N-tile), RoPE + scatter (whole heads)
#define PIC_RESID_BNS(X) X(128) X(144) X(160) X(176) X(192) X(208) X(224) X(256)
#define PIC_QKV_BNS(X) X(128) X(256)

cudaError_t prepare_gemm() {
  cudaError_t e = cudaSuccess;
  // weights are streamed once per forward: load them with an L2 evict-first policy so that the
  // activations, split-K partials and K/V pages the consumers re-read stay resident (cfg2 4.33 -> 4.18 ms)
  const int ef = getenv("PIC_WEIGHT_EVICT_FIRST") ? atoi(getenv("PIC_WEIGHT_EVICT_FIRST")) : 1;
  e = cudaMemcpyToSymbol(c_weight_evict_first, &ef, sizeof(int));
#define P1(bn) \
  if (e == cudaSuccess) e = prep_t<bn, EPI_PARTIAL>();
#define P2(bn) \
  if (e == cudaSuccess) e = prep_t<bn, EPI_SWIGLU>();
  PIC_GEMM_BNS(P1)
  PIC_SWIGLU_BNS(P2)
#undef P1
#undef P2
#define P4(bn) \
  if (e == cudaSuccess) e = prep_t<bn, EPI_RESID>();
#define P5(bn) \
  if (e == cudaSuccess) e = prep_t<bn, EPI_QKV>();
  PIC_RESID_BNS(P4)
  PIC_QKV_BNS(P5)
#undef P4
#undef P5
#define P3(bn)                                                   \
  if (e == cudaSuccess) e = prep_t<bn, EPI_PARTIAL, 2>();        \
  if (e == cudaSuccess) e = prep_t<bn, EPI_SWIGLU, 2>();         \
  if (e == cudaSuccess) e = prep_t<bn, EPI_RESID, 2>();
  PIC_PAIR_BNS(P3)
#undef P3
  if (e == cudaSuccess) e = prep_t<128, EPI_QKV, 2>();
  if (e == cudaSuccess) e = prep_t<256, EPI_QKV, 2>();
  return e;
}

bool gemm_pair_supported(int bn) {
#define C1(b) || bn == b
  return false PIC_PAIR_BNS(C1);
#undef C1
}

bool gemm_resid_supported(int bn) {
#define C1(b) || bn == b
  return false PIC_RESID_BNS(C1);
#undef C1
}

cudaError_t launch_gemm_resid(const CUtensorMap& A, const CUtensorMap& B, float* h, int M, int N, int K, int bn,
                              cudaStream_t st, const GemmNext& nx, const GemmEpi& ep, int pair) {
  if (ep.norm_gain && (N + bn - 1) / bn > kSsqStride) return cudaErrorInvalidValue;
  if (pair) {
    switch (bn) {
#define L7(b) \
  case b:     \
    return launch_gemm_t<b, EPI_RESID, 2>(A, B, h, M, N, K, 1, 0, st, nx, ep);
      PIC_PAIR_BNS(L7)
#undef L7
    }
    return cudaErrorInvalidValue;
  }
  switch (bn) {
#define L5(b) \
  case b:     \
    return launch_gemm_t<b, EPI_RESID>(A, B, h, M, N, K, 1, 0, st, nx, ep);
    PIC_RESID_BNS(L5)
#undef L5
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm_qkv(const CUtensorMap& A, const CUtensorMap& B, const GemmEpi& ep, int M, int N, int K, int bn,
                            cudaStream_t st, const GemmNext& nx, int pair) {
  if (pair) {
    if (bn == 128) return launch_gemm_t<128, EPI_QKV, 2>(A, B, nullptr, M, N, K, 1, 0, st, nx, ep);
    if (bn == 256) return launch_gemm_t<256, EPI_QKV, 2>(A, B, nullptr, M, N, K, 1, 0, st, nx, ep);
    return cudaErrorInvalidValue;
  }
  switch (bn) {
#define L6(b) \
  case b:     \
    return launch_gemm_t<b, EPI_QKV>(A, B, nullptr, M, N, K, 1, 0, st, nx, ep);
    PIC_QKV_BNS(L6)
#undef L6
  }
  return cudaErrorInvalidValue;
}

bool gemm_bn_supported(int bn, bool swiglu) {
#define C1(b) || bn == b
  return swiglu ? (false PIC_SWIGLU_BNS(C1)) : (false PIC_GEMM_BNS(C1));
#undef C1
}

cudaError_t launch_gemm_partial(const CUtensorMap& A, const CUtensorMap& B, float* out, int M, int N, int K,
                                int splits, int bn, cudaStream_t st, int pack, const GemmNext& nx, int pair) {
  if (pair) {
    switch (bn) {
#define L3(b) \
  case b:     \
    return launch_gemm_t<b, EPI_PARTIAL, 2>(A, B, out, M, N, K, splits, pack, st, nx);
      PIC_PAIR_BNS(L3)
#undef L3
    }
    return cudaErrorInvalidValue;
  }
  switch (bn) {
#define L1(b) \
  case b:     \
    return launch_gemm_t<b, EPI_PARTIAL>(A, B, out, M, N, K, splits, pack, st, nx);
    PIC_GEMM_BNS(L1)
#undef L1
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm_swiglu(const CUtensorMap& A, const CUtensorMap& B, void* u, int M, int N2, int K, int bn,
                               cudaStream_t st, int pack, const GemmNext& nx, int pair, const GemmEpi& ep) {
  if (pair) {
    switch (bn) {
#define L4(b) \
  case b:     \
    return launch_gemm_t<b, EPI_SWIGLU, 2>(A, B, u, M, N2, K, 1, pack, st, nx, ep);
      PIC_PAIR_BNS(L4)
#undef L4
    }
    return cudaErrorInvalidValue;
  }
  switch (bn) {
#define L2(b) \
  case b:     \
    return launch_gemm_t<b, EPI_SWIGLU>(A, B, u, M, N2, K, 1, pack, st, nx, ep);
    PIC_SWIGLU_BNS(L2)
#undef L2
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------------
// fp32 debug build GEMM on CUDA cores: out[M][N] = A[M][K] (fp32) · B[N][K]^T (bf16 weights, exact in
// fp32), accumulated in fp32 in ascending k.  64 x 64 output tile per CTA, 4 x 4 per thread.
__global__ void __launch_bounds__(256) gemm_simt_f32_kernel(const float* __restrict__ A, const uint16_t* __restrict__ B,
                                                            float* __restrict__ out, int M, int N, int K) {
  griddep_launch();
  griddep_wait();
  __shared__ float As[16][65], Bs[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, k = i % 16;
      As[k][r] = (m0 + r < M && k0 + k < K) ? A[(size_t)(m0 + r) * K + k0 + k] : 0.f;
      Bs[k][r] = (n0 + r < N && k0 + k < K) ? __uint_as_float((uint32_t)B[(size_t)(n0 + r) * K + k0 + k] << 16) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[k][ty * 4 + i], Bs[k][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) out[(size_t)m * N + n] = acc[i][j];
    }
}

cudaError_t launch_gemm_simt_f32(const float* A, const void* B, float* out, int M, int N, int K, cudaStream_t st) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  CUDA_TRY_LAUNCH(launch_k(gemm_simt_f32_kernel, dim3(grid), dim3(256), 0, st, A, reinterpret_cast<const uint16_t*>(B),
                           out, M, N, K));
  return cudaGetLastError();
}

}  // namespace pic
