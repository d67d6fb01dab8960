// gemm_chain.cu — one persistent kernel for the layer segment between two attentions (a7, a8, a4, a5):
//
//   O·W_oᵀ (split-K partials)  →  h += Σ partials, x = RMSNorm(h)·g2          ("O = A V_exp W_O")
//   → x·[W_g|W_u]ᵀ + SwiGLU → u  →  u·W_dᵀ (split-K partials)                   (a8, Llama MLP)
//   → h += Σ partials, x = RMSNorm(h)·g1(l+1)  →  x·W_qkvᵀ(l+1) (split-K partials) (a4, a5 of the next layer)
//
// Why one kernel: at k' = 128 rows every projection is a weight stream, and separate
// launches leave HBM idle at every boundary (epilogue, grid completion, ring refill: ~6 µs per GEMM
// measured).  Here the phases are separated by grid-wide barriers instead, and the TMA producer runs
// ahead ACROSS them: weights never depend on a barrier, only the A operands do, so the next phase's
// weight tiles stream into the smem ring while the current phase drains, the barrier resolves and the
// RMSNorm rows are computed.
//
// Same tile machinery as gemm.cu (tcgen05 M=128 UMMA, SW128 K-major TMA tiles, fp32 accumulators
// double-buffered in TMEM, split-K partials reduced by the consumer in a fixed order) with a
// byte-addressed smem ring so that phases with different N-tiles (128 / 224) keep ~200 KB in flight.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

namespace pic {

namespace chain {
constexpr int kRing = 200 * 1024;  // stage ring: A 16 KB + B bn·128 B per stage
constexpr int kStg = 16 * 1024;    // epilogue staging: 4 warps x 4 KB
constexpr int kSlots = 8;          // stage barrier slots
constexpr int kBars = 2 * kSlots + 4 + kMaxChainPhases;
constexpr int kSmem = kRing + kStg + kBars * 8 + 16;
static_assert(kSmem <= 232448, "chain smem over the 227 KB limit");
constexpr int kA = 128 * 64 * 2;
constexpr int kNormVec = 8;     // norm phase: float4 per thread, d <= 4096
constexpr int kNormSplits = 4;  // norm phase: partials summed (fixed order, zeros beyond `splits`)

// Stages of one phase tile the ring uniformly from offset 0 (at most kSlots of them).
__device__ __forceinline__ int ring_stages(int bn) {
  const int n = kRing / (kA + bn * 128);
  return n < kSlots ? n : kSlots;
}
}  // namespace chain

struct ChainMaps {
  CUtensorMap m[kMaxChainMaps];
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(192, 1)
    gemm_chain_kernel(const __grid_constant__ ChainMaps maps, const ChainParams cp) {
  using namespace chain;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();
  uint8_t* ring = smem;
  uint8_t* stg_all = smem + kRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kRing + kStg);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBars);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kSlots);
  const uint32_t tfull0 = smem_u32(bars + 2 * kSlots), tempty0 = smem_u32(bars + 2 * kSlots + 2);
  const uint32_t ready0 = smem_u32(bars + 2 * kSlots + 4);  // per phase: A operands may be loaded

  const int warp = warp_id(), lane = lane_id();
  const int G = gridDim.x;
  griddep_launch();
  unsigned long long* const tr = cp.trace ? cp.trace + 16 * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, 128);
    }
    for (int p = 0; p < kMaxChainPhases; ++p) mbar_init(ready0 + 8 * p, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto units_of = [&](const ChainPhase& ph) { return ((ph.M + 127) / 128) * ((ph.N + ph.bn - 1) / ph.bn) * ph.splits; };
  auto decode = [&](const ChainPhase& ph, int u, int& m0, int& n_idx, int& sp, int& kb0, int& nkb) {
    const int mt = (ph.M + 127) / 128;
    const int m = u % mt, r = u / mt;
    sp = r % ph.splits;
    n_idx = r / ph.splits;
    m0 = m * 128;
    kb0 = sp * ph.kper;
    nkb = max(0, min(ph.kper, ph.kblk - kb0));
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int i = 0; i < kMaxChainMaps; ++i) tma_prefetch(&maps.m[i]);
      int it = 0;  // global stage counter (barrier slot it % kSlots)
      const uint64_t wpol = l2_policy_evict_first();  // weights: streamed once
      // stages issued with B only while the phase's A operand is not ready yet (at most one ring fill)
      int pend_off[kSlots], pend_slot[kSlots], pend_kb[kSlots], pend_m0[kSlots];
      for (int p = 0; p < cp.n_phases; ++p) {
        const ChainPhase& ph = cp.ph[p];
        if (ph.type == CHAIN_NORM) continue;
        const CUtensorMap* tA = &maps.m[ph.a];
        const CUtensorMap* tB = &maps.m[ph.b];
        const int sbytes = kA + ph.bn * 128, nst = ring_stages(ph.bn);
        // the ring restarts at offset 0 for every phase: the previous phase's stages must have retired
        // (their MMAs run as soon as their data lands; the next phase's weights then stream into the
        // empty ring during the epilogue, the grid barrier and the norm phase)
        if (it > 0) mbar_wait(empty0 + 8 * ((it - 1) % kSlots), ((it - 1) / kSlots) & 1);
        const int it0 = it;
        bool ready = false;
        int npend = 0;
        auto make_ready = [&]() {
          if (p == 0)
            griddep_wait();  // A of phase 0 comes from the previous kernel
          else
            mbar_wait(ready0 + 8 * p, 0);
          fence_proxy_async_global();  // generic-proxy stores of other CTAs -> this CTA's TMA reads
          for (int k = 0; k < npend; ++k)
            tma_load_2d(smem_u32(ring + pend_off[k]), tA, full0 + 8 * pend_slot[k], pend_kb[k] * 64, pend_m0[k]);
          npend = 0;
          ready = true;
        };
        for (int u = blockIdx.x; u < units_of(ph); u += G) {
          int m0, n_idx, sp, kb0, nkb;
          decode(ph, u, m0, n_idx, sp, kb0, nkb);
          for (int kk = 0; kk < nkb; ++kk, ++it) {
            const int k = it - it0, slot = it % kSlots;
            const int off = (k % nst) * sbytes;
            if (k >= nst) {
              if (!ready) make_ready();  // the stage being recycled is still waiting for its A
              mbar_wait(empty0 + 8 * ((it - nst) % kSlots), ((it - nst) / kSlots) & 1);
            }
            mbar_expect_tx(full0 + 8 * slot, sbytes);
            tma_load_2d_hint(smem_u32(ring + off + kA), tB, full0 + 8 * slot, (kb0 + kk) * 64, n_idx * ph.bn, wpol);
            if (ready) {
              tma_load_2d(smem_u32(ring + off), tA, full0 + 8 * slot, (kb0 + kk) * 64, m0);
            } else {
              pend_off[npend] = off;
              pend_slot[npend] = slot;
              pend_kb[npend] = kb0 + kk;
              pend_m0[npend] = m0;
              ++npend;
            }
          }
          if (!ready) make_ready();
        }
        if (!ready && p == 0) griddep_wait();
      }
      if (cp.n_phases > 0 && cp.ph[0].type == CHAIN_NORM) griddep_wait();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int it = 0, i = 0;
      for (int p = 0; p < cp.n_phases; ++p) {
        const ChainPhase& ph = cp.ph[p];
        if (ph.type == CHAIN_NORM) continue;
        const uint32_t idesc = idesc_bf16(128, ph.bn, 0, 0);
        const int sbytes = kA + ph.bn * 128, nst = ring_stages(ph.bn);
        const int it0 = it;
        for (int u = blockIdx.x; u < units_of(ph); u += G, ++i) {
          int m0, n_idx, sp, kb0, nkb;
          decode(ph, u, m0, n_idx, sp, kb0, nkb);
          const int ab = i & 1;
          mbar_wait(tempty0 + 8 * ab, ((i >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + ab * 256;
          for (int kk = 0; kk < nkb; ++kk, ++it) {
            const int slot = it % kSlots;
            const int off = ((it - it0) % nst) * sbytes;
            mbar_wait(full0 + 8 * slot, (it / kSlots) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(ring + off), b = a + kA;
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              umma_bf16(d, sdesc_sw128(a + k4 * 32, 16, 1024), sdesc_sw128(b + k4 * 32, 16, 1024), idesc,
                        (kk | k4) != 0);
            umma_commit(empty0 + 8 * slot);
          }
          umma_commit(tfull0 + 8 * ab);
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue / norm warps (128 threads)
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    uint8_t* stg = stg_all + (warp - 2) * 4096;
    float* red = reinterpret_cast<float*>(stg_all);  // norm phase: block reduction scratch (staging idle)
    griddep_wait();                                  // outputs may still be read by the previous kernel
    unsigned target = 0;
    auto grid_barrier = [&](int next_phase) {
      // all epilogue threads' stores -> one gpu-scope release per CTA -> wait for every CTA
      fence_proxy_async_global();
      named_bar_sync(1, 128);
      target += G;
      if (et == 0) {
        if (tr && next_phase <= 7) tr[2 * next_phase - 1] = globaltimer();
        __threadfence();
        atomicAdd(cp.bar, 1u);
        while (ld_acquire_u32(cp.bar) < target) __nanosleep(32);
        if (tr && next_phase <= 7) tr[2 * next_phase] = globaltimer();
        if (next_phase < cp.n_phases) mbar_arrive(ready0 + 8 * next_phase);
      }
      named_bar_sync(1, 128);
    };
    int i = 0;
    for (int p = 0; p < cp.n_phases; ++p) {
      const ChainPhase& ph = cp.ph[p];
      if (ph.type == CHAIN_NORM) {
        // h[r] += Σ_s P[s][r] (fixed order); x[r] = bf16(h[r]·rsqrt(mean(h[r]²)+eps)·g)   (a4, R15)
        const int d = ph.N, n4 = d / 4;  // d <= 128·4·kNormVec
        for (int r = blockIdx.x; r < ph.M; r += G) {
          float4* hr = reinterpret_cast<float4*>(ph.h + (size_t)r * d);
          // every load of the row in flight at once: h and all split partials (unrolled, no dependences)
          float4 v[kNormVec];
          float4 w[kNormSplits][kNormVec];
#pragma unroll
          for (int j = 0; j < kNormVec; ++j) {
            const int c = et + 128 * j;
            v[j] = c < n4 ? __ldcg(hr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int s2 = 0; s2 < kNormSplits; ++s2) {
            const float4* Ps = reinterpret_cast<const float4*>(ph.P + ((size_t)s2 * ph.M + r) * d);
#pragma unroll
            for (int j = 0; j < kNormVec; ++j) {
              const int c = et + 128 * j;
              w[s2][j] = (s2 < ph.splits && c < n4) ? __ldcg(Ps + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int s2 = 0; s2 < kNormSplits; ++s2)
#pragma unroll
            for (int j = 0; j < kNormVec; ++j) {
              v[j].x += w[s2][j].x;
              v[j].y += w[s2][j].y;
              v[j].z += w[s2][j].z;
              v[j].w += w[s2][j].w;
            }
          float ss = 0.f;
#pragma unroll
          for (int j = 0; j < kNormVec; ++j) {
            const int c = et + 128 * j;
            if (c < n4) {
              hr[c] = v[j];
              ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
            }
          }
          ss = warp_sum(ss);
          if (lane == 0) red[q] = ss;
          named_bar_sync(1, 128);
          ss = (red[0] + red[1]) + (red[2] + red[3]);
          named_bar_sync(1, 128);
          const float inv = rsqrtf(ss / d + ph.eps);
          const float4* g4 = reinterpret_cast<const float4*>(ph.g);
          uint2* xo = reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(ph.out) + (size_t)r * d);
#pragma unroll
          for (int j = 0; j < kNormVec; ++j) {
            const int c = et + 128 * j;
            if (c < n4) {
              const float4 w = g4[c];
              xo[c] = make_uint2(pack_bf16(v[j].x * inv * w.x, v[j].y * inv * w.y),
                                 pack_bf16(v[j].z * inv * w.z, v[j].w * inv * w.w));
            }
          }
        }
        grid_barrier(p + 1);
        continue;
      }
      for (int u = blockIdx.x; u < units_of(ph); u += G, ++i) {
        int m0, n_idx, sp, kb0, nkb;
        decode(ph, u, m0, n_idx, sp, kb0, nkb);
        const int ab = i & 1;
        const uint32_t tl = tmem + ab * 256 + ((uint32_t)(q * 32) << 16);
        const int mrow0 = m0 + q * 32;
        mbar_wait(tfull0 + 8 * ab, (i >> 1) & 1);
        tc_fence_after();
        if (ph.type == CHAIN_GEMM) {
          float* obase = reinterpret_cast<float*>(ph.out) + (size_t)sp * ph.M * ph.N;
          const int n0 = n_idx * ph.bn, ncol = min(ph.bn, ph.N - n0);
          float4* sb = reinterpret_cast<float4*>(stg);  // [32 rows][8 float4], XOR-swizzled
          const int jj = lane & 7;
#pragma unroll 1
          for (int c = 0; c < ph.bn; c += 32) {
            float v[32];
            if (nkb > 0) {
              tmem_ld32(tl + c, v);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              sb[lane * 8 + (j ^ (lane & 7))] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int r = k * 4 + (lane >> 3);
              if (mrow0 + r < ph.M && c + 4 * jj < ncol)
                *reinterpret_cast<float4*>(obase + (size_t)(mrow0 + r) * ph.N + n0 + c + 4 * jj) =
                    sb[r * 8 + (jj ^ (r & 7))];
            }
            __syncwarp();
          }
        } else {  // CHAIN_SWIGLU: B rows = gate/up groups of bn/2; u = silu(gate) ⊙ up, bf16 [M][N/2]
          const int Gc = ph.bn / 2, F = ph.N / 2;
          uint16_t* ubase = reinterpret_cast<uint16_t*>(ph.out) + (size_t)n_idx * Gc;
          uint4* sb = reinterpret_cast<uint4*>(stg);  // [32 rows][2 uint4] (odd stride 3 -> conflict-free)
#pragma unroll 1
          for (int c = 0; c < Gc; c += 16) {
            float gv[16], uv[16];
            tmem_ld16(tl + c, gv);
            tmem_ld16(tl + Gc + c, uv);
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float g0 = gv[2 * j], g1 = gv[2 * j + 1];
              pk[j] = pack_bf16(g0 / (1.f + __expf(-g0)) * uv[2 * j], g1 / (1.f + __expf(-g1)) * uv[2 * j + 1]);
            }
            sb[lane * 3] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            sb[lane * 3 + 1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int r = k * 16 + (lane >> 1), h = lane & 1;
              if (mrow0 + r < ph.M && n_idx * Gc + c < F)
                *reinterpret_cast<uint4*>(ubase + (size_t)(mrow0 + r) * F + c + 8 * h) = sb[r * 3 + h];
            }
            __syncwarp();
          }
        }
        tc_fence_before();
        mbar_arrive(tempty0 + 8 * ab);
      }
      if (p + 1 < cp.n_phases) grid_barrier(p + 1);
    }
    // self-reset of the barrier counter for the next launch (the last CTA out)
    named_bar_sync(1, 128);
    if (tr && et == 0) tr[15] = globaltimer();
    if (et == 0) {
      __threadfence();
      if (atomicAdd(cp.bar + 1, 1u) == (unsigned)G - 1) {
        atomicExch(cp.bar, 0u);
        atomicExch(cp.bar + 1, 0u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

cudaError_t prepare_gemm_chain() {
  return cudaFuncSetAttribute(gemm_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chain::kSmem);
}

cudaError_t launch_gemm_chain(const CUtensorMap* const* maps, int n_maps, const ChainParams& cp, cudaStream_t st) {
  if (n_maps > kMaxChainMaps || cp.n_phases > kMaxChainPhases) return cudaErrorInvalidValue;
  ChainMaps m{};
  for (int i = 0; i < n_maps; ++i) m.m[i] = *maps[i];
  for (int i = n_maps; i < kMaxChainMaps; ++i) m.m[i] = *maps[0];
  CUDA_TRY_LAUNCH(launch_k(gemm_chain_kernel, dim3(148), dim3(192), chain::kSmem, st, m, cp));
  return cudaGetLastError();
}

}  // namespace pic
