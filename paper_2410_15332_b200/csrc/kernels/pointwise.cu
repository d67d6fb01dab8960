// pointwise.cu — HBM-bound kernels of the linked-prefill path: weight generator, embed gather,
// residual+RMSNorm, QKV RoPE/scatter epilogue, SwiGLU epilogue, KV link (gather + RoPE re-base),
// LM-head argmax and the CacheBlend selection kernels.  All use 16-byte vector accesses on the
// contiguous dimension and are launched with grids sized from the row counts.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

namespace pic {

cudaError_t prepare_gemm();
cudaError_t prepare_attention();
cudaError_t prepare_attention_pp();
cudaError_t prepare_attention_decode();
cudaError_t prepare_attention_qp();
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("PIC_NO_PDL") ? 0 : 1;
  return v == 1;
}

cudaError_t prepare_kernels() {
  cudaError_t e = prepare_gemm();
  if (e == cudaSuccess) e = prepare_gemm_chain();
  if (e == cudaSuccess) e = prepare_attention();
  if (e == cudaSuccess) e = prepare_attention_decode();
  if (e == cudaSuccess) e = prepare_attention_qp();
  return e == cudaSuccess ? prepare_attention_pp() : e;
}

// ================================================================================ generator
PIC_DEV uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t sm64_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t stream_key(uint64_t seed, uint64_t tag) { return sm64_host(seed ^ (tag * 0xD1B54A32D192ED03ull)); }

// bf16 bits of  bf16_rne((U>>40)·2^-23 − 1) · 2^e   (exact: the power-of-two scale keeps bf16 values)
PIC_DEV uint16_t gen_weight_bits(uint64_t key, uint64_t idx, float scale) {
  const uint64_t u = sm64(key + idx);
  const float f = (float)(uint32_t)(u >> 40) * (1.0f / 8388608.0f) - 1.0f;
  uint32_t b = __float_as_uint(f);
  b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  const float w = __uint_as_float(b) * scale;
  return (uint16_t)(__float_as_uint(w) >> 16);
}

// dst[r][c] (r < rows, c < cols) = weight at logical index (row0 + r) * logical_cols + col0 + c:
// a row slice (row0) and/or column slice (col0, logical_cols) of the logical [out][in] matrix, so a
// tensor-parallel shard gets exactly the global weights (SURVEY §8(c).6 "TP shards take slices").
__global__ void gen_matrix_kernel(uint16_t* __restrict__ dst, int64_t n8, int64_t cols, int64_t row0,
                                  int64_t logical_cols, int64_t col0, uint64_t key, float scale) {
  PIC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (8 * i) / cols, c = (8 * i) % cols;
    const uint64_t base = (uint64_t)((row0 + r) * logical_cols + col0 + c);
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = (uint32_t)gen_weight_bits(key, base + 2 * j, scale) | ((uint32_t)gen_weight_bits(key, base + 2 * j + 1, scale) << 16);
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

cudaError_t launch_gen_matrix(void* dst, int64_t rows, int64_t cols, uint64_t seed, uint64_t tag, int exp2,
                              int64_t row0, cudaStream_t st, int64_t logical_cols, int64_t col0) {
  const int64_t n = rows * cols;
  if (n % 8 || cols % 8) return cudaErrorInvalidValue;
  if (logical_cols <= 0) logical_cols = cols;
  const float scale = ldexpf(1.0f, exp2);
  CUDA_TRY_LAUNCH(launch_k(gen_matrix_kernel, dim3(148 * 8), dim3(256), 0, st, reinterpret_cast<uint16_t*>(dst), n / 8,
                           cols, row0, logical_cols, col0, stream_key(seed, tag), scale));
  return cudaGetLastError();
}

__global__ void gen_gateup_kernel(uint16_t* __restrict__ dst, int64_t F, int64_t d, uint64_t key_g, uint64_t key_u,
                                  float scale, int g, int64_t f0) {
  PIC_PDL_ENTRY();
  const int64_t n8 = 2 * F * d / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (8 * i) / d, c = (8 * i) % d;  // physical row, column
    const int64_t n = p / (2 * g), j = p % (2 * g);
    const bool up = j >= g;
    const int64_t f = f0 + n * g + (up ? j - g : j);
    const uint64_t key = up ? key_u : key_g;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t idx = (uint64_t)(f * d + c + 2 * k);
      w[k] = (uint32_t)gen_weight_bits(key, idx, scale) | ((uint32_t)gen_weight_bits(key, idx + 1, scale) << 16);
    }
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

cudaError_t launch_gen_gateup(void* dst, int64_t F, int64_t d, uint64_t seed, uint64_t tag_gate, uint64_t tag_up,
                              int exp2, int g, cudaStream_t st, int64_t f0) {
  if (d % 8 || F % g) return cudaErrorInvalidValue;
  CUDA_TRY_LAUNCH(launch_k(gen_gateup_kernel, dim3(148 * 8), dim3(256), 0, st, reinterpret_cast<uint16_t*>(dst), F, d,
                           stream_key(seed, tag_gate), stream_key(seed, tag_up), ldexpf(1.0f, exp2), g, f0));
  return cudaGetLastError();
}

__global__ void gen_gains_kernel(float* dst, int64_t n, uint64_t key) {
  PIC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = sm64(key + (uint64_t)i);
    dst[i] = 1.0f + ((float)(int)(u >> 61) - 4.0f) / 32.0f;
  }
}

cudaError_t launch_gen_gains(float* dst, int64_t n, uint64_t seed, uint64_t tag, cudaStream_t st) {
  CUDA_TRY_LAUNCH(launch_k(gen_gains_kernel, dim3(64), dim3(256), 0, st, dst, n, stream_key(seed, tag)));
  return cudaGetLastError();
}

// ================================================================================ a3 embed
// h[r] = fp32(E[tok[r]])  (P:213 step 1: "the embedding matrix E (with shape (k', d))")
__global__ void embed_kernel(const uint16_t* __restrict__ E, const int32_t* __restrict__ tok, float* __restrict__ h,
                             int d) {
  PIC_PDL_ENTRY();
  const int r = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)tok[r] * d);
  float4* dst = reinterpret_cast<float4*>(h + (size_t)r * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    const uint4 v = src[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    dst[2 * i] = make_float4(__uint_as_float(w[0] << 16), __uint_as_float(w[0] & 0xFFFF0000u),
                             __uint_as_float(w[1] << 16), __uint_as_float(w[1] & 0xFFFF0000u));
    dst[2 * i + 1] = make_float4(__uint_as_float(w[2] << 16), __uint_as_float(w[2] & 0xFFFF0000u),
                                 __uint_as_float(w[3] << 16), __uint_as_float(w[3] & 0xFFFF0000u));
  }
}

cudaError_t launch_embed(const void* E, const int32_t* tok, float* h, int M, int d, cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  CUDA_TRY_LAUNCH(launch_k(embed_kernel, dim3(M), dim3(128), 0, st, reinterpret_cast<const uint16_t*>(E), tok, h, d));
  return cudaGetLastError();
}

// Element storage of activations / KV: bf16 (product) or fp32 (the fp32 debug build, dtype = 1).
PIC_DEV uint2 pack4(float a, float b, float c, float d) { return make_uint2(pack_bf16(a, b), pack_bf16(c, d)); }
template <bool F32>
PIC_DEV void store4(void* base, size_t idx, float a, float b, float c, float d) {
  if constexpr (F32)
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + idx) = make_float4(a, b, c, d);
  else
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + idx) = pack4(a, b, c, d);
}
template <bool F32>
PIC_DEV float load1(const void* base, size_t idx) {
  if constexpr (F32)
    return reinterpret_cast<const float*>(base)[idx];
  else
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
}

// ================================================================================ a4 RMSNorm
template <int NT>
PIC_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

PIC_DEV float block_sum_dyn(float v, float* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;
}

PIC_DEV void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Σ_s P4[s·stride4 + off4]: the split loads are independent (unrolled) so they overlap in flight
PIC_DEV float4 sum_splits4(const float4* __restrict__ P4, int splits, size_t stride4, size_t off4) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
  for (int s = 0; s < splits; ++s) add4(acc, __ldg(P4 + s * stride4 + off4));
  return acc;
}

// h[r] += Σ_k src_k[r];  x[out] = bf16(h · rsqrt(mean h² + ε) · g)   (reading R4, fp32 residual R15)
// The sources are the split-K partials of the producing GEMM, or — under tensor parallelism — every
// rank's reduced partial read directly from peer memory in rank order (the all-reduce fused into the
// consumer; deterministic and identical on all ranks).  One CTA per row, one float4 per thread.
template <bool F32>
__global__ void __launch_bounds__(1024) residual_rmsnorm_kernel(float* __restrict__ h, Srcs srcs,
                                                                 const float* __restrict__ g,
                                                                 void* __restrict__ x,
                                                                 const int32_t* __restrict__ out_map, int M, int d,
                                                                 float eps) {
  griddep_launch();
  __shared__ float red[32];
  constexpr int VPT = 8;  // float4 per thread kept in registers between the two passes
  const int r = blockIdx.x;
  const int n4 = d / 4;
  // weights and the host-built row map do not depend on the upstream kernel: fetch them first
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4 gv[VPT];
  const int orow = (x && out_map) ? out_map[r] : r;
  if (x) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= n4) break;
      gv[k] = g4[i];
    }
  }
  griddep_wait();
  float4* hr = reinterpret_cast<float4*>(h + (size_t)r * d);
  float4 vc[VPT];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i >= n4) break;
    float4 v = hr[i];
    if (srcs.n) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int s = 0; s < srcs.n; ++s)
        add4(acc, __ldcg(reinterpret_cast<const float4*>(srcs.p[s]) + (size_t)r * n4 + i));
      add4(v, acc);
      hr[i] = v;
    }
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    vc[k] = v;
  }
  if (!x) return;
  ss = block_sum_dyn(ss, red);
  if (orow < 0) return;
  const float inv = rsqrtf(ss / d + eps);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i >= n4) break;
    const float4 v = vc[k], w = gv[k];
    store4<F32>(x, (size_t)orow * d + 4 * i, v.x * inv * w.x, v.y * inv * w.y, v.z * inv * w.z, v.w * inv * w.w);
  }
}

cudaError_t launch_residual_rmsnorm_srcs(float* h, const Srcs& srcs, const float* g, void* x, const int32_t* out_map,
                                         int M, int d, float eps, cudaStream_t st, int f32) {
  if (M == 0) return cudaSuccess;
  // One CTA per row.  Few rows (a link's k'): one float4 per thread, the most threads in flight for a
  // latency-bound launch between two GEMMs (cfg2 4.13 vs 4.28 ms with four).  Many rows (batched links,
  // CacheBlend's layer 0): four float4 per thread, 8 rows resident per SM (cfg4 6.7 -> 5.0 ms per link).
  const int n4 = d / 4;
  const int vpt = M >= 2048 ? 4 : 1;
  const int nt = std::max(32, std::min(1024, ((n4 + vpt - 1) / vpt + 31) / 32 * 32));
  if ((n4 + nt - 1) / nt > 8) return cudaErrorInvalidValue;
  if (f32)
    CUDA_TRY_LAUNCH(launch_k(residual_rmsnorm_kernel<true>, dim3(M), dim3(nt), 0, st, h, srcs, g, x, out_map, M, d, eps));
  else
    CUDA_TRY_LAUNCH(launch_k(residual_rmsnorm_kernel<false>, dim3(M), dim3(nt), 0, st, h, srcs, g, x, out_map, M, d, eps));
  return cudaGetLastError();
}

cudaError_t launch_residual_rmsnorm(float* h, const float* P, int splits, const float* g, void* x,
                                    const int32_t* out_map, int M, int d, float eps, cudaStream_t st, int f32) {
  Srcs s{};
  s.n = P ? splits : 0;
  if (s.n > kMaxSrcs) return cudaErrorInvalidValue;
  for (int k = 0; k < s.n; ++k) s.p[k] = P + (size_t)k * M * d;
  return launch_residual_rmsnorm_srcs(h, s, g, x, out_map, M, d, eps, st, f32);
}

// ================================================================================ tensor parallel
// out[r] = Σ_s P[s][r]  (this rank's split-K partials reduced before the cross-rank exchange)
__global__ void tp_reduce_local_kernel(const float4* __restrict__ P, int splits, size_t n4, float4* __restrict__ out) {
  PIC_PDL_ENTRY();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int s = 0; s < splits; ++s) add4(acc, P[s * n4 + i]);
    out[i] = acc;
  }
}

cudaError_t launch_tp_reduce_local(const float* P, int splits, int M, int d, float* out, cudaStream_t st) {
  const size_t n4 = (size_t)M * d / 4;
  const int blocks = (int)std::min<size_t>((n4 + 255) / 256, (size_t)148 * 8);
  CUDA_TRY_LAUNCH(launch_k(tp_reduce_local_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<const float4*>(P),
                           splits, n4, reinterpret_cast<float4*>(out)));
  return cudaGetLastError();
}

// Cross-rank epoch barrier over peer memory: every rank writes the new epoch into slot [rank] of every
// rank's flag array (system-scope release), then waits until all slots of its own array reach it
// (acquire).  The epoch counter lives in device memory, so CUDA-graph replays stay in lockstep.
__global__ void tp_barrier_kernel(long long* counter, Peers flags, int rank, int tp) {
  PIC_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  const long long epoch = *counter + 1;
  *counter = epoch;
  __threadfence_system();
  for (int p = 0; p < tp; ++p) {
    long long* slot = reinterpret_cast<long long*>(flags.p[p]) + rank;
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
  }
  const long long* mine = reinterpret_cast<const long long*>(flags.p[rank]);
  for (int p = 0; p < tp; ++p) {
    long long v;
    do {
      asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(mine + p) : "memory");
    } while (v < epoch);
  }
}

cudaError_t launch_tp_barrier(long long* counter, const Peers& flags, int rank, int tp, cudaStream_t st) {
  CUDA_TRY_LAUNCH(launch_k(tp_barrier_kernel, dim3(1), dim3(32), 0, st, counter, flags, rank, tp));
  return cudaGetLastError();
}

// ================================================================================ a5 epilogue
PIC_DEV float sum_partials(const float* P, int splits, size_t split_stride, size_t off) {
  float a = 0.f;
  for (int s = 0; s < splits; ++s) a += P[s * split_stride + off];
  return a;
}


// Q = RoPE(Σ q, p), K = RoPE(Σ k, p) -> pool slot, V = Σ v -> pool slot  (P:213 steps 2-3; written
// BEFORE attention so the selected rows also see each other).  Grid (rows, column groups); a RoPE
// thread owns 4 NeoX pairs (j..j+3, j+D/2..j+D/2+3) of one q/k head, a V thread 4 values.
template <bool F32>
__global__ void __launch_bounds__(128) qkv_rope_scatter_kernel(
    const float* __restrict__ P, int splits, int P_rows, const int32_t* __restrict__ src_row,
    const int32_t* __restrict__ pos, const int32_t* __restrict__ slot, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, void* __restrict__ Q, void* __restrict__ Kp, void* __restrict__ Vp, int Hq,
    int Hkv, int D, int static_plan, const int32_t* __restrict__ kpos) {
  griddep_launch();
  const int r = blockIdx.x;
  const int t = blockIdx.y * blockDim.x + threadIdx.x;
  const int half = D / 2, q8 = D / 8;
  const int n_rope = (Hq + Hkv) * q8, n_v = Hkv * (D / 4);
  if (t >= n_rope + n_v) {
    griddep_wait();
    return;
  }
  // host-uploaded positions / slots (and the RoPE angles they select) are complete before the graph
  // starts: fetch them while the upstream GEMM drains; CacheBlend's re-selected rows are device-side
  int p = 0, sl = 0;
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f), s = c;
  const int j = (t % q8) * 4;
  auto fetch_plan = [&]() {
    sl = slot[r];
    if (t < n_rope) {
      // K heads of a row in a chunk-frame block are rotated at the row's compile position (kpos)
      p = (kpos && t >= Hq * q8) ? kpos[r] : pos[r];
      c = *reinterpret_cast<const float4*>(cos_t + (size_t)p * half + j);
      s = *reinterpret_cast<const float4*>(sin_t + (size_t)p * half + j);
    }
  };
  if (static_plan) fetch_plan();
  griddep_wait();
  if (!static_plan) fetch_plan();
  const int srow = src_row ? src_row[r] : r;
  const int ncol4 = (Hq + 2 * Hkv) * D / 4;
  const size_t stride4 = (size_t)P_rows * ncol4;
  const float4* P4 = reinterpret_cast<const float4*>(P) + (size_t)srow * ncol4;
  const size_t kv_base = ((size_t)(sl / 16) * Hkv) * 16 * D + (size_t)(sl % 16) * D;  // + g*16*D + d
  if (t < n_rope) {
    const int hd = t / q8;
    const int col4 = (hd * D + j) / 4;
    const float4 a = sum_splits4(P4, splits, stride4, col4);
    const float4 b = sum_splits4(P4, splits, stride4, col4 + half / 4);
    void* dst = hd < Hq ? Q : Kp;
    const size_t o = hd < Hq ? ((size_t)r * Hq + hd) * D : kv_base + (size_t)(hd - Hq) * 16 * D;
    float ra[4], rb[4];
    rope_pair(a.x, b.x, c.x, s.x, ra[0], rb[0]);
    rope_pair(a.y, b.y, c.y, s.y, ra[1], rb[1]);
    rope_pair(a.z, b.z, c.z, s.z, ra[2], rb[2]);
    rope_pair(a.w, b.w, c.w, s.w, ra[3], rb[3]);
    store4<F32>(dst, o + j, ra[0], ra[1], ra[2], ra[3]);
    store4<F32>(dst, o + j + half, rb[0], rb[1], rb[2], rb[3]);
  } else {
    const int u = t - n_rope;
    const int hd = u / (D / 4), j = (u % (D / 4)) * 4;
    const float4 v = sum_splits4(P4, splits, stride4, ((Hq + Hkv) * D + hd * D + j) / 4);
    store4<F32>(Vp, kv_base + (size_t)hd * 16 * D + j, v.x, v.y, v.z, v.w);
  }
}

cudaError_t launch_qkv_rope_scatter(const float* P, int splits, int P_rows, const int32_t* src_row, const int32_t* pos,
                                    const int32_t* slot, const float* cos_t, const float* sin_t, void* Q,
                                    void* Kpool_l, void* Vpool_l, int M, int Hq, int Hkv, int D, cudaStream_t st,
                                    int f32, int static_plan, const int32_t* kpos) {
  if (M == 0) return cudaSuccess;
  const int threads = (Hq + Hkv) * (D / 8) + Hkv * (D / 4);
  dim3 grid(M, (threads + 127) / 128);
  if (f32)
    CUDA_TRY_LAUNCH(launch_k(qkv_rope_scatter_kernel<true>, dim3(grid), dim3(128), 0, st, P, splits, P_rows, src_row,
                             pos, slot, cos_t, sin_t, Q, Kpool_l, Vpool_l, Hq, Hkv, D, static_plan, kpos));
  else
    CUDA_TRY_LAUNCH(launch_k(qkv_rope_scatter_kernel<false>, dim3(grid), dim3(128), 0, st, P, splits, P_rows, src_row,
                             pos, slot, cos_t, sin_t, Q, Kpool_l, Vpool_l, Hq, Hkv, D, static_plan, kpos));
  return cudaGetLastError();
}

// ================================================================================ a8 SwiGLU
// u = bf16(silu(Σ gate) ⊙ Σ up), 4 columns per thread
template <bool F32>
__global__ void swiglu_kernel(const float* __restrict__ P, int splits, void* __restrict__ u, int M, int F) {
  PIC_PDL_ENTRY();
  const size_t n4 = (size_t)M * F / 4;
  const size_t F4 = F / 4;
  const size_t stride4 = (size_t)M * 2 * F4;
  const float4* P4 = reinterpret_cast<const float4*>(P);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / F4, f = i % F4;
    const float4 g = sum_splits4(P4, splits, stride4, r * 2 * F4 + f);
    const float4 up = sum_splits4(P4, splits, stride4, r * 2 * F4 + F4 + f);
    store4<F32>(u, 4 * i, g.x / (1.f + expf(-g.x)) * up.x, g.y / (1.f + expf(-g.y)) * up.y,
                g.z / (1.f + expf(-g.z)) * up.z, g.w / (1.f + expf(-g.w)) * up.w);
  }
}

cudaError_t launch_swiglu(const float* P, int splits, void* u, int M, int F, cudaStream_t st, int f32) {
  if (M == 0) return cudaSuccess;
  const size_t n4 = (size_t)M * F / 4;
  const int blocks = (int)std::min<size_t>((n4 + 255) / 256, (size_t)148 * 16);
  if (f32)
    CUDA_TRY_LAUNCH(launch_k(swiglu_kernel<true>, dim3(blocks), dim3(256), 0, st, P, splits, u, M, F));
  else
    CUDA_TRY_LAUNCH(launch_k(swiglu_kernel<false>, dim3(blocks), dim3(256), 0, st, P, splits, u, M, F));
  return cudaGetLastError();
}

// ================================================================================ a2 KV link
// For every cached, unselected row w and layer l >= layer0:
//   K_lnk = R(Δ_w) · K_store   (bf16 -> fp32 rotate -> bf16; reading R1, Δ = s_c − c0)
//   V_lnk = V_store            (bit copy)
// (P:213 step 3: "incorporating the cached KV vectors of the N − k' unselected tokens at correct
// positions").  One thread = one 16-byte chunk of the first half of a K head-row plus its RoPE
// partner chunk D/2 further (NeoX pairs), or one 16-byte chunk of a V head-row.
// One warp per (layer, linked row): src / dst slots and Δ are read once per row, lane (g, c) covers the
// 16-B chunk c of head g's first K half plus its NeoX partner chunk c + D/16 (rotated together) and V
// chunks c and c + D/16; every load of the row is in flight before the first store.  A (row, layer) moves
// 4·H_kv·D bytes each way.  (The earlier one-thread-per-chunk kernel spent its issue slots on 64-bit
// index arithmetic and reached 70% of HBM.)
__global__ void __launch_bounds__(256) kv_link_kernel(uint4* __restrict__ Kpool, uint4* __restrict__ Vpool,
                                                      const int32_t* __restrict__ src_slot,
                                                      const int32_t* __restrict__ dst_slot,
                                                      const int32_t* __restrict__ delta, int n_rows, int layer0,
                                                      int n_layers, int64_t layer_stride16, int Hkv, int D,
                                                      const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                                      int rebase, const int32_t* __restrict__ vcopy, int copy_k) {
  PIC_PDL_ENTRY();
  const int cK = D / 16;              // 16-B chunks per half row
  const int rowq = D / 8;             // 16-B chunks per head-row
  const int per = Hkv * cK;           // (head, chunk) lanes of a row
  const int lane = threadIdx.x & 31;
  const int64_t units = (int64_t)n_layers * n_rows;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += wstride) {
    const int w = (int)(u % n_rows);
    const int l = layer0 + (int)(u / n_rows);
    const int ss = src_slot[w], ds = dst_slot[w];
    const int dl = rebase ? delta[w] : 0;
    const bool cv = vcopy == nullptr || vcopy[w] != 0;
    const int64_t lo = (int64_t)l * layer_stride16;
    const int64_t sb = lo + (int64_t)(ss >> 4) * Hkv * 16 * rowq + (ss & 15) * rowq;
    const int64_t db = lo + (int64_t)(ds >> 4) * Hkv * 16 * rowq + (ds & 15) * rowq;
    for (int i0 = 0; i0 < per; i0 += 32) {
      const int i = i0 + lane;
      if (i >= per) break;
      const int g = i / cK, c = i % cK;
      const int64_t so = sb + (int64_t)g * 16 * rowq + c, dof = db + (int64_t)g * 16 * rowq + c;
      if (cv) {
        const uint4 va = Vpool[so], vb = Vpool[so + cK];
        Vpool[dof] = va;
        Vpool[dof + cK] = vb;
      }
      if (!copy_k) continue;
      const uint4 xa = Kpool[so], xb = Kpool[so + cK];
      if (dl == 0) {
        Kpool[dof] = xa;
        Kpool[dof + cK] = xb;
        continue;
      }
      const int ad = dl < 0 ? -dl : dl;
      const float sg = dl < 0 ? -1.f : 1.f;
      const float4* cp = reinterpret_cast<const float4*>(cos_t + (size_t)ad * (D / 2) + c * 8);
      const float4* sp = reinterpret_cast<const float4*>(sin_t + (size_t)ad * (D / 2) + c * 8);
      const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
      const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const uint32_t a4[4] = {xa.x, xa.y, xa.z, xa.w}, b4[4] = {xb.x, xb.y, xb.z, xb.w};
      uint32_t oa[4], ob[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a0 = __uint_as_float(a4[k] << 16), a1 = __uint_as_float(a4[k] & 0xFFFF0000u);
        const float b0 = __uint_as_float(b4[k] << 16), b1 = __uint_as_float(b4[k] & 0xFFFF0000u);
        float ra0, rb0, ra1, rb1;
        rebase_pair(a0, b0, cs[2 * k], sg * sn[2 * k], ra0, rb0);
        rebase_pair(a1, b1, cs[2 * k + 1], sg * sn[2 * k + 1], ra1, rb1);
        oa[k] = pack_bf16(ra0, ra1);
        ob[k] = pack_bf16(rb0, rb1);
      }
      Kpool[dof] = make_uint4(oa[0], oa[1], oa[2], oa[3]);
      Kpool[dof + cK] = make_uint4(ob[0], ob[1], ob[2], ob[3]);
    }
  }
}

// fp32 debug build: same gather + re-base on fp32 pools, one thread per NeoX pair (K) or element (V)
__global__ void kv_link_f32_kernel(float* __restrict__ Kpool, float* __restrict__ Vpool, const int32_t* __restrict__ src_slot,
                                   const int32_t* __restrict__ dst_slot, const int32_t* __restrict__ delta, int n_rows,
                                   int layer0, int n_layers, int64_t layer_stride, int Hkv, int D,
                                   const float* __restrict__ cos_t, const float* __restrict__ sin_t, int rebase,
                                   const int32_t* __restrict__ vcopy, int copy_k) {
  PIC_PDL_ENTRY();
  const int half = D / 2;
  const int64_t per_row = (int64_t)Hkv * (half + D);
  const int64_t total = (int64_t)n_layers * n_rows * per_row;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t;
    const int e = (int)(u % per_row);
    u /= per_row;
    const int w = (int)(u % n_rows);
    const int l = layer0 + (int)(u / n_rows);
    const int ss = src_slot[w], ds = dst_slot[w];
    const bool isK = e < Hkv * half;
    const int g = isK ? e / half : (e - Hkv * half) / D;
    const int j = isK ? e % half : (e - Hkv * half) % D;
    const int64_t so = (int64_t)l * layer_stride + ((int64_t)(ss / 16) * Hkv + g) * 16 * D + (int64_t)(ss % 16) * D;
    const int64_t dof = (int64_t)l * layer_stride + ((int64_t)(ds / 16) * Hkv + g) * 16 * D + (int64_t)(ds % 16) * D;
    if (!isK) {
      if (vcopy == nullptr || vcopy[w] != 0) Vpool[dof + j] = Vpool[so + j];
      continue;
    }
    if (!copy_k) continue;
    const float a = Kpool[so + j], b = Kpool[so + j + half];
    const int dl = rebase ? delta[w] : 0;
    const int ad = dl < 0 ? -dl : dl;
    const float c = cos_t[(size_t)ad * half + j], sn = (dl < 0 ? -1.f : 1.f) * sin_t[(size_t)ad * half + j];
    float ra = a, rb = b;
    if (dl) rebase_pair(a, b, c, sn, ra, rb);
    Kpool[dof + j] = ra;
    Kpool[dof + j + half] = rb;
  }
}

cudaError_t launch_kv_link(void* Kpool, void* Vpool, const int32_t* src_slot, const int32_t* dst_slot,
                           const int32_t* delta, int n_rows, int layer0, int n_layers, int64_t layer_stride_elems,
                           int Hkv, int D, const float* cos_t, const float* sin_t, int rebase, cudaStream_t st,
                           int f32, int max_ctas, const int32_t* vcopy, int copy_k) {
  if (n_rows == 0 || n_layers == 0) return cudaSuccess;
  if (f32) {
    CUDA_TRY_LAUNCH(launch_k(kv_link_f32_kernel, dim3(148 * 8), dim3(256), 0, st, reinterpret_cast<float*>(Kpool),
                             reinterpret_cast<float*>(Vpool), src_slot, dst_slot, delta, n_rows, layer0, n_layers,
                             layer_stride_elems, Hkv, D, cos_t, sin_t, rebase, vcopy, copy_k));
    return cudaGetLastError();
  }
  const int64_t warps = (int64_t)n_layers * n_rows;  // one warp per (layer, row)
  const int blocks = (int)std::min<int64_t>((warps + 7) / 8, max_ctas);
  CUDA_TRY_LAUNCH(launch_k(kv_link_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<uint4*>(Kpool), reinterpret_cast<uint4*>(Vpool), src_slot,
                                         dst_slot, delta, n_rows, layer0, n_layers, layer_stride_elems / 8, Hkv, D,
                                         cos_t, sin_t, rebase, vcopy, copy_k));
  return cudaGetLastError();
}

// ================================================================================ a10 argmax
__global__ void __launch_bounds__(1024) logits_argmax_kernel(const float* __restrict__ P, int splits,
                                                             float* __restrict__ logits, int32_t* __restrict__ amax,
                                                             int n_req, int V) {
  PIC_PDL_ENTRY();
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int r = blockIdx.x;
  float best = -INFINITY;
  int bidx = 0x7FFFFFFF;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += P[((size_t)k * n_req + r) * V + v];
    logits[(size_t)r * V + v] = s;
    if (s > best || (s == best && v < bidx)) {
      best = s;
      bidx = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) {
      best = ov;
      bidx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bi[threadIdx.x >> 5] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < bidx)) {
        best = bv[w];
        bidx = bi[w];
      }
    amax[r] = bidx;
  }
}

cudaError_t launch_logits_argmax(const float* P, int splits, float* logits, int32_t* argmax, int n_req, int V,
                                 cudaStream_t st) {
  if (n_req == 0) return cudaSuccess;
  CUDA_TRY_LAUNCH(launch_k(logits_argmax_kernel, dim3(n_req), dim3(1024), 0, st, P, splits, logits, argmax, n_req, V));
  return cudaGetLastError();
}

// ================================================================================ a9 CacheBlend
// Deviation of the check layer's fresh K (roped at p_i = i) and V from the linked (re-based) K/V
// (P:170 step 3; readings R9/R10).  Non-candidates (dynamic rows and the forced last row) get −1.
template <bool F32>
__global__ void cb_deviation_kernel(const float* __restrict__ P, int splits, const int32_t* __restrict__ cand,
                                    const int32_t* __restrict__ slot, const float* __restrict__ cos_t,
                                    const float* __restrict__ sin_t, const void* __restrict__ Kp,
                                    const void* __restrict__ Vp, float* __restrict__ dev, int N, int Hq,
                                    int Hkv, int D) {
  PIC_PDL_ENTRY();
  __shared__ float red[8];
  const int i = blockIdx.x;
  if (!cand[i]) {
    if (threadIdx.x == 0) dev[i] = -1.f;
    return;
  }
  const int half = D / 2, ncol = (Hq + 2 * Hkv) * D;
  const size_t sstride = (size_t)N * ncol;
  const float* prow = P + (size_t)i * ncol;
  const int sl = slot[i];
  const size_t kv_base = ((size_t)(sl / 16) * Hkv) * 16 * D + (size_t)(sl % 16) * D;
  float acc = 0.f;
  for (int t = threadIdx.x; t < Hkv * half; t += blockDim.x) {
    const int hd = t / half, j = t % half;
    const int col = Hq * D + hd * D + j;
    const float a = sum_partials(prow, splits, sstride, col), b = sum_partials(prow, splits, sstride, col + half);
    const float c = cos_t[(size_t)i * half + j], s = sin_t[(size_t)i * half + j];
    const size_t o = kv_base + (size_t)hd * 16 * D + j;
    const float d1 = a * c - b * s - load1<F32>(Kp, o);
    const float d2 = b * c + a * s - load1<F32>(Kp, o + half);
    acc += d1 * d1 + d2 * d2;
  }
  for (int t = threadIdx.x; t < Hkv * D; t += blockDim.x) {
    const int hd = t / D, j = t % D;
    const float v = sum_partials(prow, splits, sstride, (Hq + Hkv) * D + t);
    const float dd = v - load1<F32>(Vp, kv_base + (size_t)hd * 16 * D + j);
    acc += dd * dd;
  }
  acc = block_sum<256>(acc, red);
  if (threadIdx.x == 0) dev[i] = acc;
}

cudaError_t launch_cb_deviation(const float* P, int splits, const int32_t* cand, const int32_t* slot,
                                const float* cos_t, const float* sin_t, const void* Kpool_l, const void* Vpool_l,
                                float* dev, int N, int Hq, int Hkv, int D, cudaStream_t st, int f32) {
  if (f32)
    CUDA_TRY_LAUNCH(launch_k(cb_deviation_kernel<true>, dim3(N), dim3(256), 0, st, P, splits, cand, slot, cos_t, sin_t,
                             Kpool_l, Vpool_l, dev, N, Hq, Hkv, D));
  else
    CUDA_TRY_LAUNCH(launch_k(cb_deviation_kernel<false>, dim3(N), dim3(256), 0, st, P, splits, cand, slot, cos_t,
                             sin_t, Kpool_l, Vpool_l, dev, N, Hq, Hkv, D));
  return cudaGetLastError();
}

// rank_i = #{j : dev_j > dev_i or (dev_j == dev_i and j < i)}; keep the T best candidates (R13)
__global__ void cb_rank_kernel(const float* __restrict__ dev, int32_t* __restrict__ keep, int N, int T) {
  PIC_PDL_ENTRY();
  __shared__ float tile[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float di = i < N ? dev[i] : -1.f;
  int rank = 0;
  for (int j0 = 0; j0 < N; j0 += 256) {
    const int j = j0 + threadIdx.x;
    tile[threadIdx.x] = j < N ? dev[j] : -2.f;
    __syncthreads();
    const int lim = min(256, N - j0);
    for (int k = 0; k < lim; ++k) {
      const float dj = tile[k];
      rank += (dj > di) || (dj == di && j0 + k < i);
    }
    __syncthreads();
  }
  if (i < N) keep[i] = (di >= 0.f && rank < T) ? 1 : 0;
}

cudaError_t launch_cb_rank(const float* dev, int32_t* keep, int N, int T, cudaStream_t st) {
  CUDA_TRY_LAUNCH(launch_k(cb_rank_kernel, dim3((N + 255) / 256), dim3(256), 0, st, dev, keep, N, T));
  return cudaGetLastError();
}

// single-CTA ordered compaction (exclusive scan in 1024-wide chunks)
__global__ void __launch_bounds__(1024) cb_compact_kernel(const int32_t* __restrict__ keep, const int32_t* __restrict__ forced,
                                                          const int32_t* __restrict__ bt, int32_t* __restrict__ sel,
                                                          int32_t* __restrict__ pos, int32_t* __restrict__ slot,
                                                          int32_t* __restrict__ count, int N) {
  PIC_PDL_ENTRY();
  __shared__ int wsum[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = 0; c0 < N; c0 += 1024) {
    const int i = c0 + threadIdx.x;
    const int f = (i < N) && (keep[i] || forced[i]);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int k = 0; k < w; ++k) off += wsum[k];
    if (f) {
      const int o = off + pre;
      sel[o] = i;
      pos[o] = i;
      slot[o] = bt[i / 16] * 16 + i % 16;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int k = 0; k < 32; ++k) t += wsum[k];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

cudaError_t launch_cb_compact(const int32_t* keep, const int32_t* forced, const int32_t* bt, int32_t* sel, int32_t* pos,
                              int32_t* slot, int32_t* count, int N, cudaStream_t st) {
  CUDA_TRY_LAUNCH(launch_k(cb_compact_kernel, dim3(1), dim3(1024), 0, st, keep, forced, bt, sel, pos, slot, count, N));
  return cudaGetLastError();
}

__global__ void gather_rows_kernel(const float4* __restrict__ src, const int32_t* __restrict__ idx,
                                   float4* __restrict__ dst, int d4) {
  PIC_PDL_ENTRY();
  const int r = blockIdx.x;
  const float4* s = src + (size_t)idx[r] * d4;
  float4* o = dst + (size_t)r * d4;
  for (int i = threadIdx.x; i < d4; i += blockDim.x) o[i] = s[i];
}

cudaError_t launch_gather_rows(const float* src, const int32_t* idx, float* dst, int M, int d, cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  CUDA_TRY_LAUNCH(launch_k(gather_rows_kernel, dim3(M), dim3(256), 0, st, reinterpret_cast<const float4*>(src), idx, reinterpret_cast<float4*>(dst), d / 4));
  return cudaGetLastError();
}

}  // namespace pic
