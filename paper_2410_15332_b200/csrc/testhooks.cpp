// testhooks.cpp — kernel-level test entry points (include/pic_test.h).  Tests only.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pic_test.h"
#include "kernels/kernels.h"

using namespace pic;

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}
bool tmap(CUtensorMap* m, void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box) {
  uint32_t es[5] = {1, 1, 1, 1, 1};
  auto fn = encoder();
  return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

static int g_attn_iters = 0;
static float g_attn_us = 0.f;

#define TCK(x)                                   \
  do {                                           \
    if ((x) != cudaSuccess) return PIC_E_CUDA;   \
  } while (0)

extern "C" pic_status pic_test_gemm(const uint16_t* A, const uint16_t* B, int32_t M, int32_t N, int32_t K, int32_t bn,
                                    int32_t splits, float* out) {
  if (!A || !B || !out || M <= 0 || N <= 0 || K <= 0 || K % 64 || N % 32 || splits <= 0) return PIC_E_INVALID_ARG;
  const int pair = bn < 0;  // negative bn: CTA-pair kernel (cta_group::2) with N-tile |bn|
  bn = bn < 0 ? -bn : bn;
  if (pair ? !gemm_pair_supported(bn) : (bn != 64 && bn != 128 && bn != 256)) return PIC_E_INVALID_ARG;
  TCK(prepare_kernels());
  DevBuf a, b, p;
  TCK(cudaMalloc(&a.p, (size_t)M * K * 2));
  TCK(cudaMalloc(&b.p, (size_t)N * K * 2));
  TCK(cudaMalloc(&p.p, (size_t)splits * M * N * 4));
  TCK(cudaMemcpy(a.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(b.p, B, (size_t)N * K * 2, cudaMemcpyHostToDevice));
  CUtensorMap ta, tb;
  uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, db[2] = {(uint64_t)K, (uint64_t)N}, st[1] = {(uint64_t)K * 2};
  uint32_t ba[2] = {64, 128}, bb[2] = {64, (uint32_t)(pair ? bn / 2 : bn)};
  if (!tmap(&ta, a.p, 2, da, st, ba) || !tmap(&tb, b.p, 2, db, st, bb)) return PIC_E_CUDA;
  TCK(launch_gemm_partial(ta, tb, reinterpret_cast<float*>(p.p), M, N, K, splits, bn, 0, 0, GemmNext{}, pair));
  TCK(cudaDeviceSynchronize());
  std::vector<float> part((size_t)splits * M * N);
  TCK(cudaMemcpy(part.data(), p.p, part.size() * 4, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < (size_t)M * N; ++i) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[(size_t)k * M * N + i];
    out[i] = s;
  }
  return PIC_OK;
}

static int g_attn_version = 2, g_attn_grid = 0;

namespace pic {
extern int g_attn_force;
extern int g_attn_last_kind;
}
extern "C" int32_t pic_test_last_attention_kernel(void) { return pic::g_attn_last_kind; }

extern "C" pic_status pic_test_set_attention_kernel(int32_t version) {
  if (version < 0 || version > 2) return PIC_E_INVALID_ARG;
  pic::g_attn_force = version;
  return PIC_OK;
}

extern "C" pic_status pic_test_attention_v(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                                           int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv,
                                           const int32_t* block_perm, int32_t num_blocks, int32_t n_splits,
                                           int32_t version, int32_t grid, uint16_t* O) {
  if (version != 1 && version != 2) return PIC_E_INVALID_ARG;
  g_attn_version = version;
  g_attn_grid = grid;
  extern pic_status pic_test_attention(const uint16_t*, const uint16_t*, const uint16_t*, const int32_t*, int32_t,
                                       int32_t, int32_t, int32_t, const int32_t*, int32_t, int32_t, uint16_t*);
  const pic_status s = pic_test_attention(Q, K, V, pos, M, n_keys, Hq, Hkv, block_perm, num_blocks, n_splits, O);
  g_attn_version = 2;
  g_attn_grid = 0;
  return s;
}

extern "C" pic_status pic_test_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                                         int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv,
                                         const int32_t* block_perm, int32_t num_blocks, int32_t n_splits,
                                         uint16_t* O) {
  const int D = 128;
  if (!Q || !K || !V || !pos || !block_perm || !O || M <= 0 || n_keys <= 0 || Hq % Hkv || 128 % (Hq / Hkv))
    return PIC_E_INVALID_ARG;
  const int nb = (n_keys + 15) / 16;
  TCK(prepare_kernels());
  // paged pools [num_blocks][Hkv][16][D]
  const size_t pool = (size_t)num_blocks * Hkv * 16 * D;
  std::vector<uint16_t> kp(pool, 0), vp(pool, 0);
  for (int t = 0; t < n_keys; ++t)
    for (int g = 0; g < Hkv; ++g) {
      const size_t dst = (((size_t)block_perm[t / 16] * Hkv + g) * 16 + t % 16) * D;
      std::memcpy(&kp[dst], K + ((size_t)t * Hkv + g) * D, D * 2);
      std::memcpy(&vp[dst], V + ((size_t)t * Hkv + g) * D, D * 2);
    }
  const int G = Hq / Hkv, qpt = 128 / G;
  std::vector<int32_t> tiles;
  for (int a = 0; a < M; a += qpt) {
    tiles.push_back(0);
    tiles.push_back(a);
    tiles.push_back(std::min(qpt, M - a));
  }
  const int n_tiles = (int)tiles.size() / 3;
  std::vector<int> n_kv(n_tiles);
  for (int t = 0; t < n_tiles; ++t) n_kv[t] = pos[tiles[3 * t + 1] + tiles[3 * t + 2] - 1] / 128 + 1;
  std::vector<int32_t> work(4 * (n_kv.size() + 64 * n_tiles)), nsplit(M, 1);
  int n_work = 0;
  // the test forces up to n_splits pieces per tile by asking for n_splits x more CTAs than tiles
  const bool pp = g_attn_version == 2;
  if (pp) {  // same split targets as the one-lane schedule: 2 lanes per "SM" of the pairing rule
    std::vector<int32_t> items;
    attn_schedule_pp(tiles.data(), n_tiles, n_kv.data(), Hkv, std::max(1, n_tiles * Hkv * n_splits / 2), n_splits,
                     items, nsplit.data());
    n_work = (int)items.size() / 8;
    work = items;
  } else {
    attn_schedule(tiles.data(), n_tiles, n_kv.data(), Hkv, n_tiles * Hkv * n_splits, n_splits, work.data(), &n_work,
                  nsplit.data());
  }
  const int wints = pp ? 8 : 4;
  const int grid = g_attn_grid > 0 ? g_attn_grid : 148;
  DevBuf dw, dns;
  TCK(cudaMalloc(&dw.p, wints * n_work * 4));
  TCK(cudaMalloc(&dns.p, M * 4));
  TCK(cudaMemcpy(dw.p, work.data(), wints * n_work * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dns.p, nsplit.data(), M * 4, cudaMemcpyHostToDevice));
  DevBuf dq, dk, dv, dpos, dt, dbt, doff, dop, dml, dout;
  TCK(cudaMalloc(&dq.p, (size_t)M * Hq * D * 2));
  TCK(cudaMalloc(&dk.p, pool * 2));
  TCK(cudaMalloc(&dv.p, pool * 2));
  TCK(cudaMalloc(&dpos.p, M * 4));
  TCK(cudaMalloc(&dt.p, tiles.size() * 4));
  TCK(cudaMalloc(&dbt.p, nb * 4));
  TCK(cudaMalloc(&doff.p, 4));
  TCK(cudaMalloc(&dop.p, (size_t)n_splits * M * Hq * D * 4));
  TCK(cudaMalloc(&dml.p, (size_t)n_splits * M * Hq * 2 * 4));
  TCK(cudaMalloc(&dout.p, (size_t)M * Hq * D * 2));
  TCK(cudaMemcpy(dq.p, Q, (size_t)M * Hq * D * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dk.p, kp.data(), pool * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dv.p, vp.data(), pool * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dpos.p, pos, M * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dt.p, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dbt.p, block_perm, nb * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemset(doff.p, 0, 4));
  CUtensorMap tq, tk, tv, tk8, tv8;
  {
    uint64_t dims[3] = {(uint64_t)D, (uint64_t)Hq, (uint64_t)M};
    uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)Hq * D * 2};
    uint32_t box[3] = {64, (uint32_t)G, (uint32_t)qpt};
    if (!tmap(&tq, dq.p, 3, dims, strides, box)) return PIC_E_CUDA;
  }
  {
    uint64_t dims[4] = {(uint64_t)D, 16, (uint64_t)Hkv, (uint64_t)num_blocks};
    uint64_t strides[3] = {(uint64_t)D * 2, (uint64_t)16 * D * 2, (uint64_t)Hkv * 16 * D * 2};
    uint32_t box[4] = {64, 16, 1, 1}, box8[4] = {64, 16, 1, 8};
    if (!tmap(&tk, dk.p, 4, dims, strides, box) || !tmap(&tv, dv.p, 4, dims, strides, box)) return PIC_E_CUDA;
    if (!tmap(&tk8, dk.p, 4, dims, strides, box8) || !tmap(&tv8, dv.p, 4, dims, strides, box8)) return PIC_E_CUDA;
  }
  AttnArgs a{};
  a.tiles = reinterpret_cast<int32_t*>(dt.p);
  a.seq_bt_off = reinterpret_cast<int32_t*>(doff.p);
  a.bt = reinterpret_cast<int32_t*>(dbt.p);
  a.row_pos = reinterpret_cast<int32_t*>(dpos.p);
  a.work = reinterpret_cast<int32_t*>(dw.p);
  a.n_work = n_work;
  a.M = M;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.layer = 0;
  a.num_blocks = num_blocks;
  a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  a.o_part = reinterpret_cast<float*>(dop.p);
  a.ml_part = reinterpret_cast<float*>(dml.p);
  a.Q = dq.p;
  a.row_nsplit = reinterpret_cast<int32_t*>(dns.p);
  a.O = dout.p;
  DevBuf dctr;
  TCK(cudaMalloc(&dctr.p, 8));
  TCK(cudaMemset(dctr.p, 0, 8));
  a.item_ctr = reinterpret_cast<unsigned*>(dctr.p);
  auto launch = [&]() -> cudaError_t {
    return pp ? launch_attention_pp(tq, tk, tv, tk8, tv8, a, grid, 0) : launch_attention_tc(tq, tk, tv, tk8, tv8, a, 0);
  };
  TCK(launch());
  TCK(launch_attn_combine(a.o_part, a.ml_part, reinterpret_cast<int32_t*>(dns.p), dout.p, M, Hq, D, 0));
  TCK(cudaDeviceSynchronize());
  if (g_attn_iters > 0) {
    cudaEvent_t e0, e1;
    TCK(cudaEventCreate(&e0));
    TCK(cudaEventCreate(&e1));
    TCK(cudaEventRecord(e0, 0));
    for (int i = 0; i < g_attn_iters; ++i) TCK(launch());
    TCK(cudaEventRecord(e1, 0));
    TCK(cudaEventSynchronize(e1));
    float ms = 0;
    TCK(cudaEventElapsedTime(&ms, e0, e1));
    g_attn_us = ms * 1000.f / g_attn_iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  TCK(cudaMemcpy(O, dout.p, (size_t)M * Hq * D * 2, cudaMemcpyDeviceToHost));
  return PIC_OK;
}

extern "C" pic_status pic_test_kv_link(uint16_t* Kpool, uint16_t* Vpool, int32_t n_layers, int32_t num_blocks,
                                       int32_t Hkv, int32_t D, const int32_t* src_slot, const int32_t* dst_slot,
                                       const int32_t* delta, int32_t n_rows, int32_t layer0, int32_t rebase,
                                       double theta, int32_t max_pos) {
  if (!Kpool || !Vpool || n_rows < 0 || D % 16) return PIC_E_INVALID_ARG;
  const size_t stride = (size_t)num_blocks * Hkv * 16 * D;
  const size_t pool = (size_t)n_layers * stride;
  const int half = D / 2;
  std::vector<float> cs((size_t)max_pos * half), sn((size_t)max_pos * half);
  for (int p = 0; p < max_pos; ++p)
    for (int j = 0; j < half; ++j) {
      const double ang = (double)p * std::pow(theta, -2.0 * j / (double)D);
      cs[(size_t)p * half + j] = (float)std::cos(ang);
      sn[(size_t)p * half + j] = (float)std::sin(ang);
    }
  DevBuf dk, dv, ds, dd, de, dc, dsn;
  TCK(cudaMalloc(&dk.p, pool * 2));
  TCK(cudaMalloc(&dv.p, pool * 2));
  TCK(cudaMalloc(&ds.p, std::max(1, n_rows) * 4));
  TCK(cudaMalloc(&dd.p, std::max(1, n_rows) * 4));
  TCK(cudaMalloc(&de.p, std::max(1, n_rows) * 4));
  TCK(cudaMalloc(&dc.p, cs.size() * 4));
  TCK(cudaMalloc(&dsn.p, sn.size() * 4));
  TCK(cudaMemcpy(dk.p, Kpool, pool * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dv.p, Vpool, pool * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(ds.p, src_slot, n_rows * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dd.p, dst_slot, n_rows * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(de.p, delta, n_rows * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dc.p, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(dsn.p, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  TCK(launch_kv_link(dk.p, dv.p, (int32_t*)ds.p, (int32_t*)dd.p, (int32_t*)de.p, n_rows, layer0, n_layers - layer0,
                     stride, Hkv, D, (float*)dc.p, (float*)dsn.p, rebase, 0));
  TCK(cudaDeviceSynchronize());
  TCK(cudaMemcpy(Kpool, dk.p, pool * 2, cudaMemcpyDeviceToHost));
  TCK(cudaMemcpy(Vpool, dv.p, pool * 2, cudaMemcpyDeviceToHost));
  return PIC_OK;
}

extern "C" pic_status pic_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t bn, int32_t splits, int32_t iters,
                                     float* us_per_launch) {
  if (M <= 0 || N <= 0 || K % 64 || N % 32 || splits <= 0 || iters <= 0 || !us_per_launch) return PIC_E_INVALID_ARG;
  const int pair = bn < 0;  // negative bn: CTA-pair kernel with N-tile |bn|
  bn = bn < 0 ? -bn : bn;
  if (pair && !gemm_pair_supported(bn)) return PIC_E_INVALID_ARG;
  TCK(prepare_kernels());
  const size_t wbytes = (size_t)N * K * 2;
  const int copies = (int)std::max<size_t>(2, (size_t)(512u << 20) / wbytes + 1);  // > L2 in total
  DevBuf a, b, p;
  TCK(cudaMalloc(&a.p, (size_t)M * K * 2));
  TCK(cudaMalloc(&b.p, wbytes * copies));
  TCK(cudaMalloc(&p.p, (size_t)splits * M * N * 4));
  if (getenv("PIC_BENCH_RANDOM")) {  // seeded random operands: tensor-core power (and clocks) as in the engine
    TCK(launch_gen_matrix(a.p, M, K, 1, 1, 0, 0, 0));
    TCK(launch_gen_matrix(b.p, (int64_t)N * copies, K, 2, 2, -6, 0, 0));
    TCK(cudaDeviceSynchronize());
  } else {
    TCK(cudaMemset(a.p, 0, (size_t)M * K * 2));
    TCK(cudaMemset(b.p, 0, wbytes * copies));
  }
  CUtensorMap ta;
  std::vector<CUtensorMap> tb(copies);
  const int pack = getenv("PIC_BENCH_PACK") ? atoi(getenv("PIC_BENCH_PACK")) : 0;
  uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, db[2] = {(uint64_t)K, (uint64_t)N}, st[1] = {(uint64_t)K * 2};
  uint32_t ba[2] = {64, 128}, bb[2] = {64, (uint32_t)(pair ? bn / 2 : bn)};
  if (pack) {  // packed view: rows of 64 elements
    db[0] = 64;
    db[1] = (uint64_t)N * K / 64;
    st[0] = 128;
    bb[1] = (uint32_t)pack;
  }
  uint64_t sta[1] = {(uint64_t)K * 2};
  if (!tmap(&ta, a.p, 2, da, sta, ba)) return PIC_E_CUDA;
  for (int c = 0; c < copies; ++c)
    if (!tmap(&tb[c], (char*)b.p + wbytes * c, 2, db, st, bb)) return PIC_E_CUDA;
  cudaStream_t s;
  TCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  TCK(cudaEventCreate(&e0));
  TCK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i)
    TCK(launch_gemm_partial(ta, tb[i % copies], reinterpret_cast<float*>(p.p), M, N, K, splits, bn, s, pack,
                            GemmNext{}, pair));
  const int pfk = getenv("PIC_BENCH_PFK") ? atoi(getenv("PIC_BENCH_PFK")) : 0;  // next-GEMM L2 prefetch depth
  TCK(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i)
    TCK(launch_gemm_partial(ta, tb[i % copies], reinterpret_cast<float*>(p.p), M, N, K, splits, bn, s, pack,
                            gemm_next(pack || pair ? nullptr : &tb[(i + 1) % copies], M, N, K, splits, bn, pfk), pair));
  TCK(cudaEventRecord(e1, s));
  TCK(cudaEventSynchronize(e1));
  float ms = 0;
  TCK(cudaEventElapsedTime(&ms, e0, e1));
  *us_per_launch = ms * 1000.f / iters;
  if (getenv("PIC_GEMM_TRACE") && !pair) {  // one more pair of launches with the per-CTA timeline of the second
    DevBuf tr;
    TCK(cudaMalloc(&tr.p, 148 * 6 * 8));
    TCK(cudaMemset(tr.p, 0, 148 * 6 * 8));
    TCK(launch_gemm_partial(ta, tb[0], reinterpret_cast<float*>(p.p), M, N, K, splits, bn, s, pack));
    g_gemm_trace = reinterpret_cast<unsigned long long*>(tr.p);
    TCK(launch_gemm_partial(ta, tb[1 % copies], reinterpret_cast<float*>(p.p), M, N, K, splits, bn, s, pack));
    g_gemm_trace = nullptr;
    TCK(cudaStreamSynchronize(s));
    std::vector<unsigned long long> t(148 * 6);
    TCK(cudaMemcpy(t.data(), tr.p, t.size() * 8, cudaMemcpyDeviceToHost));
    const int units = ((N + bn - 1) / bn) * ((M + 127) / 128) * splits, grid = std::min(units, 148);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, t[b * 6]);
    const char* nm[5] = {"entry", "wait_done", "first_full", "last_mma", "epi_done"};
    for (int k = 0; k < 5; ++k) {
      std::vector<double> v;
      for (int b = 0; b < grid; ++b) v.push_back((double)(t[b * 6 + k] - t0) / 1e3);
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  %-10s min %7.2f  med %7.2f  max %7.2f us\n", nm[k], v[0], v[v.size() / 2], v.back());
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  return PIC_OK;
}

extern "C" pic_status pic_bench_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* pos,
                                          int32_t M, int32_t n_keys, int32_t Hq, int32_t Hkv,
                                          const int32_t* block_perm, int32_t num_blocks, int32_t n_splits,
                                          int32_t iters, float* us) {
  std::vector<uint16_t> O((size_t)M * Hq * 128);
  g_attn_iters = iters;
  pic_status s = pic_test_attention(Q, K, V, pos, M, n_keys, Hq, Hkv, block_perm, num_blocks, n_splits, O.data());
  g_attn_iters = 0;
  if (us) *us = g_attn_us;
  return s;
}

extern "C" pic_status pic_test_gemm_swiglu(const uint16_t* A, const uint16_t* B, int32_t M, int32_t N2, int32_t K,
                                           int32_t bn, uint16_t* u) {
  const int pair = bn < 0;  // negative bn: CTA-pair kernel with N-tile |bn|
  bn = bn < 0 ? -bn : bn;
  if (!A || !B || !u || M <= 0 || N2 <= 0 || K % 64 || N2 % bn) return PIC_E_INVALID_ARG;
  if (pair ? !gemm_pair_supported(bn) : !gemm_bn_supported(bn, true)) return PIC_E_INVALID_ARG;
  TCK(prepare_kernels());
  DevBuf a, b, p;
  TCK(cudaMalloc(&a.p, (size_t)M * K * 2));
  TCK(cudaMalloc(&b.p, (size_t)N2 * K * 2));
  TCK(cudaMalloc(&p.p, (size_t)M * (N2 / 2) * 2));
  TCK(cudaMemcpy(a.p, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
  TCK(cudaMemcpy(b.p, B, (size_t)N2 * K * 2, cudaMemcpyHostToDevice));
  CUtensorMap ta, tb;
  uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, db[2] = {(uint64_t)K, (uint64_t)N2}, st[1] = {(uint64_t)K * 2};
  uint32_t ba[2] = {64, 128}, bb[2] = {64, (uint32_t)(pair ? bn / 2 : bn)};
  if (!tmap(&ta, a.p, 2, da, st, ba) || !tmap(&tb, b.p, 2, db, st, bb)) return PIC_E_CUDA;
  TCK(launch_gemm_swiglu(ta, tb, p.p, M, N2, K, bn, 0, 0, GemmNext{}, pair));
  TCK(cudaDeviceSynchronize());
  TCK(cudaMemcpy(u, p.p, (size_t)M * (N2 / 2) * 2, cudaMemcpyDeviceToHost));
  return PIC_OK;
}
