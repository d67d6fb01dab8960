// attention_qp.cu — a6 for chunk-frame links (kv_share 3 with one frame Δ per 128-key K tile, reading
// R24): the one-lane Q-side re-base kernel (attention.cu, attn_tc_kernel<G, true, true>) made PERSISTENT.
//
// Same Eq. (1) (P:215 A = softmax(Q K_expᵀ · MASK), O = A V_exp; P:213 sparse queries, P:217 causal mask,
// reading R3) and the same arithmetic as the one-lane QROT kernel, bit for bit: q·R(Δ)k = (R(−Δ)q)·k with
// R(−Δ)·q built per chunk frame by the rotation warps into TMEM, S = Q_Δ·Kᵀ as a TS MMA, O += P·V with P
// in TMEM, lazy 2^8 rescale, 8 softmax warps (2 per row).  What changes is the schedule: 148 CTAs walk the
// host work list (item = (kv-head, piece), head-major, pieces longest first) through a dynamic queue, and
// every ring (K/V slots, S/P buffers, R(−Δ)Q buffers, O commits) keeps running across items, so the next
// item's K/V tiles, first S MMAs and first frame rotation overlap the current item's last softmax steps
// and epilogue.  The one-CTA-per-item kernel paid ~5.5 µs of prologue (barrier init, TMEM alloc, Q load +
// rotation, first K tile) and ~3.4 µs of epilogue per ~51 µs CTA at cfg4 (17%, PIC_ATTN_TRACE).
// Only O is single-buffered: the first PV of an item waits until the previous item's epilogue has read it.
// The item's Q tile is TMA-loaded into smem (reloaded once the rotation warps are done with the previous
// item's frames); O leaves TMEM straight to global (the K ring the one-CTA kernel stages it through is busy).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

#define CUDA_TRY_LAUNCH(x)              \
  do {                                 \
    cudaError_t e__ = (x);             \
    if (e__ != cudaSuccess) return e__; \
  } while (0)

#ifndef PIC_V1_POLY8
#define PIC_V1_POLY8 1  // pairs of every 8 whose exponential runs on the FMA-pipe polynomial (as attention.cu)
#endif

namespace pic {

namespace attnq {
constexpr int kTile = 16384;                  // one [128 rows][64 cols] bf16 SW128 half tile
constexpr int kStages = 3;                    // K and V ring depth
constexpr int kK = 0;
constexpr int kV = kK + kStages * 2 * kTile;
constexpr int kQ = kV + kStages * 2 * kTile;  // the item's Q tile (TMA, 2 halves): the rotation warps' source
constexpr int kX = kQ + 2 * kTile;            // softmax pair exchange: [2 parity][2 halves][128] fp32
constexpr int kBar = kX + 2 * 2 * 128 * 4;
constexpr int kIR = 4;  // item-index ring (producer -> the other 13 warps)
// k/v full/empty; s_full, p_full, o_full, qd_full, qd_empty; o_free; item ring full/empty; q_full, q_empty;
// l_full
constexpr int kNumBars = 4 * kStages + 2 * 5 + 1 + 2 * kIR + 2 + 1;
// + TMEM address slot (16 B), item ring, l_row[128] (the softmax's row sums for the offloaded epilogue)
constexpr int kSmem = kBar + kNumBars * 8 + 16 + kIR * 4 + 128 * 4 + 16;
static_assert(kSmem <= 232448, "attention smem over the 227 KB limit");
constexpr uint32_t kTmS = 0;    // S double buffer [0, 256); P(t) (bf16 pairs) overwrites S(t)
constexpr uint32_t kTmO = 256;  // O accumulator [256, 384)
constexpr uint32_t kTmQd = 384;  // two R(−Δ)·Q buffers (bf16 pairs, 64 columns each) [384, 512)
// PIC_QP_SMEMQ=1: R(−Δ)·Q in shared memory instead (S = Q_Δ·Kᵀ an SS MMA, no TS A-operand reads competing
// with the softmax's TMEM loads): the two buffers take V slot 2 and the Q tile, the rotation warps keep the
// item's q rows in registers (loaded once per item from global Q) and write every frame's R(−Δ)·q as SW128
#ifndef PIC_QP_SMEMQ
#define PIC_QP_SMEMQ 0  // measured at cfg4: attention 181-185 vs 167-168 ms per step (the 2-slot V ring costs more)
#endif
constexpr bool kQsm = PIC_QP_SMEMQ != 0;
constexpr int kSV = kQsm ? 2 : kStages;  // V ring depth
constexpr int kQd = kV + 2 * 2 * kTile;  // kQsm: R(−Δ)·Q buffers [2][two 16 KB halves]
static_assert(kQd + 2 * 2 * kTile == kX, "smem R(-Δ)Q buffers must end where the Q tile ends");
// The rotation warps (idle once an item's frames are rotated) write unsplit items' O: the softmax warps hand
// over the row sums and go straight on to the next item instead of waiting for its last PV and storing O
// (TMEM R(−Δ)Q variant; split items keep the softmax epilogue)
#ifndef PIC_QP_OFFLOAD
#define PIC_QP_OFFLOAD 1
#endif
constexpr bool kOffload = !kQsm && PIC_QP_OFFLOAD;
// PIC_QP_PSMEM=1: P goes to shared memory (the Q tile's 32 KB, SW128 K-major) and O += P·V is an SS MMA, so
// the only TMEM A-operand reads left are R(−Δ)Q's; the rotation warps keep the item's q rows in registers
// (one global load per item) instead of reading a TMA'd Q tile
#ifndef PIC_QP_PSMEM
#define PIC_QP_PSMEM 0  // measured at cfg4: attention 188.5 vs 162.4 ms per step (the smem port saturates)
#endif
constexpr bool kPsm = PIC_QP_PSMEM != 0 && !kQsm;
constexpr int kP = kQ;  // kPsm: the P tile [128 rows][128 keys] bf16, two 64-key halves
constexpr int kThreads = 448;   // warp 0 TMA, warp 1 MMA, warps 2-9 softmax, warps 10-13 frame rotation
}  // namespace attnq

// The item's q-tile: rows [row_start, row_start + row_count) of sequence seq, KV tiles [j0, j0 + n).
struct QpItem {
  int tile, split, g, seq, row_start, row_count, max_p, j0, n, last_blk;
};
PIC_DEV QpItem qp_item(const AttnArgs& a, int item) {
  QpItem it;
  // head-major (as the one-CTA-per-item grid): the CTAs work through one kv-head's pieces (longest first)
  // at a time, so a request's K/V of that head stays L2-resident across its q-tiles (the piece-major
  // order — one piece for all kv-heads side by side — measured 199 vs 178 ms per cfg4 step)
  it.g = item / a.n_work;
  const int w = item - it.g * a.n_work;
  const int* wk = a.work + 4 * w;
  it.tile = wk[0];
  it.split = wk[3];
  it.seq = a.tiles[3 * it.tile];
  it.row_start = a.tiles[3 * it.tile + 1];
  it.row_count = a.tiles[3 * it.tile + 2];
  int mp = 0;
  for (int i = lane_id(); i < it.row_count; i += 32) mp = max(mp, a.row_pos[it.row_start + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mp = max(mp, __shfl_xor_sync(0xffffffffu, mp, o));
  it.max_p = mp;
  it.j0 = wk[1];
  it.n = max(0, min(mp / 128 + 1, wk[2]) - it.j0);
  it.last_blk = mp / 16;
  return it;
}

template <int G>
__global__ void __launch_bounds__(attnq::kThreads, 1)
    attn_qp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV,
                   const __grid_constant__ CUtensorMap tmK8, const __grid_constant__ CUtensorMap tmV8,
                   const AttnArgs a) {
  griddep_launch();
  using namespace attnq;
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
  const uint32_t o_free = smem_u32(bars + 4 * S + 10);
  const uint32_t i_full = smem_u32(bars + 4 * S + 11), i_empty = smem_u32(bars + 4 * S + 11 + kIR);
  const uint32_t q_full = smem_u32(bars + 4 * S + 11 + 2 * kIR), q_empty = smem_u32(bars + 4 * S + 12 + 2 * kIR);
  const uint32_t l_full = smem_u32(bars + 4 * S + 13 + 2 * kIR);
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
      mbar_init(p_full + 8 * b, 256);
      mbar_init(o_full + 8 * b, 1);
      mbar_init(qd_full + 8 * b, 4);
      mbar_init(qd_empty + 8 * b, 1);
    }
    mbar_init(o_free, kOffload ? 12 : 8);  // 8 softmax warps (+ 4 rotation warps when they store O)
    mbar_init(l_full, 128);                // the hc = 0 softmax threads, one row sum each
    mbar_init(q_full, 1);
    mbar_init(q_empty, 4);  // the 4 rotation warps, after an item's last frame
    for (int s = 0; s < kIR; ++s) {
      mbar_init(i_full + 8 * s, 1);
      mbar_init(i_empty + 8 * s, 13);  // MMA warp, 4 rotation warps, 8 softmax warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // Q and the recomputed rows' K/V come from the upstream kernel
  const int n_items = a.n_work * a.Hkv;
  // Dynamic item queue (list order: head-major, longest pieces first — LPT over the 148 CTAs): the producer
  // draws the next item from the global counter and hands it to the other warps through a smem ring; -1 ends.
  int* const iring = reinterpret_cast<int*>(tmem_slot + 4);
  float* const lrow = reinterpret_cast<float*>(iring + kIR);  // [128] row sums of the item in its epilogue
  auto next_item = [&](int k) -> int {  // consumer warps (whole warp)
    const int sl = k % kIR;
    mbar_wait(i_full + 8 * sl, (k / kIR) & 1);
    const int it = *reinterpret_cast<volatile int*>(iring + sl);
    __syncwarp();
    if (lane == 0) mbar_arrive(i_empty + 8 * sl);
    return it;
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (K, V), all items
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmK8);
      tma_prefetch(&tmV8);
    }
    const int kv_base = a.layer * a.num_blocks;
    int kt = 0, kq = 0;  // K/V tiles and Q tiles loaded by this CTA so far
    auto load = [&](const CUtensorMap* t1, const CUtensorMap* t8, const int* tb, uint32_t dst, uint32_t full,
                    uint32_t empty, uint32_t ph, int j, int last_blk, int g) {
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
    for (int k = 0;; ++k) {
      int item = 0;
      if (lane == 0) {
        const int sl = k % kIR;
        mbar_wait(i_empty + 8 * sl, ((k / kIR) & 1) ^ 1);
        item = (int)atomicAdd(reinterpret_cast<unsigned*>(a.item_ctr), 1u);
        if (item >= n_items) item = -1;
        iring[sl] = item;
        mbar_arrive(i_full + 8 * sl);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item < 0) break;
      const QpItem it = qp_item(a, item);
      if (it.n == 0) continue;
      if (!kQsm && !kPsm && lane == 0) {
        // Q: 128 MMA rows = (128/G queries) x (G heads of kv-head g), one 3-D box per 64-dim half, once the
        // rotation warps are done with the previous item's frames
        mbar_wait(q_empty, (kq & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * kTile);
        for (int h = 0; h < 2; ++h) tma_load_3d(base + kQ + h * kTile, &tmQ, q_full, h * 64, it.g * G, it.row_start);
      }
      ++kq;
      const int* bt = a.bt + a.seq_bt_off[it.seq];
      const int* vbt = a.vbt ? a.vbt + a.seq_bt_off[it.seq] : bt;
      for (int t = 0; t < it.n; ++t, ++kt) {
        const int s = kt % S;
        const uint32_t ph = (kt / S) & 1;
        load(&tmK, &tmK8, bt, base + kK + 2 * s * kTile, k_full + 8 * s, k_empty + 8 * s, ph, it.j0 + t, it.last_blk, it.g);
        const int vs = kt % kSV;
        load(&tmV, &tmV8, vbt, base + kV + 2 * vs * kTile, v_full + 8 * vs, v_empty + 8 * vs, (kt / kSV) & 1, it.j0 + t,
             it.last_blk, it.g);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (whole warp, elect.sync)
    constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // R(−Δ)Q (TMEM, K-major) x K (smem, K-major)
    constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (TMEM, K-major) x V (smem, MN-major)
    const uint64_t dK0 = sdesc_sw128(base + kK, 16, 1024), dV0 = sdesc_sw128(base + kV, kTile, 1024);
    const uint64_t dQd = sdesc_sw128(base + kQd, 16, 1024);  // kQsm: R(−Δ)·Q buffer 0 (buffer 1: +32 KB)
    int kt = 0, fi = -1, kdone = 0;
    auto issue_pv = [&](int u, bool first) {
      const int pb = u & 1, vs = u % kSV;
      mbar_wait(p_full + 8 * pb, (u >> 1) & 1);
      mbar_wait(v_full + 8 * vs, (u / kSV) & 1);
      if (first && kdone > 0) mbar_wait(o_free, (kdone - 1) & 1);  // previous item's epilogue has read O
      tc_fence_after();
      const uint64_t dv = dV0 + (uint64_t)(vs * (2 * kTile / 16));
      if constexpr (kPsm) {  // A = P in smem (K-major: keys 16kk.. at half kk/4, +32 B per 16 keys)
        const uint64_t dP = sdesc_sw128(base + kP, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_e(tmem + kTmO, dP + (uint64_t)(((kk >> 2) * kTile + (kk & 3) * 32) >> 4),
                      dv + (uint64_t)(kk * 2048 / 16), idO, (first && kk == 0) ? 0u : 1u);
      } else {
        umma_ts_k128(tmem + kTmO, tmem + kTmS + pb * 128, dv, idO, first ? 0u : 1u);
      }
      umma_commit_e(o_full + 8 * pb);
      umma_commit_e(v_empty + 8 * vs);
    };
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      const QpItem it = qp_item(a, item);
      if (it.n == 0) continue;
      const int* bdq = a.bdelta + a.seq_bt_off[it.seq];
      int fr_cur = 0, fr_next = bdq[min(it.j0 * 8, it.last_blk)];
      for (int t = 0; t < it.n; ++t, ++kt) {
        const int sb = kt & 1, ks = kt % S;
        const int fr = fr_next;
        fr_next = t + 1 < it.n ? bdq[min((it.j0 + t + 1) * 8, it.last_blk)] : fr;
        if (t == 0 || fr != fr_cur) {  // a new frame: wait for its rotated Q
          ++fi;
          mbar_wait(qd_full + 8 * (fi & 1), (fi >> 1) & 1);
        }
        fr_cur = fr;
        const int qb = fi & 1;
        const bool frame_end = t + 1 == it.n || fr_next != fr;
        mbar_wait(k_full + 8 * ks, (kt / S) & 1);
        tc_fence_after();
        // S(kt) overwrites the buffer of P(kt-2): PV(kt-2) was issued before and MMAs run in order
        const uint64_t dk = dK0 + (uint64_t)(ks * (2 * kTile / 16));
        if constexpr (kQsm)
          umma_ss_k128(tmem + kTmS + sb * 128, dQd + (uint64_t)(qb * (2 * kTile / 16)), dk, idS, 0, kTile);
        else
          umma_tsk_k128(tmem + kTmS + sb * 128, tmem + kTmQd + qb * 64, dk, idS, kTile);
        umma_commit_e(s_full + 8 * sb);
        umma_commit_e(k_empty + 8 * ks);
        if (frame_end) umma_commit_e(qd_empty + 8 * qb);  // this frame's Q buffer may be rewritten
        if (t >= 1) issue_pv(kt - 1, t == 1);
      }
      issue_pv(kt - 1, it.n == 1);
      ++kdone;
    }
  } else if (kQsm && warp >= 10) {
    // ------------------------------------------------------------------ Q re-base per chunk frame (smem)
    // Thread u owns the 16-B chunk cc = u & 7 (dims 8cc.. and partners 64+8cc..) of rows rg + 16i, rg = u >> 3:
    // the item's 8 rows x 2 chunks stay in registers (one global load per item), every frame writes its
    // R(−Δ)·q chunk pairs in the SW128 K-major layout of the S MMA's A operand.
    const int u = threadIdx.x - 320;
    const int cc = u & 7, rg = u >> 3;
    const uint16_t* Qg = reinterpret_cast<const uint16_t*>(a.Q);
    int fi = -1;
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      const QpItem it = qp_item(a, item);
      if (it.n == 0) continue;
      const int* bdq = a.bdelta + a.seq_bt_off[it.seq];
      uint4 xa[8], xb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rg + 16 * i, qi = r / G;
        xa[i] = xb[i] = make_uint4(0u, 0u, 0u, 0u);
        if (qi < it.row_count) {
          const uint4* src = reinterpret_cast<const uint4*>(Qg + ((size_t)(it.row_start + qi) * a.Hq + it.g * G + r % G) * 128 + cc * 8);
          xa[i] = __ldg(src);
          xb[i] = __ldg(src + 8);
        }
      }
      int fr_cur = 0;
      for (int t = 0; t < it.n; ++t) {
        const int fr = bdq[min((it.j0 + t) * 8, it.last_blk)];
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
        mbar_wait(qd_empty + 8 * (fi & 1), ((fi >> 1) & 1) ^ 1);  // the MMAs of frame fi−2 are done
        const uint32_t qb = base + kQd + (fi & 1) * (2 * kTile);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint4 oa = xa[i], ob = xb[i];
          if (fr != 0) {
            uint32_t a4[4] = {xa[i].x, xa[i].y, xa[i].z, xa[i].w}, b4[4] = {xb[i].x, xb[i].y, xb[i].z, xb[i].w};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const float a0 = __uint_as_float(a4[kk] << 16), a1 = __uint_as_float(a4[kk] & 0xFFFF0000u);
              const float b0 = __uint_as_float(b4[kk] << 16), b1 = __uint_as_float(b4[kk] & 0xFFFF0000u);
              float ra0, rb0, ra1, rb1;
              rebase_pair(a0, b0, cs[2 * kk], sn[2 * kk], ra0, rb0);
              rebase_pair(a1, b1, cs[2 * kk + 1], sn[2 * kk + 1], ra1, rb1);
              a4[kk] = pack_bf16(ra0, ra1);
              b4[kk] = pack_bf16(rb0, rb1);
            }
            oa = make_uint4(a4[0], a4[1], a4[2], a4[3]);
            ob = make_uint4(b4[0], b4[1], b4[2], b4[3]);
          }
          const int r = rg + 16 * i;
          const uint32_t off = (uint32_t)(r * 128 + ((cc ^ (r & 7)) << 4));  // SW128: chunk cc of row r
          sts128(qb + off, oa);
          sts128(qb + kTile + off, ob);
        }
        fence_async_smem();  // generic-proxy smem writes -> visible to the tcgen05.mma operand reads
        __syncwarp();
        if (lane == 0) mbar_arrive(qd_full + 8 * (fi & 1));
      }
    }
  } else if (warp >= 10) {
    // ------------------------------------------------------------------ Q re-base per chunk frame + O epilogue
    // Row r of the MMA (query r / G, head g·G + r % G) = TMEM lane r; this warp owns lanes 32·(warp % 4)...
    // For every frame Δ met along an item's KV range (in tile order), write R(−Δ)·q (NeoX pairs (j, j+64),
    // fp32 rotation of the bf16 q, rounded to bf16 — the one-lane QROT arithmetic) into the buffer of the
    // frame's parity, from the item's TMA-staged Q tile.  Between the first frame of item k and its later
    // frames, store the O rows of item k-1 (unsplit items): frame 0 of item k is ready before the MMA warp
    // needs it, and the softmax warps are already on item k.
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(qq * 32) << 16;
    int fi = -1, kq = 0, kt = 0, kd = 0;
    uint4 qreg[16];  // kPsm: this row's q (chunks 0..7 of half 0, then half 1), loaded once per item
    // O of an unsplit item: its last PV (u_last) has landed and the softmax published the row sums
    auto epilogue = [&](int row_start, int row_count, int g, int u_last, int kdi) {
      mbar_wait(l_full, kdi & 1);
      if (a.row_nsplit[row_start] != 1) {  // split item: the softmax warps store the partials
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
        return;
      }
      mbar_wait(o_full + 8 * (u_last & 1), (u_last >> 1) & 1);
      tc_fence_after();
      const int qi = r / G;
      const bool valid = qi < row_count;
      const float inv = 1.f / lrow[r];
      const size_t orow = ((size_t)(row_start + qi) * a.Hq + g * G + r % G) * 128;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float ov[32];
        tmem_ld32(tmem + lane_addr + kTmO + c * 32, ov);  // warp-collective
        if (c == 3) {  // O fully read: the next item's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_free);
        }
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.O) + orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(ov[8 * i] * inv, ov[8 * i + 1] * inv), pack_bf16(ov[8 * i + 2] * inv, ov[8 * i + 3] * inv),
                                pack_bf16(ov[8 * i + 4] * inv, ov[8 * i + 5] * inv), pack_bf16(ov[8 * i + 6] * inv, ov[8 * i + 7] * inv));
        }
      }
    };
    int prv_rs = 0, prv_rc = 0, prv_g = 0, prv_last = -1;  // the previous item's q-tile and last tile
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      const QpItem it = qp_item(a, item);
      if (it.n == 0) continue;
      const int* bdq = a.bdelta + a.seq_bt_off[it.seq];
      if constexpr (kPsm) {
        const int qi = r / G;
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.Q) +
                                                          ((size_t)(it.row_start + qi) * a.Hq + it.g * G + r % G) * 128);
#pragma unroll
        for (int c = 0; c < 16; ++c) qreg[c] = qi < it.row_count ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
      } else {
        mbar_wait(q_full, kq & 1);  // this item's Q tile
        ++kq;
      }
      int fr_cur = 0;
      for (int t = 0; t < it.n; ++t) {
        const int fr = bdq[min((it.j0 + t) * 8, it.last_blk)];
        if (t > 0 && fr == fr_cur) continue;
        fr_cur = fr;
        {  // rotate frame fr into the next R(−Δ)Q buffer
        ++fi;
        const int ad = fr < 0 ? -fr : fr;
        const float sg = fr < 0 ? 1.f : -1.f;  // R(−Δ): sin(−Δθ) = −sign(Δ)·sin(|Δ|θ)
        mbar_wait(qd_empty + 8 * (fi & 1), ((fi >> 1) & 1) ^ 1);  // the MMAs of frame fi−2 are done
        const uint32_t qbase = tmem + lane_addr + kTmQd + (fi & 1) * 64;
  #pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {  // dims 32hh..32hh+31 and their partners 64+32hh..
          uint32_t oa[16], ob[16];
  #pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = 4 * hh + cc;  // 16-B chunk: dims 8c..8c+7 (half 0) and 64+8c.. (half 1)
            uint4 xa, xb;
            if constexpr (kPsm) {
              xa = qreg[c];
              xb = qreg[8 + c];
            } else {
              const uint32_t off = (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4));
              xa = lds128(base + kQ + off);
              xb = lds128(base + kQ + kTile + off);
            }
            const float4* cp = reinterpret_cast<const float4*>(a.cos_t + (size_t)ad * 64 + c * 8);
            const float4* sp = reinterpret_cast<const float4*>(a.sin_t + (size_t)ad * 64 + c * 8);
            const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
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
        if (kOffload && prv_last >= 0) {  // after this item's first frame: the previous item's O
          epilogue(prv_rs, prv_rc, prv_g, prv_last, kd - 1);
          prv_last = -1;
        }
      }
      __syncwarp();
      if (!kPsm && lane == 0) mbar_arrive(q_empty);  // every frame of this item rotated: the Q tile may be reloaded
      kt += it.n;
      prv_rs = it.row_start;
      prv_rc = it.row_count;
      prv_g = it.g;
      prv_last = kt - 1;
      ++kd;
    }
    if (kOffload && prv_last >= 0) epilogue(prv_rs, prv_rc, prv_g, prv_last, kd - 1);
  } else {
    // ------------------------------------------------------------------ softmax warps (2-9) + epilogue
    // warps w and w+4 share TMEM lane quarter q = w % 4 (rows 32q..32q+31); warp half hc owns keys
    // [64hc, 64hc+64) of every S tile (= P half hc) and O columns [64hc, 64hc+64)
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int qi = r / G, hh = r % G;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t oAddr = tmem + lane_addr + kTmO + hc * 64;
    float* xmax = reinterpret_cast<float*>(smem + kX);  // [2 parity][2 halves][128 rows]
    const float sc = a.scale_log2;
    int kt = 0, ks = 0;  // tiles and (non-empty) items this CTA's softmax has processed
    for (int k = 0;; ++k) {
      const int item = next_item(k);
      if (item < 0) break;
      const QpItem it = qp_item(a, item);
      const bool valid = qi < it.row_count;
      const int row = it.row_start + qi;
      const int head = it.g * G + hh;
      const bool direct = a.row_nsplit[it.row_start] == 1;
      if (it.n == 0) {  // an empty split piece (positions end before it): neutral partial for combine
        if (valid && !direct) {
          const size_t idx = ((size_t)it.split * a.M + row) * a.Hq + head;
          float4* dst = reinterpret_cast<float4*>(a.o_part + idx * 128 + hc * 64);
          for (int i = 0; i < 16; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (hc == 0) {
            a.ml_part[2 * idx] = -INFINITY;
            a.ml_part[2 * idx + 1] = 0.f;
          }
        }
        continue;
      }
      const int pos = valid ? a.row_pos[row] : it.max_p;
      float m_ref = -INFINITY, l = 0.f;
      for (int t = 0; t < it.n; ++t, ++kt) {
        const int sb = kt & 1;
        const int key0 = (it.j0 + t) * 128 + hc * 64;
        mbar_wait(s_full + 8 * sb, (kt >> 1) & 1);
        tc_fence_after();
        const uint32_t sAddr = tmem + lane_addr + kTmS + sb * 128 + hc * 64;
        float sv[64];
        tmem_ld64(sAddr, sv);
        if (key0 + 63 > pos) {  // part of the half lies beyond the row's causal limit
#pragma unroll
          for (int i = 0; i < 64; ++i) sv[i] = (key0 + i <= pos) ? sv[i] : -INFINITY;
        }
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
        xmax[(sb * 2 + hc) * 128 + r] = mx;
        named_bar_sync(1 + q, 64);
        mx = fmaxf(mx, xmax[(sb * 2 + (hc ^ 1)) * 128 + r]);
        const bool grow = mx > m_ref + 8.f;
        const bool need = grow && m_ref != -INFINITY;
        if (__any_sync(0xffffffffu, need)) {
          // rescale O (every PV of this item up to tile t-1 must have landed) and l to the new reference
          mbar_wait(o_full + 8 * ((kt - 1) & 1), ((kt - 1) >> 1) & 1);
          tc_fence_after();
          const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            float ov[32];
            tmem_ld32(oAddr + c * 32, ov);
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] *= alpha;
            tmem_st32_wait(oAddr + c * 32, ov);
          }
          tmem_wait_st();
          l *= alpha;
        }
        if (grow) m_ref = mx;
        const float nmu = (m_ref == -INFINITY) ? 0.f : -m_ref;
        const float2 sc2 = make_float2(sc, sc), nmu2 = make_float2(nmu, nmu);
        float2 la = make_float2(0.f, 0.f), lb = make_float2(0.f, 0.f);
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {  // p = 2^(s·scale − m_ref); masked keys are −inf → 0
          const float2 xv = fma2(make_float2(sv[2 * c], sv[2 * c + 1]), sc2, nmu2);
          float2 pv;
          if ((c & 7) < PIC_V1_POLY8)
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
        if constexpr (kPsm) {
          // the single P tile was last read by PV(kt-1) (this item's or the previous item's last): wait for it
          if (kt >= 1) mbar_wait(o_full + 8 * ((kt - 1) & 1), ((kt - 1) >> 1) & 1);
          // this thread's 64 keys of row r = one 128-B SW128 row of half hc
          const uint32_t prow = base + kP + hc * kTile + r * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(prow + ((c ^ (r & 7)) << 4), make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
          fence_async_smem();  // generic-proxy smem writes -> visible to the PV MMA's operand reads
        } else {
          tmem_st32u(sAddr, pk);  // P(t) overwrites this half's S(t) columns; PV(t) reads it from TMEM
          tmem_wait_st();
          // consume every o_full phase (PV(t-1) of this item has long finished): none completes unobserved
          if (t >= 1) mbar_wait(o_full + 8 * ((kt - 1) & 1), ((kt - 1) >> 1) & 1);
        }
        tc_fence_before();
        mbar_arrive(p_full + 8 * sb);
      }
      // row sum = both halves' partial sums, through the exchange slot of the next tile's parity, then a
      // second barrier before that slot is reused by the next item's row max
      xmax[((kt & 1) * 2 + hc) * 128 + r] = l;
      named_bar_sync(1 + q, 64);
      const float l_row = l + xmax[((kt & 1) * 2 + (hc ^ 1)) * 128 + r];
      named_bar_sync(1 + q, 64);
      if (kOffload) {
        if (hc == 0) {  // hand the row sums to the rotation warps (they read lrow of item ks-1 before o_free)
          if (ks > 0) mbar_wait(o_free, (ks - 1) & 1);
          lrow[r] = l_row;
          mbar_arrive(l_full);
        }
      }
      ++ks;
      if (kOffload && direct) {  // the rotation warps store O; this warp never reads it again
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
        continue;
      }
      // epilogue: the item's last PV, then O
      const int u = kt - 1;
      mbar_wait(o_full + 8 * (u & 1), (u >> 1) & 1);
      tc_fence_after();
      const float inv = direct ? 1.f / l_row : 1.f;
      // O straight from TMEM to global (the K ring is busy with the next item's tiles): this thread's row,
      // 64 columns of half hc = one 128-B bf16 segment (direct) or 256 B of fp32 partials (split)
      const size_t orow = ((size_t)row * a.Hq + head) * 128 + hc * 64;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float ov[32];
        tmem_ld32(oAddr + c * 32, ov);  // warp-collective
        if (c == 1) {  // O fully read: the next item's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_free);
        }
        if (valid) {
          if (direct) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.O) + orow + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(pack_bf16(ov[8 * i] * inv, ov[8 * i + 1] * inv), pack_bf16(ov[8 * i + 2] * inv, ov[8 * i + 3] * inv),
                                  pack_bf16(ov[8 * i + 4] * inv, ov[8 * i + 5] * inv), pack_bf16(ov[8 * i + 6] * inv, ov[8 * i + 7] * inv));
          } else {
            float4* dst = reinterpret_cast<float4*>(a.o_part + (size_t)it.split * a.M * a.Hq * 128 + orow + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(ov[4 * i], ov[4 * i + 1], ov[4 * i + 2], ov[4 * i + 3]);
          }
        }
      }
      if (valid && hc == 0 && !direct) {
        const size_t idx = ((size_t)it.split * a.M + row) * a.Hq + head;
        a.ml_part[2 * idx] = m_ref;
        a.ml_part[2 * idx + 1] = l_row;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0) {  // every producer has drawn its final -1: the last CTA re-arms the queue
    __threadfence();
    if (atomicAdd(a.item_ctr + 1, 1u) == gridDim.x - 1) {
      a.item_ctr[0] = 0;
      a.item_ctr[1] = 0;
      __threadfence();
    }
  }
}

template <int G>
static cudaError_t launch_qp_g(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                               const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                               cudaStream_t st) {
  const int n_items = a.n_work * a.Hkv;
  CUDA_TRY_LAUNCH(launch_k(attn_qp_kernel<G>, dim3(n_items < n_sms ? n_items : n_sms), dim3(attnq::kThreads),
                           attnq::kSmem, st, tmQ, tmK, tmV, tmK8, tmV8, a));
  return cudaGetLastError();
}

cudaError_t prepare_attention_qp() {
  cudaError_t e = cudaSuccess;
  for (auto k : {attn_qp_kernel<1>, attn_qp_kernel<2>, attn_qp_kernel<4>, attn_qp_kernel<8>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, attnq::kSmem);
  return e;
}

cudaError_t launch_attention_qp(const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                                const CUtensorMap& tmK8, const CUtensorMap& tmV8, const AttnArgs& a, int n_sms,
                                cudaStream_t st) {
  if (a.n_work <= 0) return cudaSuccess;
  switch (a.Hq / a.Hkv) {
    case 1: return launch_qp_g<1>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 2: return launch_qp_g<2>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 4: return launch_qp_g<4>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    case 8: return launch_qp_g<8>(tmQ, tmK, tmV, tmK8, tmV8, a, n_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pic
