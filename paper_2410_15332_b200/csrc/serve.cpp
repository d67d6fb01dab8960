// serve.cpp — open-loop Poisson serving of link requests.
//
// A host-side scheduler over the public C ABI: arrival times from a seeded counter-based generator,
// FIFO admission into pic_link_batch calls bounded by the free block pool, max_rows and max_batch
// (CacheBlend: one request per call), TTFT measured on the wall clock from arrival to the first
// token on the host, throughput over the window.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <thread>
#include <vector>

#include "engine.h"

namespace {

uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Exponential inter-arrival times of each user's Poisson process (rate / n_users), merged.
void arrivals(int n_users, double rate, double duration, uint64_t seed, std::vector<double>& t, std::vector<int>& u) {
  t.clear();
  u.clear();
  if (n_users <= 0 || rate <= 0 || duration <= 0) return;
  const double lam = rate / n_users;
  std::vector<std::pair<double, int>> all;
  for (int k = 0; k < n_users; ++k) {
    double now = 0;
    for (uint64_t i = 0;; ++i) {
      const uint64_t r = splitmix(seed ^ ((uint64_t)(k + 1) << 40) ^ i);
      const double U = ((r >> 11) + 1) * (1.0 / 9007199254740992.0);  // (0, 1]
      now += -std::log(U) / lam;
      if (now >= duration) break;
      all.emplace_back(now, k);
    }
  }
  std::sort(all.begin(), all.end());
  for (auto& a : all) {
    t.push_back(a.first);
    u.push_back(a.second);
  }
}

}  // namespace

extern "C" pic_status pic_serve_arrivals(int32_t n_users, double rate, double duration_s, uint64_t seed,
                                         double* times, int32_t* users, int32_t* n_inout) {
  if (!n_inout || (*n_inout > 0 && (!times || !users))) return pic_fail(PIC_E_INVALID_ARG, "serve_arrivals: NULL output");
  std::vector<double> t;
  std::vector<int> u;
  arrivals(n_users, rate, duration_s, seed, t, u);
  if ((int64_t)t.size() > *n_inout) {
    *n_inout = (int32_t)t.size();
    return pic_fail(PIC_E_CAPACITY, "serve_arrivals: %zu arrivals exceed the output capacity", t.size());
  }
  for (size_t i = 0; i < t.size(); ++i) {
    times[i] = t[i];
    users[i] = u[i];
  }
  *n_inout = (int32_t)t.size();
  return PIC_OK;
}

extern "C" pic_status pic_serve_poisson(pic_engine* e, const pic_serve_config* cfg, void* stream,
                                        pic_serve_stats* out) {
  if (!e || !cfg || !out || cfg->n_users <= 0 || !cfg->user_segs || !cfg->user_n_segs)
    return pic_fail(PIC_E_INVALID_ARG, "serve_poisson: NULL argument or no users");
  if (cfg->max_batch <= 0 || cfg->max_batch > e->lim.max_requests)
    return pic_fail(PIC_E_INVALID_ARG, "serve_poisson: max_batch %d outside [1, max_requests]", cfg->max_batch);
  const bool cb = cfg->params.alg == PIC_CACHEBLEND;
  const int max_batch = cb ? 1 : cfg->max_batch;
  // per-user footprint: linked blocks and recomputed rows (the planner's own numbers)
  std::vector<int> blocks(cfg->n_users), rows(cfg->n_users), ntok(cfg->n_users);
  for (int k = 0; k < cfg->n_users; ++k) {
    const int cap = e->lim.max_tokens;
    std::vector<int32_t> sel(cap), tok(cap), src(2 * (size_t)cap), ch(3 * (size_t)cap), bt(cap), slot(cap);
    pic_plan_out po{cap, 0, 0, 0, 0, sel.data(), tok.data(), src.data(), ch.data(), bt.data(), slot.data(), nullptr, 0};
    pic_status s = pic_plan(e, cfg->user_segs[k], cfg->user_n_segs[k], &cfg->params, &po);
    if (s != PIC_OK) return s;
    ntok[k] = po.n_tokens;
    blocks[k] = po.n_blocks - po.n_shared;  // fresh blocks only (kv_share links chunk-store blocks by reference)
    rows[k] = cb ? po.n_tokens : po.n_sel;
    if (rows[k] > e->lim.max_rows)
      return pic_fail(PIC_E_CAPACITY, "serve_poisson: user %d recomputes %d rows > max_rows", k, rows[k]);
  }
  pic_stats st0{};
  pic_get_stats(e, &st0);
  std::vector<double> at;
  std::vector<int> au;
  arrivals(cfg->n_users, cfg->rate, cfg->duration_s, cfg->seed, at, au);
  *out = pic_serve_stats{};
  out->n_requests = (int64_t)at.size();
  out->ccr = st0.total_blocks > 0 ? (double)(st0.total_blocks - st0.free_blocks) / st0.total_blocks : 0.0;
  if (at.empty()) return PIC_OK;

  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto elapsed = [&]() { return std::chrono::duration<double>(clk::now() - t0).count(); };
  std::deque<int> q;
  size_t next = 0;
  std::vector<double> ttft;
  ttft.reserve(at.size());
  double last_done = 0, tokens = 0;
  std::vector<const pic_segment*> segs;
  std::vector<int32_t> nsegs;
  std::vector<pic_link_result> res;
  while (ttft.size() < at.size()) {
    double now = elapsed();
    while (next < at.size() && at[next] <= now) q.push_back((int)next++);
    if (q.empty()) {
      std::this_thread::sleep_until(t0 + std::chrono::duration_cast<clk::duration>(std::chrono::duration<double>(at[next])));
      continue;
    }
    // FIFO admission: batch size, free pool and max_rows
    pic_stats st{};
    pic_get_stats(e, &st);
    int64_t free_b = st.free_blocks, rows_left = e->lim.max_rows;
    std::vector<int> batch;
    while (!q.empty() && (int)batch.size() < max_batch) {
      const int k = au[q.front()];
      if (blocks[k] > free_b || rows[k] > rows_left) break;
      free_b -= blocks[k];
      rows_left -= rows[k];
      batch.push_back(q.front());
      q.pop_front();
    }
    if (batch.empty())  // one request alone does not fit the pool
      return pic_fail(PIC_E_CAPACITY, "serve_poisson: one request alone does not fit the free pool");
    segs.clear();
    nsegs.clear();
    for (int i : batch) {
      segs.push_back(cfg->user_segs[au[i]]);
      nsegs.push_back(cfg->user_n_segs[au[i]]);
    }
    res.assign(batch.size(), pic_link_result{});
    pic_status s = pic_link_batch(e, (int32_t)batch.size(), segs.data(), nsegs.data(), &cfg->params, stream, nullptr,
                                  res.data());
    if (s != PIC_OK) return s;
    const double done = elapsed();  // the call returned with every first token on the host
    for (int i : batch) {
      ttft.push_back((done - at[i]) * 1e3);
      tokens += ntok[au[i]];
    }
    last_done = done;
    ++out->n_batches;
  }
  out->n_completed = (int64_t)ttft.size();
  out->elapsed_s = last_done - at.front();
  if (out->elapsed_s <= 0) out->elapsed_s = last_done;
  out->throughput_rps = out->n_completed / out->elapsed_s;
  out->tokens_per_s = tokens / out->elapsed_s;
  double sum = 0;
  for (double v : ttft) sum += v;
  out->ttft_mean_ms = sum / ttft.size();
  std::sort(ttft.begin(), ttft.end());
  auto pct = [&](double p) { return ttft[std::min(ttft.size() - 1, (size_t)(p * (ttft.size() - 1) + 0.5))]; };
  out->ttft_p50_ms = pct(0.50);
  out->ttft_p90_ms = pct(0.90);
  out->ttft_p99_ms = pct(0.99);
  out->ttft_max_ms = ttft.back();
  out->mean_batch = (double)out->n_completed / std::max<int64_t>(1, out->n_batches);
  return PIC_OK;
}
