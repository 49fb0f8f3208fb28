// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference sources, which are compiled
// in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libevsim_ref.so.  Nothing from the reference is copied into
// this repository.  Used to (1) pin the C restatement (oracle/evsim_oracle.c)
// bit-for-bit, (2) generate tests/golden fixtures, and (3) time the
// reference's own CPU implementation (bench.py --impl reference).
//
// Log mode has no reference implementation; evsim_ref_log_* run the
// reference's own flow / interpolation (src/flow.cpp, src/simulate.cpp:91-121)
// and apply the log rule of DESIGN.md §3 on top — the decomposition SURVEY.md
// §8c prescribes for the log-mode baseline.
#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <optional>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "evsim/flow.hpp"
#include "evsim/io.hpp"
#include "evsim/metrics.hpp"
#include "evsim/scenes.hpp"
#include "evsim/simulate.hpp"

extern "C" {
#include "evsim_gpu.h"
}

static_assert(sizeof(evsim::Event) == sizeof(evsim_event), "Event layout");
static_assert(offsetof(evsim::Event, t) == offsetof(evsim_event, t), "Event layout");
static_assert(offsetof(evsim::Event, p) == offsetof(evsim_event, p), "Event layout");

namespace {

thread_local std::string g_err;

evsim::SimulatorConfig to_ref(const evsim_gpu_config* c) {
  evsim::SimulatorConfig r;
  r.method = static_cast<evsim::Method>(c->method);
  r.c_pos = c->c_pos;
  r.c_neg = c->c_neg;
  r.n_interp = c->n_interp;
  r.flow_preset = static_cast<evsim::FlowQuality>(c->flow_preset);
  r.selection_threshold = c->selection_threshold;
  r.events_per_crossing = static_cast<evsim::EventsPerCrossing>(c->events_per_crossing);
  r.include_endpoints = c->include_endpoints != 0;
  return r;
}

evsim::FlowPreset preset_of(const evsim_gpu_config* c) {
  if (c->pyramid_levels || c->iterations_per_level || c->patch_radius)
    return evsim::FlowPreset{c->pyramid_levels, c->iterations_per_level, c->patch_radius};
  return evsim::flow_preset(static_cast<evsim::FlowQuality>(c->flow_preset));
}

evsim::Frame make_frame(const uint8_t* px, int w, int h, int64_t t) {
  evsim::Frame f(w, h, t);
  std::memcpy(f.pixels.data(), px, f.pixels.size());
  return f;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EVSIM_GPU_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EVSIM_GPU_RUNTIME;
  }
}

// Stub backends: hand caller-supplied flow to the reference pipelines.
class FixedDense final : public evsim::DenseFlowEstimator {
 public:
  FixedDense(const float* du, const float* dv, int w, int h) : f_(w, h) {
    std::memcpy(f_.du.data(), du, f_.du.size() * sizeof(float));
    std::memcpy(f_.dv.data(), dv, f_.dv.size() * sizeof(float));
  }
  evsim::FlowField estimate(const evsim::Frame&, const evsim::Frame&) const override { return f_; }

 private:
  evsim::FlowField f_;
};

class FixedSparse final : public evsim::SparseFlowEstimator {
 public:
  FixedSparse(const float* disp, const uint8_t* st, int64_t m) {
    for (int64_t i = 0; i < m; ++i) {
      d_.push_back({disp[2 * i], disp[2 * i + 1]});
      s_.push_back(st[i]);
    }
  }
  evsim::SparseFlow estimate(const evsim::Frame&, const evsim::Frame&,
                             const std::vector<evsim::PixelPoint>& pts) const override {
    if (pts.size() != d_.size()) throw std::invalid_argument("FixedSparse: point count mismatch");
    evsim::SparseFlow f;
    f.points = pts;
    f.displacements = d_;
    f.status = s_;
    return f;
  }

 private:
  std::vector<evsim::Displacement> d_;
  std::vector<std::uint8_t> s_;
};

// ---- log-mode restatement on top of the reference's stages ---------------
void log_link(const evsim_gpu_config* c, const float* lut, const uint8_t* after, int w, int y0, int y1,
              int64_t t, float* ref, std::vector<evsim::Event>& out) {
  const bool mag = c->events_per_crossing == EVSIM_EVENTS_MAGNITUDE;
  for (int y = y0; y < y1; ++y)
    for (int x = 0; x < w; ++x) {
      const std::size_t i = static_cast<std::size_t>(y) * w + x;
      const float lk = lut[after[i]];
      const float d = lk - ref[i];
      if (d > c->c_pos_log) {
        const int n = mag ? static_cast<int>(std::floor(d / c->c_pos_log)) : 1;
        for (int k = 0; k < n; ++k)
          out.push_back({static_cast<std::uint16_t>(x), static_cast<std::uint16_t>(y), t, 1});
        ref[i] = lk;
      } else if (d < c->c_neg_log) {
        const int n = mag ? static_cast<int>(std::floor(d / c->c_neg_log)) : 1;
        for (int k = 0; k < n; ++k)
          out.push_back({static_cast<std::uint16_t>(x), static_cast<std::uint16_t>(y), t, -1});
        ref[i] = lk;
      }
    }
}

// Intermediate chain frames of one pair in log mode: the reference's own
// flow + interpolate_frames (dense), or its selection / sparse LK / splat
// (simulate.cpp:145-199, restated here because it is inline in
// simulate_sparse) with the log-mode selection of DESIGN.md §3.
std::vector<evsim::Frame> log_chain_frames(const evsim_gpu_config* c, const float* lut, const evsim::Frame& pf,
                                           const evsim::Frame& f) {
  const int w = f.width, h = f.height;
  const int64_t t = f.timestamp;
  std::vector<evsim::Frame> inter;
  if (c->method == EVSIM_METHOD_DENSE && c->n_interp > 0) {
    const evsim::FlowField fl = evsim::estimate_dense_flow(pf, f, preset_of(c));
    inter = evsim::interpolate_frames(pf, f, fl, c->n_interp);
  } else if (c->method == EVSIM_METHOD_SPARSE && c->n_interp > 0) {
    const float sel = c->sel_log > 0.0f ? c->sel_log : c->c_pos_log;
    std::vector<evsim::PixelPoint> pts;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        if (std::fabs(lut[f.at(x, y)] - lut[pf.at(x, y)]) > sel) pts.push_back({x, y});
    if (!pts.empty()) {
      const evsim::SparseFlow fl = evsim::estimate_sparse_flow(pf, f, pts, preset_of(c));
      std::vector<int> mark(pf.pixel_count(), -1), chg(pf.pixel_count(), 0);
      for (int k = 1; k <= c->n_interp; ++k) {
        const float alpha = static_cast<float>(k) / static_cast<float>(c->n_interp + 1);
        evsim::Frame fr = pf;
        fr.timestamp = evsim::sub_interval_end(pf.timestamp, t, k, c->n_interp + 1);
        for (std::size_t j = 0; j < pts.size(); ++j) {
          if (!fl.status[j]) continue;
          const int tx = static_cast<int>(std::lround(static_cast<float>(pts[j].x) + alpha * fl.displacements[j].du));
          const int ty = static_cast<int>(std::lround(static_cast<float>(pts[j].y) + alpha * fl.displacements[j].dv));
          if (tx < 0 || tx >= w || ty < 0 || ty >= h) continue;
          const std::size_t idx = static_cast<std::size_t>(ty) * w + tx;
          const std::uint8_t value = pf.at(pts[j].x, pts[j].y);
          const int change = std::abs(static_cast<int>(value) - static_cast<int>(pf.pixels[idx]));
          if (mark[idx] != k) {
            mark[idx] = k;
            chg[idx] = change;
            fr.pixels[idx] = value;
          } else if (change > chg[idx]) {
            chg[idx] = change;
            fr.pixels[idx] = value;
          }
        }
        inter.push_back(std::move(fr));
      }
    }
  }
  return inter;
}

}  // namespace

struct evsim_ref_sim {
  evsim_gpu_config cfg;
  std::unique_ptr<evsim::Simulator> sim;  // linear mode: the reference itself
  evsim::EventStream last;
  // log mode state
  std::optional<evsim::Frame> prev;
  std::vector<float> ref;
  float lut[256];
};

extern "C" {

const char* evsim_ref_last_error(void) { return g_err.c_str(); }

int evsim_ref_create(const evsim_gpu_config* cfg, evsim_ref_sim** out) {
  return guarded([&] {
    auto s = std::make_unique<evsim_ref_sim>();
    s->cfg = *cfg;
    if (cfg->contrast_mode == EVSIM_CONTRAST_LINEAR) {
      const evsim::FlowPreset p = preset_of(cfg);
      s->sim = std::make_unique<evsim::Simulator>(to_ref(cfg),
                                                  std::make_shared<evsim::PyramidalPatchFlow>(p),
                                                  std::make_shared<evsim::PyramidalLucasKanade>(p));
    } else {
      if (cfg->method == EVSIM_METHOD_DIFFERENCE_INTERP)
        throw std::invalid_argument("SimulatorConfig: difference_interp has no log contrast mode");
      to_ref(cfg).validate();
      for (int i = 0; i < 256; ++i) s->lut[i] = std::log(static_cast<float>(i) / 255.0f + 1e-3f);
    }
    *out = s.release();
  });
}

void evsim_ref_destroy(evsim_ref_sim* s) { delete s; }

int evsim_ref_reset(evsim_ref_sim* s) {
  if (s->sim) s->sim->reset();
  s->prev.reset();
  return 0;
}

int evsim_ref_push_frame(evsim_ref_sim* s, const uint8_t* px, int32_t w, int32_t h, int64_t t,
                         const evsim_event** ev, int64_t* n) {
  return guarded([&] {
    const evsim::Frame f = make_frame(px, w, h, t);
    if (s->sim) {
      s->last = s->sim->push_frame(f);
    } else {
      // log mode: reference stages + restated rule
      const evsim_gpu_config* c = &s->cfg;
      s->last = evsim::EventStream{w, h, {}};
      if (s->prev) {
        if (t <= s->prev->timestamp)
          throw std::invalid_argument("push_frame: timestamps must be strictly increasing");
        const evsim::Frame& pf = *s->prev;
        std::vector<evsim::Frame> inter = log_chain_frames(c, s->lut, pf, f);
        std::vector<const evsim::Frame*> chain;
        if (c->method == EVSIM_METHOD_DIFFERENCE_ONLY || c->include_endpoints) chain.push_back(&pf);
        for (const auto& fr : inter) chain.push_back(&fr);
        if (c->method == EVSIM_METHOD_DIFFERENCE_ONLY || c->include_endpoints) chain.push_back(&f);
        for (std::size_t i = 1; i < chain.size(); ++i)
          log_link(c, s->lut, chain[i]->pixels.data(), w, 0, h, chain[i]->timestamp, s->ref.data(),
                   s->last.events);
        if (!std::is_sorted(s->last.events.begin(), s->last.events.end(), evsim::event_order))
          std::stable_sort(s->last.events.begin(), s->last.events.end(), evsim::event_order);
      } else {
        s->ref.resize(f.pixel_count());
        for (std::size_t i = 0; i < f.pixel_count(); ++i) s->ref[i] = s->lut[f.pixels[i]];
      }
      s->prev = f;
    }
    *ev = reinterpret_cast<const evsim_event*>(s->last.events.data());
    *n = static_cast<int64_t>(s->last.events.size());
  });
}

int evsim_ref_dense_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                         int32_t levels, int32_t iters, int32_t radius, float* du, float* dv) {
  return guarded([&] {
    const evsim::FlowField f = evsim::estimate_dense_flow(
        make_frame(prev, w, h, 0), make_frame(curr, w, h, 1), evsim::FlowPreset{levels, iters, radius});
    std::memcpy(du, f.du.data(), f.du.size() * sizeof(float));
    std::memcpy(dv, f.dv.data(), f.dv.size() * sizeof(float));
  });
}

int evsim_ref_sparse_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                          int32_t levels, int32_t iters, int32_t radius, const int32_t* pts,
                          int64_t m, float* disp, uint8_t* status) {
  return guarded([&] {
    std::vector<evsim::PixelPoint> p(static_cast<std::size_t>(m));
    for (int64_t i = 0; i < m; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
    const evsim::SparseFlow f = evsim::estimate_sparse_flow(
        make_frame(prev, w, h, 0), make_frame(curr, w, h, 1), p, evsim::FlowPreset{levels, iters, radius});
    for (int64_t i = 0; i < m; ++i) {
      disp[2 * i] = f.displacements[i].du;
      disp[2 * i + 1] = f.displacements[i].dv;
      status[i] = f.status[i];
    }
  });
}

int evsim_ref_interpolate_frames(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                 int64_t t0, int64_t t1, const float* du, const float* dv,
                                 int32_t n, uint8_t* out, int64_t* out_t) {
  return guarded([&] {
    evsim::FlowField fl(w, h);
    std::memcpy(fl.du.data(), du, fl.du.size() * sizeof(float));
    std::memcpy(fl.dv.data(), dv, fl.dv.size() * sizeof(float));
    const auto fr = evsim::interpolate_frames(make_frame(prev, w, h, t0), make_frame(curr, w, h, t1), fl, n);
    for (int k = 0; k < n; ++k) {
      std::memcpy(out + static_cast<std::size_t>(k) * w * h, fr[k].pixels.data(), fr[k].pixels.size());
      out_t[k] = fr[k].timestamp;
    }
  });
}

static int copy_out(const evsim::EventStream& s, evsim_event** ev, int64_t* n) {
  *n = static_cast<int64_t>(s.events.size());
  *ev = static_cast<evsim_event*>(std::malloc(std::max<std::size_t>(1, s.events.size()) * sizeof(evsim_event)));
  std::memcpy(*ev, s.events.data(), s.events.size() * sizeof(evsim_event));
  return 0;
}

int evsim_ref_dense_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                     int64_t t0, int64_t t1, const float* du, const float* dv,
                                     const evsim_gpu_config* cfg, evsim_event** ev, int64_t* n) {
  return guarded([&] {
    const FixedDense est(du, dv, w, h);
    copy_out(evsim::simulate_dense(make_frame(prev, w, h, t0), make_frame(curr, w, h, t1), to_ref(cfg), est), ev, n);
  });
}

int evsim_ref_sparse_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                      int64_t t0, int64_t t1, const float* disp, const uint8_t* st,
                                      int64_t m, const evsim_gpu_config* cfg, evsim_event** ev,
                                      int64_t* n) {
  return guarded([&] {
    const FixedSparse est(disp, st, m);
    copy_out(evsim::simulate_sparse(make_frame(prev, w, h, t0), make_frame(curr, w, h, t1), to_ref(cfg), est), ev, n);
  });
}

void evsim_ref_free(void* p) { std::free(p); }

// ---- multi-threaded sequence runner (bench.py --impl reference, cpu_baseline)
//
// Runs the reference over frames[0..n) with `threads` host threads and
// reports, per frame, the event count and the checksum of
// paper_2209_04634_b200/seqhash.py — output identical to ONE streaming
// Simulator (verified against tests/golden/sequences.json):
//  * linear mode: the reference Simulator keeps no state across pairs but
//    the previous frame (simulate.cpp:306-347), so the sequence is split into
//    contiguous chunks overlapping by one frame, one Simulator per thread;
//  * log mode: per pair the reference's intermediate frames
//    (log_chain_frames) are computed in parallel over pairs (a window of
//    `threads` pairs at a time), then the per-pixel log rule runs pair by
//    pair in stream order, in parallel over row bands (the rule is per pixel;
//    a link's events are the bands' events concatenated, (y, x) order).
}  // extern "C"

namespace {
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
struct FrameSum {
  uint64_t h = 0;
  int64_t n = 0;
  void add(const evsim::Event& e, int64_t t_prev) {
    const uint64_t v = (uint64_t)e.x | ((uint64_t)e.y << 16) | ((uint64_t)(e.p < 0) << 31) |
                       ((uint64_t)(e.t - t_prev) << 32);
    h += mix64(v + (uint64_t)n * 0x9E3779B97F4A7C15ull);
    ++n;
  }
};
template <class F>
void parallel_for(int n, int threads, F&& f) {
  std::atomic<int> next{0};
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex m;
  for (int i = 0; i < std::max(1, std::min(threads, n)); ++i)
    th.emplace_back([&] {
      try {
        for (int j; (j = next.fetch_add(1)) < n;) f(j);
      } catch (...) {
        std::lock_guard<std::mutex> g(m);
        err = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}
}  // namespace

extern "C" {

int evsim_ref_run_sequence(const evsim_gpu_config* cfg, const uint8_t* frames, int32_t n, int32_t w, int32_t h,
                           const int64_t* ts, int32_t threads, int64_t* counts, uint64_t* hashes) {
  return guarded([&] {
    const std::size_t P = static_cast<std::size_t>(w) * h;
    threads = std::max(1, threads);
    for (int k = 0; k < n; ++k) counts[k] = 0, hashes[k] = 0;
    if (n < 2) return;
    auto finish_frame = [&](int k, const std::vector<evsim::Event>& ev) {
      FrameSum s;
      for (const auto& e : ev) s.add(e, ts[k - 1]);
      counts[k] = s.n;
      hashes[k] = s.h;
    };
    if (cfg->contrast_mode == EVSIM_CONTRAST_LINEAR) {
      const int T = std::min(threads, n - 1);
      parallel_for(T, T, [&](int c) {
        const int lo = (int)((int64_t)(n - 1) * c / T), hi = (int)((int64_t)(n - 1) * (c + 1) / T);
        const evsim::FlowPreset p = preset_of(cfg);
        evsim::Simulator sim(to_ref(cfg), std::make_shared<evsim::PyramidalPatchFlow>(p),
                             std::make_shared<evsim::PyramidalLucasKanade>(p));
        for (int k = lo; k <= hi; ++k) {
          const evsim::EventStream es = sim.push_frame(make_frame(frames + k * P, w, h, ts[k]));
          if (k > lo) finish_frame(k, es.events);
        }
      });
      return;
    }
    if (cfg->method == EVSIM_METHOD_DIFFERENCE_INTERP)
      throw std::invalid_argument("SimulatorConfig: difference_interp has no log contrast mode");
    to_ref(cfg).validate();
    float lut[256];
    for (int i = 0; i < 256; ++i) lut[i] = std::log(static_cast<float>(i) / 255.0f + 1e-3f);
    std::vector<float> ref(P);
    for (std::size_t i = 0; i < P; ++i) ref[i] = lut[frames[i]];
    const bool ends = cfg->method == EVSIM_METHOD_DIFFERENCE_ONLY || cfg->include_endpoints;
    const int bands = std::min(threads, h);
    for (int a = 1; a < n; a += threads) {
      const int np = std::min(threads, n - a);  // pairs (a-1, a) .. (a+np-2, a+np-1)
      std::vector<std::vector<evsim::Frame>> inter(np);
      parallel_for(np, threads, [&](int i) {
        const int k = a + i;
        inter[i] = log_chain_frames(cfg, lut, make_frame(frames + (k - 1) * P, w, h, ts[k - 1]),
                                    make_frame(frames + k * P, w, h, ts[k]));
      });
      for (int i = 0; i < np; ++i) {
        const int k = a + i;
        std::vector<const uint8_t*> px;
        std::vector<int64_t> tl;
        for (const auto& fr : inter[i]) px.push_back(fr.pixels.data()), tl.push_back(fr.timestamp);
        if (ends) px.push_back(frames + k * P), tl.push_back(ts[k]);
        // links in order; each link's bands in row order
        std::vector<evsim::Event> ev;
        std::vector<std::vector<std::vector<evsim::Event>>> lb(px.size(), std::vector<std::vector<evsim::Event>>(bands));
        parallel_for(bands, bands, [&](int b) {
          const int y0 = (int)((int64_t)h * b / bands), y1 = (int)((int64_t)h * (b + 1) / bands);
          for (std::size_t l = 0; l < px.size(); ++l) log_link(cfg, lut, px[l], w, y0, y1, tl[l], ref.data(), lb[l][b]);
        });
        for (auto& l : lb)
          for (auto& b : l) ev.insert(ev.end(), b.begin(), b.end());
        if (!std::is_sorted(ev.begin(), ev.end(), evsim::event_order))
          std::stable_sort(ev.begin(), ev.end(), evsim::event_order);
        finish_frame(k, ev);
        inter[i].clear();
        inter[i].shrink_to_fit();
      }
    }
  });
}

// ---- reference scenes (src/scenes.cpp), for fixtures --------------------
int evsim_ref_textured_frame(int32_t w, int32_t h, uint32_t seed, uint8_t lo, uint8_t hi, uint8_t* out) {
  return guarded([&] {
    const auto f = evsim::scenes::textured_frame(w, h, 0, seed, lo, hi);
    std::memcpy(out, f.pixels.data(), f.pixels.size());
  });
}

static int copy_frames(const std::vector<evsim::Frame>& fr, uint8_t* out, int64_t* ts) {
  std::size_t off = 0;
  for (std::size_t k = 0; k < fr.size(); ++k) {
    std::memcpy(out + off, fr[k].pixels.data(), fr[k].pixels.size());
    off += fr[k].pixels.size();
    ts[k] = fr[k].timestamp;
  }
  return 0;
}

int evsim_ref_panning_texture(int32_t w, int32_t h, int32_t n, int32_t dx, int32_t dy, double fps,
                              uint32_t seed, uint8_t* out, int64_t* ts) {
  return guarded([&] { copy_frames(evsim::scenes::panning_texture(w, h, n, dx, dy, fps, seed), out, ts); });
}

int evsim_ref_moving_disk(int32_t w, int32_t h, int32_t n, double radius, double step, double fps,
                          uint8_t bg, uint8_t fg, uint32_t seed, uint8_t* out, int64_t* ts) {
  return guarded([&] {
    copy_frames(evsim::scenes::moving_disk(w, h, n, radius, step, fps, bg, fg, seed).frames, out, ts);
  });
}

int evsim_ref_translating_square(int32_t w, int32_t h, int32_t n, int32_t size, int32_t x0, int32_t y0,
                                 int32_t dx, int32_t dy, double fps, uint8_t* out, int64_t* ts) {
  return guarded([&] {
    copy_frames(evsim::scenes::translating_square(w, h, n, size, x0, y0, dx, dy, fps), out, ts);
  });
}

}  // extern "C"

// ---- frame ingestion, event files, metrics (io.cpp, metrics.cpp) ----------
namespace {
evsim::EventStream make_stream(const evsim_event* ev, int64_t n, int w, int h) {
  evsim::EventStream s{w, h, {}};
  s.events.resize(static_cast<std::size_t>(n));
  if (n) std::memcpy(s.events.data(), ev, static_cast<std::size_t>(n) * sizeof(evsim_event));
  return s;
}
}  // namespace

extern "C" {

uint8_t evsim_ref_luma_bt601(uint8_t r, uint8_t g, uint8_t b) { return evsim::luma_bt601(r, g, b); }

int evsim_ref_resize_bilinear(const uint8_t* src, int32_t w, int32_t h, int32_t tw, int32_t th, uint8_t* dst) {
  return guarded([&] {
    const evsim::Frame f = make_frame(src, w, h, 0);
    const evsim::Frame r = evsim::resize_bilinear(f, tw, th);
    std::memcpy(dst, r.pixels.data(), r.pixels.size());
  });
}

int evsim_ref_write_events_binary(const evsim_event* ev, int64_t n, int32_t w, int32_t h, const char* path) {
  return guarded([&] { evsim::write_events_binary(make_stream(ev, n, w, h), path); });
}

int evsim_ref_write_events_text(const evsim_event* ev, int64_t n, int32_t w, int32_t h, const char* path) {
  return guarded([&] { evsim::write_events_text(make_stream(ev, n, w, h), path); });
}

int evsim_ref_events_per_pixel_second(const evsim_event* ev, int64_t n, int32_t w, int32_t h, double duration,
                                      double* out3, uint64_t* total) {
  return guarded([&] {
    const evsim::EventRateStats st = evsim::events_per_pixel_second(make_stream(ev, n, w, h), duration);
    out3[0] = st.mean_rate;
    out3[1] = st.std_rate;
    out3[2] = st.duration;
    *total = st.total_events;
  });
}

int evsim_ref_accumulate(const evsim_event* ev, int64_t n, int32_t w, int32_t h, int64_t t0, int64_t t1,
                         uint8_t* classes) {
  return guarded([&] {
    const evsim::AccumulatedFrame a = evsim::accumulate(make_stream(ev, n, w, h), t0, t1);
    std::memcpy(classes, a.classes.data(), a.classes.size());
  });
}

}  // extern "C"
