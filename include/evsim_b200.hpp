// evsim_b200.hpp — C++ drop-in for the reference's evsim hot-path API,
// backed by the sm_100a library (libevsim_gpu.so, include/evsim_gpu.h).
//
// Same type, function and member names as the reference
// (/root/reference/proj/include/evsim/{types,flow,simulate}.hpp), same
// argument meaning, same exceptions and messages: code written against
// `evsim::` switches by changing the namespace (or `namespace evsim =
// evsim_b200;`).  Header-only; link with -levsim_gpu.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "evsim_gpu.h"

namespace evsim_b200 {

using time_us = std::int64_t;

// ---- types.hpp:14-131 -------------------------------------------------------
struct Frame {
  int width = 0;
  int height = 0;
  time_us timestamp = 0;
  std::vector<std::uint8_t> pixels;

  Frame() = default;
  Frame(int w, int h, time_us t, std::uint8_t fill = 0)
      : width(w), height(h), timestamp(t), pixels(static_cast<std::size_t>(w) * static_cast<std::size_t>(h), fill) {
    if (w <= 0 || h <= 0) throw std::invalid_argument("Frame: width and height must be positive");
  }
  std::uint8_t& at(int x, int y) { return pixels[static_cast<std::size_t>(y) * width + x]; }
  std::uint8_t at(int x, int y) const { return pixels[static_cast<std::size_t>(y) * width + x]; }
  std::size_t pixel_count() const { return static_cast<std::size_t>(width) * static_cast<std::size_t>(height); }
};

// Signed per-pixel intensity delta (types.hpp:33-46)
struct DifferenceFrame {
  int width = 0;
  int height = 0;
  time_us t_start = 0;
  time_us t_end = 0;
  std::vector<std::int16_t> values;

  DifferenceFrame() = default;
  DifferenceFrame(int w, int h, time_us t0, time_us t1)
      : width(w), height(h), t_start(t0), t_end(t1), values(static_cast<std::size_t>(w) * static_cast<std::size_t>(h), 0) {}
  std::int16_t& at(int x, int y) { return values[static_cast<std::size_t>(y) * width + x]; }
  std::int16_t at(int x, int y) const { return values[static_cast<std::size_t>(y) * width + x]; }
};

struct Event {
  std::uint16_t x = 0;
  std::uint16_t y = 0;
  time_us t = 0;
  std::int8_t p = 1;
  friend bool operator==(const Event& a, const Event& b) { return a.x == b.x && a.y == b.y && a.t == b.t && a.p == b.p; }
};
static_assert(sizeof(Event) == sizeof(evsim_event), "Event must keep evsim::Event's layout");

inline bool event_order(const Event& a, const Event& b) {
  if (a.t != b.t) return a.t < b.t;
  if (a.y != b.y) return a.y < b.y;
  if (a.x != b.x) return a.x < b.x;
  return a.p < b.p;
}

struct EventStream {
  int width = 0;
  int height = 0;
  std::vector<Event> events;
  void append(const EventStream& other) { events.insert(events.end(), other.events.begin(), other.events.end()); }
};

enum class Method { difference_only, dense, sparse, difference_interp };
enum class FlowQuality { low_quality, high_quality };
enum class EventsPerCrossing { single, magnitude };
enum class ContrastMode { linear, log };  // extension (BASELINE.json configs)

inline const char* method_name(Method m) {  // types.hpp:133-142
  switch (m) {
    case Method::difference_only: return "difference_only";
    case Method::dense: return "dense";
    case Method::sparse: return "sparse";
    case Method::difference_interp: return "difference_interp";
  }
  return "?";
}

struct SimulatorConfig {
  Method method = Method::difference_only;
  int c_pos = 2;
  int c_neg = -2;
  int n_interp = 0;
  FlowQuality flow_preset = FlowQuality::low_quality;
  int selection_threshold = 0;
  EventsPerCrossing events_per_crossing = EventsPerCrossing::single;
  bool include_endpoints = true;
  // extension
  ContrastMode contrast_mode = ContrastMode::linear;
  float c_pos_log = 0.2f;
  float c_neg_log = -0.2f;
  float sel_log = 0.0f;

  static SimulatorConfig defaults(Method m) {
    evsim_gpu_config c;
    evsim_gpu_config_defaults(static_cast<int32_t>(m), &c);
    return from_c(c);
  }
  int effective_selection_threshold() const { return selection_threshold > 0 ? selection_threshold : c_pos; }
  void validate() const;

  evsim_gpu_config to_c() const {
    evsim_gpu_config c{};
    c.method = static_cast<int32_t>(method);
    c.c_pos = c_pos;
    c.c_neg = c_neg;
    c.n_interp = n_interp;
    c.flow_preset = static_cast<int32_t>(flow_preset);
    c.selection_threshold = selection_threshold;
    c.events_per_crossing = static_cast<int32_t>(events_per_crossing);
    c.include_endpoints = include_endpoints ? 1 : 0;
    c.contrast_mode = static_cast<int32_t>(contrast_mode);
    c.c_pos_log = c_pos_log;
    c.c_neg_log = c_neg_log;
    c.sel_log = sel_log;
    return c;
  }
  static SimulatorConfig from_c(const evsim_gpu_config& c) {
    SimulatorConfig r;
    r.method = static_cast<Method>(c.method);
    r.c_pos = c.c_pos;
    r.c_neg = c.c_neg;
    r.n_interp = c.n_interp;
    r.flow_preset = static_cast<FlowQuality>(c.flow_preset);
    r.selection_threshold = c.selection_threshold;
    r.events_per_crossing = static_cast<EventsPerCrossing>(c.events_per_crossing);
    r.include_endpoints = c.include_endpoints != 0;
    r.contrast_mode = static_cast<ContrastMode>(c.contrast_mode);
    r.c_pos_log = c.c_pos_log;
    r.c_neg_log = c.c_neg_log;
    r.sel_log = c.sel_log;
    return r;
  }
};

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string msg = evsim_gpu_last_error();
  if (rc == EVSIM_GPU_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void check(int rc) {
  if (rc != EVSIM_GPU_OK) raise(rc);
}
}  // namespace detail

inline void SimulatorConfig::validate() const {
  const evsim_gpu_config c = to_c();
  detail::check(evsim_gpu_config_validate(&c));
}

// ---- core.hpp:8-19 -------------------------------------------------------------
inline DifferenceFrame difference_frame(const Frame& prev, const Frame& curr) {
  if (prev.width != curr.width || prev.height != curr.height)
    throw std::invalid_argument("difference_frame: incompatible input frames (" + std::to_string(prev.width) + "x" +
                                std::to_string(prev.height) + " vs " + std::to_string(curr.width) + "x" +
                                std::to_string(curr.height) + ")");
  DifferenceFrame d(prev.width, prev.height, prev.timestamp, curr.timestamp);
  if (!d.values.empty())
    detail::check(evsim_gpu_difference_frame(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                             d.values.data()));
  return d;
}

inline void threshold_events_into(const DifferenceFrame& diff, const SimulatorConfig& config, time_us event_time,
                                  std::vector<Event>& out) {
  const evsim_gpu_config c = config.to_c();
  int64_t n = 0;
  detail::check(evsim_gpu_threshold_events(diff.values.data(), diff.width, diff.height, &c, event_time, nullptr, 0, &n));
  const std::size_t at = out.size();
  out.resize(at + static_cast<std::size_t>(n));
  if (n)
    detail::check(evsim_gpu_threshold_events(diff.values.data(), diff.width, diff.height, &c, event_time,
                                             reinterpret_cast<evsim_event*>(out.data() + at), n, &n));
}

inline std::vector<Event> threshold_events(const DifferenceFrame& diff, const SimulatorConfig& config,
                                           time_us event_time) {
  std::vector<Event> out;
  threshold_events_into(diff, config, event_time, out);
  return out;
}

// ---- flow.hpp:9-110 ----------------------------------------------------------
struct FlowField {
  int width = 0;
  int height = 0;
  std::vector<float> du;
  std::vector<float> dv;
  FlowField() = default;
  FlowField(int w, int h)
      : width(w), height(h), du(static_cast<std::size_t>(w) * h, 0.0f), dv(static_cast<std::size_t>(w) * h, 0.0f) {}
  float u_at(int x, int y) const { return du[static_cast<std::size_t>(y) * width + x]; }
  float v_at(int x, int y) const { return dv[static_cast<std::size_t>(y) * width + x]; }
};

struct PixelPoint {
  int x = 0;
  int y = 0;
};
struct Displacement {
  float du = 0.0f;
  float dv = 0.0f;
};
struct SparseFlow {
  std::vector<PixelPoint> points;
  std::vector<Displacement> displacements;
  std::vector<std::uint8_t> status;
};

struct FlowPreset {
  int pyramid_levels = 3;
  int iterations_per_level = 2;
  int patch_radius = 4;
  void validate() const {
    if (pyramid_levels < 1 || iterations_per_level < 1 || patch_radius < 1)
      throw std::invalid_argument("FlowPreset: all fields must be >= 1");
  }
};

inline FlowPreset flow_preset(FlowQuality q) {
  return q == FlowQuality::low_quality ? FlowPreset{3, 2, 4} : FlowPreset{5, 16, 6};
}

inline void check_pair(const Frame& prev, const Frame& curr, const char* who) {
  if (prev.width <= 0 || prev.height <= 0 || curr.width <= 0 || curr.height <= 0)
    throw std::invalid_argument(std::string(who) + ": empty frame");
  if (prev.width != curr.width || prev.height != curr.height)
    throw std::invalid_argument(std::string(who) + ": incompatible input frames");
}

inline FlowField estimate_dense_flow(const Frame& prev, const Frame& curr, const FlowPreset& preset) {
  preset.validate();
  check_pair(prev, curr, "estimate_dense_flow");
  FlowField f(prev.width, prev.height);
  detail::check(evsim_gpu_dense_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                     preset.pyramid_levels, preset.iterations_per_level, preset.patch_radius,
                                     f.du.data(), f.dv.data()));
  return f;
}

inline SparseFlow estimate_sparse_flow(const Frame& prev, const Frame& curr, const std::vector<PixelPoint>& points,
                                       const FlowPreset& preset) {
  preset.validate();
  check_pair(prev, curr, "estimate_sparse_flow");
  SparseFlow out;
  out.points = points;
  out.displacements.assign(points.size(), Displacement{});
  out.status.assign(points.size(), 0);
  std::vector<int32_t> pts(points.size() * 2);
  for (std::size_t i = 0; i < points.size(); ++i) {
    pts[2 * i] = points[i].x;
    pts[2 * i + 1] = points[i].y;
  }
  detail::check(evsim_gpu_sparse_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                      preset.pyramid_levels, preset.iterations_per_level, preset.patch_radius,
                                      pts.data(), static_cast<int64_t>(points.size()),
                                      reinterpret_cast<float*>(out.displacements.data()), out.status.data()));
  return out;
}

class DenseFlowEstimator {
 public:
  virtual ~DenseFlowEstimator() = default;
  virtual FlowField estimate(const Frame& prev, const Frame& curr) const = 0;
};

class SparseFlowEstimator {
 public:
  virtual ~SparseFlowEstimator() = default;
  virtual SparseFlow estimate(const Frame& prev, const Frame& curr, const std::vector<PixelPoint>& points) const = 0;
};

class PyramidalPatchFlow final : public DenseFlowEstimator {
 public:
  explicit PyramidalPatchFlow(FlowPreset preset) : preset_(preset) { preset_.validate(); }
  FlowField estimate(const Frame& prev, const Frame& curr) const override {
    return estimate_dense_flow(prev, curr, preset_);
  }
  const FlowPreset& preset() const { return preset_; }

 private:
  FlowPreset preset_;
};

class PyramidalLucasKanade final : public SparseFlowEstimator {
 public:
  explicit PyramidalLucasKanade(FlowPreset preset) : preset_(preset) { preset_.validate(); }
  SparseFlow estimate(const Frame& prev, const Frame& curr, const std::vector<PixelPoint>& points) const override {
    return estimate_sparse_flow(prev, curr, points, preset_);
  }
  const FlowPreset& preset() const { return preset_; }

 private:
  FlowPreset preset_;
};

// ---- simulate.hpp:15-55 ------------------------------------------------------
inline time_us sub_interval_end(time_us t0, time_us t1, int k, int n_steps) {
  const time_us dt = t1 - t0;
  const time_us num = static_cast<time_us>(k) * dt;
  return t0 + (num + n_steps - 1) / n_steps;
}

inline std::vector<Frame> interpolate_frames(const Frame& prev, const Frame& curr, const FlowField& flow, int n) {
  if (prev.width != curr.width || prev.height != curr.height)
    throw std::invalid_argument("interpolate_frames: incompatible input frames");
  if (flow.width != prev.width || flow.height != prev.height)
    throw std::invalid_argument("interpolate_frames: flow dimensions do not match the frames");
  if (n < 0) throw std::invalid_argument("interpolate_frames: n must be >= 0");
  const std::size_t P = prev.pixel_count();
  std::vector<std::uint8_t> buf(P * static_cast<std::size_t>(n > 0 ? n : 1));
  std::vector<int64_t> ts(static_cast<std::size_t>(n > 0 ? n : 1));
  detail::check(evsim_gpu_interpolate_frames(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                             prev.timestamp, curr.timestamp, flow.du.data(), flow.dv.data(), n,
                                             buf.data(), ts.data()));
  std::vector<Frame> out;
  for (int k = 0; k < n; ++k) {
    Frame f(prev.width, prev.height, ts[k]);
    std::memcpy(f.pixels.data(), buf.data() + k * P, P);
    out.push_back(std::move(f));
  }
  return out;
}

namespace detail {
template <class F>
EventStream collect_events(int w, int h, F&& call) {
  int64_t n = 0;
  detail::check(call(nullptr, 0, &n));
  EventStream s{w, h, {}};
  s.events.resize(static_cast<std::size_t>(n));
  if (n) detail::check(call(reinterpret_cast<evsim_event*>(s.events.data()), n, &n));
  return s;
}
}  // namespace detail

inline EventStream dense_events_with_flow(const Frame& prev, const Frame& curr, const FlowField& flow,
                                          const SimulatorConfig& config) {
  config.validate();
  if (flow.width != prev.width || flow.height != prev.height)
    throw std::invalid_argument("interpolate_frames: flow dimensions do not match the frames");
  const evsim_gpu_config c = config.to_c();
  return detail::collect_events(prev.width, prev.height, [&](evsim_event* ev, int64_t cap, int64_t* n) {
    return evsim_gpu_dense_events_with_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                            prev.timestamp, curr.timestamp, flow.du.data(), flow.dv.data(), &c, ev,
                                            cap, n);
  });
}

inline EventStream sparse_events_with_flow(const Frame& prev, const Frame& curr, const SparseFlow& flow,
                                           const SimulatorConfig& config) {
  config.validate();
  std::vector<int32_t> pts(flow.points.size() * 2);
  for (std::size_t i = 0; i < flow.points.size(); ++i) {
    pts[2 * i] = flow.points[i].x;
    pts[2 * i + 1] = flow.points[i].y;
  }
  const evsim_gpu_config c = config.to_c();
  return detail::collect_events(prev.width, prev.height, [&](evsim_event* ev, int64_t cap, int64_t* n) {
    return evsim_gpu_sparse_events_with_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                             prev.timestamp, curr.timestamp, pts.data(),
                                             static_cast<int64_t>(flow.points.size()),
                                             reinterpret_cast<const float*>(flow.displacements.data()),
                                             flow.status.data(), &c, ev, cap, n);
  });
}

// simulate_dense (simulate.hpp:37-39, simulate.cpp:129-142): the flow from
// the estimator (default: PyramidalPatchFlow of config.flow_preset, on the
// GPU), interpolation and events on the GPU.
inline EventStream simulate_dense(const Frame& prev, const Frame& curr, const SimulatorConfig& config,
                                  const DenseFlowEstimator& estimator) {
  config.validate();
  check_pair(prev, curr, "simulate_dense");
  if (config.n_interp == 0) return dense_events_with_flow(prev, curr, FlowField(prev.width, prev.height), config);
  return dense_events_with_flow(prev, curr, estimator.estimate(prev, curr), config);
}
inline EventStream simulate_dense(const Frame& prev, const Frame& curr, const SimulatorConfig& config) {
  return simulate_dense(prev, curr, config, PyramidalPatchFlow(flow_preset(config.flow_preset)));
}

// simulate_sparse (simulate.hpp:44-46, simulate.cpp:144-201): selection as
// the reference, the tracks from the estimator (default PyramidalLucasKanade
// on the GPU), splat + chain on the GPU.
inline EventStream simulate_sparse(const Frame& prev, const Frame& curr, const SimulatorConfig& config,
                                   const SparseFlowEstimator& estimator) {
  config.validate();
  check_pair(prev, curr, "simulate_sparse");
  const int select = config.effective_selection_threshold();
  if (select <= 0) throw std::invalid_argument("simulate_sparse: selection threshold must be > 0");
  std::vector<PixelPoint> points;
  for (int y = 0; y < prev.height; ++y)
    for (int x = 0; x < prev.width; ++x) {
      const int d = static_cast<int>(curr.at(x, y)) - static_cast<int>(prev.at(x, y));
      if ((d < 0 ? -d : d) > select) points.push_back({x, y});
    }
  SparseFlow flow;
  if (!points.empty() && config.n_interp > 0) flow = estimator.estimate(prev, curr, points);
  return sparse_events_with_flow(prev, curr, flow, config);
}
inline EventStream simulate_sparse(const Frame& prev, const Frame& curr, const SimulatorConfig& config) {
  return simulate_sparse(prev, curr, config, PyramidalLucasKanade(flow_preset(config.flow_preset)));
}

// ---- simulate.hpp:60-94 ------------------------------------------------------
class Simulator {
 public:
  explicit Simulator(SimulatorConfig config, int device = 0) : config_(config) {
    const evsim_gpu_config c = config_.to_c();
    evsim_gpu_sim* h = nullptr;
    detail::check(evsim_gpu_create(&c, device, &h));
    h_.reset(h);
  }
  // Alternate flow backends (simulate.hpp:68-77): the flow comes from the
  // estimators; the stream's state (prev frame, log reference state) and
  // everything else stay on the GPU (evsim_gpu_push_frame_with_flow /
  // _with_tracks), so both contrast modes work through the seam.
  Simulator(SimulatorConfig config, std::shared_ptr<const DenseFlowEstimator> dense_flow,
            std::shared_ptr<const SparseFlowEstimator> sparse_flow, int device = 0)
      : config_(config), dense_(std::move(dense_flow)), sparse_(std::move(sparse_flow)), custom_(true) {
    config_.validate();
    if (!dense_ || !sparse_) throw std::invalid_argument("Simulator: flow estimators must not be null");
    if (config_.method == Method::difference_interp)
      throw std::invalid_argument("Simulator: custom flow estimators are not supported for difference_interp");
    const evsim_gpu_config c = config_.to_c();
    evsim_gpu_sim* h = nullptr;
    detail::check(evsim_gpu_create(&c, device, &h));
    h_.reset(h);
  }

  EventStream push_frame(const Frame& frame) {
    if (frame.width <= 0 || frame.height <= 0 || frame.pixels.size() != frame.pixel_count())
      throw std::invalid_argument("push_frame: malformed frame");
    if (custom_) return push_custom(frame);
    evsim_gpu_events ev{};
    detail::check(evsim_gpu_push_frame(h_.get(), frame.pixels.data(), frame.width, frame.height, frame.timestamp, 0,
                                       &ev));
    return collect(ev);
  }

  // Batched push (extension): identical to push_frame over each frame, with
  // the event streams concatenated.
  EventStream push_frames(const std::vector<Frame>& frames) {
    EventStream all{frames.empty() ? 0 : frames[0].width, frames.empty() ? 0 : frames[0].height, {}};
    if (frames.empty()) return all;
    if (custom_) {
      for (const auto& f : frames) all.append(push_frame(f));
      return all;
    }
    const int w = frames[0].width, hgt = frames[0].height;
    const std::size_t P = frames[0].pixel_count();
    const int cap = evsim_gpu_max_batch(h_.get(), w, hgt);
    for (std::size_t a = 0; a < frames.size(); a += cap) {
      const std::size_t nb = std::min<std::size_t>(cap, frames.size() - a);
      std::vector<std::uint8_t> px(nb * P);
      std::vector<int64_t> ts(nb);
      for (std::size_t k = 0; k < nb; ++k) {
        const Frame& f = frames[a + k];
        if (f.width != w || f.height != hgt || f.pixels.size() != P)
          throw std::invalid_argument("push_frame: malformed frame");
        std::memcpy(px.data() + k * P, f.pixels.data(), P);
        ts[k] = f.timestamp;
      }
      evsim_gpu_events ev{};
      detail::check(evsim_gpu_push_frames(h_.get(), px.data(), static_cast<int32_t>(nb), w, hgt, ts.data(), 0, &ev));
      all.append(collect(ev));
    }
    return all;
  }

  // write_events_binary / write_events_text (io.hpp:30-36) of the last push's
  // events, formatted on the device (library handle only).
  void write_events_binary(const std::string& path) {
    detail::check(evsim_gpu_write_events_binary(h_.get(), path.c_str()));
  }
  void write_events_text(const std::string& path) {
    detail::check(evsim_gpu_write_events_text(h_.get(), path.c_str()));
  }

  // Row band (evsim_gpu_set_row_band): emit only rows [y0, y1); stream start only.
  void set_row_band(int y0, int y1) {
    if (custom_) throw std::invalid_argument("set_row_band: not available with custom flow estimators");
    detail::check(evsim_gpu_set_row_band(h_.get(), y0, y1));
  }

  const SimulatorConfig& config() const { return config_; }
  void reset() {
    prev_.reset();
    detail::check(evsim_gpu_reset(h_.get()));
  }

 private:
  struct Deleter {
    void operator()(evsim_gpu_sim* s) const { evsim_gpu_destroy(s); }
  };

  EventStream collect(const evsim_gpu_events& ev) {
    EventStream s{ev.width, ev.height, {}};
    s.events.resize(static_cast<std::size_t>(ev.n_events));
    if (ev.n_events)
      detail::check(evsim_gpu_copy_events(h_.get(), s.events.data(), ev.n_events, 1));
    return s;
  }

  EventStream push_custom(const Frame& frame) {
    if (prev_) {
      if (frame.width != prev_->width || frame.height != prev_->height)
        throw std::invalid_argument("push_frame: frame dimensions changed mid-stream");
      if (frame.timestamp <= prev_->timestamp)
        throw std::invalid_argument("push_frame: timestamps must be strictly increasing");
    }
    evsim_gpu_events ev{};
    if (config_.method == Method::sparse && config_.n_interp > 0) {
      // the points the reference selects (simulate.cpp:150-157, scan order)
      // and the estimator's tracks for them
      std::vector<int32_t> pts;
      SparseFlow fl;
      if (prev_) {
        std::vector<PixelPoint> sel;
        const int t = config_.effective_selection_threshold();
        const bool logm = config_.contrast_mode == ContrastMode::log;
        float lut[256];
        if (logm) evsim_gpu_log_lut(lut);  // log mode: |L[curr] - L[prev]| > sel_log
        const float tl = config_.sel_log > 0.0f ? config_.sel_log : config_.c_pos_log;
        for (int y = 0; y < frame.height; ++y)
          for (int x = 0; x < frame.width; ++x) {
            const int a = prev_->at(x, y), c = frame.at(x, y);
            const bool take = logm ? std::fabs(lut[c] - lut[a]) > tl : (c - a < 0 ? a - c : c - a) > t;
            if (take) sel.push_back({x, y});
          }
        if (!sel.empty()) fl = sparse_->estimate(*prev_, frame, sel);
        pts.reserve(sel.size() * 2);
        for (const auto& p : sel) pts.push_back(p.x), pts.push_back(p.y);
      }
      detail::check(evsim_gpu_push_frame_with_tracks(
          h_.get(), frame.pixels.data(), frame.width, frame.height, frame.timestamp, pts.data(),
          static_cast<int64_t>(pts.size() / 2), reinterpret_cast<const float*>(fl.displacements.data()),
          fl.status.data(), &ev));
    } else {
      FlowField fl;
      const bool flow = prev_ && config_.method == Method::dense && config_.n_interp > 0;
      if (flow) fl = dense_->estimate(*prev_, frame);
      detail::check(evsim_gpu_push_frame_with_flow(h_.get(), frame.pixels.data(), frame.width, frame.height,
                                                   frame.timestamp, flow ? fl.du.data() : nullptr,
                                                   flow ? fl.dv.data() : nullptr, &ev));
    }
    prev_ = std::make_unique<Frame>(frame);
    return collect(ev);
  }

  SimulatorConfig config_;
  std::unique_ptr<evsim_gpu_sim, Deleter> h_;
  std::shared_ptr<const DenseFlowEstimator> dense_;
  std::shared_ptr<const SparseFlowEstimator> sparse_;
  bool custom_ = false;
  std::unique_ptr<Frame> prev_;
};

// simulate_difference (simulate.hpp:48-55, simulate.cpp:287-301): the
// difference_interp events of (f1, f2] from f1 - f0 and f2 - f1.
inline EventStream simulate_difference(const Frame& f0, const Frame& f1, const Frame& f2,
                                       const SimulatorConfig& config) {
  config.validate();
  if (f0.width != f1.width || f0.height != f1.height || f1.width != f2.width || f1.height != f2.height)
    throw std::invalid_argument("simulate_difference: incompatible input frames");
  if (!(f0.timestamp < f1.timestamp && f1.timestamp < f2.timestamp))
    throw std::invalid_argument("simulate_difference: timestamps must be strictly increasing");
  SimulatorConfig c = config;
  c.method = Method::difference_interp;
  Simulator sim(c);
  sim.push_frame(f0);
  sim.push_frame(f1);
  return sim.push_frame(f2);
}

// ---- io.hpp / metrics.hpp (the data formats either side of the path) -------
// luma_bt601 (io.cpp:41-43)
inline std::uint8_t luma_bt601(std::uint8_t r, std::uint8_t g, std::uint8_t b) {
  return static_cast<std::uint8_t>((299 * r + 587 * g + 114 * b + 500) / 1000);
}

// resize_bilinear (io.cpp:45-70), on the device
inline Frame resize_bilinear(const Frame& src, int width, int height) {
  if (width <= 0 || height <= 0) throw std::invalid_argument("resize_bilinear: target must be positive");
  Frame dst(width, height, src.timestamp);
  detail::check(evsim_gpu_ingest_frames(src.pixels.data(), 1, src.width, src.height, 1, width, height,
                                        dst.pixels.data()));
  return dst;
}

struct EventRateStats {  // metrics.hpp:9-14
  double mean_rate = 0.0;
  double std_rate = 0.0;
  double duration = 0.0;
  std::uint64_t total_events = 0;
};

enum class PixelClass : std::uint8_t { none = 0, positive = 1, negative = 2, both = 3 };

struct AccumulatedFrame {  // metrics.hpp:19-27
  int width = 0;
  int height = 0;
  time_us t_start = 0;
  time_us t_end = 0;
  std::vector<PixelClass> classes;
  PixelClass at(int x, int y) const { return classes[static_cast<std::size_t>(y) * width + x]; }
};

// events_per_pixel_second (metrics.cpp:7-39): counts on the device
inline EventRateStats events_per_pixel_second(const EventStream& stream, double duration) {
  EventRateStats st;
  detail::check(evsim_gpu_events_per_pixel_second(reinterpret_cast<const evsim_event*>(stream.events.data()),
                                                  static_cast<int64_t>(stream.events.size()), stream.width,
                                                  stream.height, duration, &st.mean_rate, &st.std_rate,
                                                  &st.total_events));
  st.duration = duration;
  return st;
}

// accumulate (metrics.cpp:41-69), on the device
inline AccumulatedFrame accumulate(const EventStream& stream, time_us t_start, time_us t_end) {
  AccumulatedFrame f;
  f.width = stream.width;
  f.height = stream.height;
  f.t_start = t_start;
  f.t_end = t_end;
  std::vector<std::uint8_t> cls(
      static_cast<std::size_t>(stream.width > 0 ? stream.width : 0) * (stream.height > 0 ? stream.height : 0));
  detail::check(evsim_gpu_accumulate(reinterpret_cast<const evsim_event*>(stream.events.data()),
                                     static_cast<int64_t>(stream.events.size()), stream.width, stream.height,
                                     t_start, t_end, cls.data()));
  f.classes.resize(cls.size());
  for (std::size_t i = 0; i < cls.size(); ++i) f.classes[i] = static_cast<PixelClass>(cls[i]);
  return f;
}

}  // namespace evsim_b200
