// flow_plugin_check.cpp — INTEGRATION.md §4 compiled for real: the GPU flow
// estimators plugged into the REFERENCE's own Simulator through its seam
// (include/evsim/simulate.hpp:68-77, flow.hpp:74-85), the reference linked
// from oracle/_ref/libevsim_ref.so (its sources compiled in place), the flow
// from libevsim_gpu.so.  The events must equal those of the reference's
// default CPU estimators (PyramidalPatchFlow / PyramidalLucasKanade) on the
// reference's own scenes, since the GPU flow is bit-exact.
//
// Built by oracle/Makefile (target `plugin`), run by tests/test_refsuite.py.
// Exit 0 and one summary line on success.
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <vector>

#include "evsim/scenes.hpp"
#include "evsim/simulate.hpp"
#include "evsim_gpu.h"

namespace {

class GpuPatchFlow final : public evsim::DenseFlowEstimator {
 public:
  explicit GpuPatchFlow(evsim::FlowPreset p) : p_(p) { p_.validate(); }
  evsim::FlowField estimate(const evsim::Frame& prev, const evsim::Frame& curr) const override {
    evsim::FlowField f(prev.width, prev.height);
    const int rc = evsim_gpu_dense_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                        p_.pyramid_levels, p_.iterations_per_level, p_.patch_radius, f.du.data(),
                                        f.dv.data());
    if (rc == EVSIM_GPU_INVALID_ARGUMENT) throw std::invalid_argument(evsim_gpu_last_error());
    if (rc != EVSIM_GPU_OK) throw std::runtime_error(evsim_gpu_last_error());
    return f;
  }

 private:
  evsim::FlowPreset p_;
};

class GpuLucasKanade final : public evsim::SparseFlowEstimator {
 public:
  explicit GpuLucasKanade(evsim::FlowPreset p) : p_(p) { p_.validate(); }
  evsim::SparseFlow estimate(const evsim::Frame& prev, const evsim::Frame& curr,
                             const std::vector<evsim::PixelPoint>& points) const override {
    evsim::SparseFlow out;
    out.points = points;
    out.displacements.assign(points.size(), evsim::Displacement{});
    out.status.assign(points.size(), 0);
    std::vector<int32_t> pts(points.size() * 2);
    for (std::size_t i = 0; i < points.size(); ++i) {
      pts[2 * i] = points[i].x;
      pts[2 * i + 1] = points[i].y;
    }
    const int rc = evsim_gpu_sparse_flow(prev.pixels.data(), curr.pixels.data(), prev.width, prev.height,
                                         p_.pyramid_levels, p_.iterations_per_level, p_.patch_radius, pts.data(),
                                         static_cast<int64_t>(points.size()),
                                         reinterpret_cast<float*>(out.displacements.data()), out.status.data());
    if (rc == EVSIM_GPU_INVALID_ARGUMENT) throw std::invalid_argument(evsim_gpu_last_error());
    if (rc != EVSIM_GPU_OK) throw std::runtime_error(evsim_gpu_last_error());
    return out;
  }

 private:
  evsim::FlowPreset p_;
};

int run(const char* name, evsim::SimulatorConfig cfg, const std::vector<evsim::Frame>& frames) {
  evsim::Simulator cpu(cfg);
  const auto preset = evsim::flow_preset(cfg.flow_preset);
  evsim::Simulator gpu(cfg, std::make_shared<GpuPatchFlow>(preset), std::make_shared<GpuLucasKanade>(preset));
  std::size_t n = 0;
  for (std::size_t k = 0; k < frames.size(); ++k) {
    const auto a = cpu.push_frame(frames[k]).events;
    const auto b = gpu.push_frame(frames[k]).events;
    if (a != b) {
      std::printf("[plugin] %s: frame %zu differs (%zu vs %zu events)\n", name, k, a.size(), b.size());
      return 1;
    }
    n += a.size();
  }
  std::printf("[plugin] %s: %zu frames, %zu events identical\n", name, frames.size(), n);
  return 0;
}

}  // namespace

int main() {
  int bad = 0;
  const auto pan = evsim::scenes::panning_texture(160, 120, 5, 3, 1, 20.0, 17);
  for (const auto q : {evsim::FlowQuality::low_quality, evsim::FlowQuality::high_quality}) {
    auto c = evsim::SimulatorConfig::defaults(evsim::Method::dense);
    c.flow_preset = q;
    bad += run(q == evsim::FlowQuality::low_quality ? "dense lq pan" : "dense hq pan", c, pan);
  }
  const auto disk = evsim::scenes::moving_disk(128, 96, 5, 6.0, 6.0, 100.0, 70, 235, 0);
  bad += run("sparse disk", evsim::SimulatorConfig::defaults(evsim::Method::sparse), disk.frames);
  auto m = evsim::SimulatorConfig::defaults(evsim::Method::dense);
  m.events_per_crossing = evsim::EventsPerCrossing::magnitude;
  m.include_endpoints = false;
  bad += run("dense magnitude no-endpoints", m, pan);
  std::printf("[plugin] %s\n", bad ? "FAILED" : "ok");
  return bad ? 1 : 0;
}
