// Exercise include/evsim_b200.hpp (the C++ drop-in for evsim::) through
// libevsim_gpu.so.
//   wrapper_check cpu                 host-only checks (no GPU needed)
//   wrapper_check gpu IN OUT1 OUT2    IN: "w h n method mode" header + n frames (u8) + n int64 stamps;
//                                     OUT1: events of push_frame x n, OUT2: events of push_frames
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

#include "evsim_b200.hpp"

namespace ev = evsim_b200;

static int fails = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                      \
    }                                                               \
  } while (0)

template <class E, class F>
static std::string throws_msg(F&& f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (...) {
    return "<other exception>";
  }
  return "<no exception>";
}

static int cpu_checks() {
  // SimulatorConfig::defaults  types.hpp:101-120
  const auto d = ev::SimulatorConfig::defaults(ev::Method::dense);
  EXPECT(d.c_pos == 2 && d.c_neg == -2 && d.n_interp == 10);
  const auto s = ev::SimulatorConfig::defaults(ev::Method::sparse);
  EXPECT(s.c_pos == 10 && s.c_neg == -10 && s.n_interp == 10 && s.effective_selection_threshold() == 10);
  // validate  types.hpp:126-130, exact messages
  ev::SimulatorConfig bad = d;
  bad.c_pos = 0;
  EXPECT(throws_msg<std::invalid_argument>([&] { bad.validate(); }) == "SimulatorConfig: c_pos must be > 0");
  bad = d;
  bad.n_interp = -1;
  EXPECT(throws_msg<std::invalid_argument>([&] { bad.validate(); }) == "SimulatorConfig: n_interp must be >= 0");
  EXPECT(throws_msg<std::invalid_argument>([&] { ev::FlowPreset{0, 1, 1}.validate(); }) ==
         "FlowPreset: all fields must be >= 1");
  EXPECT(ev::sub_interval_end(0, 1100, 1, 4) == 275);
  // luma_bt601  io.cpp:41-43 (values from the compiled reference)
  EXPECT(ev::luma_bt601(10, 200, 30) == 124 && ev::luma_bt601(255, 255, 255) == 255);
  EXPECT(throws_msg<std::invalid_argument>([&] { ev::Frame(0, 3, 0); }) == "Frame: width and height must be positive");
  std::puts(fails ? "cpu checks FAILED" : "cpu checks ok");
  return fails ? 1 : 0;
}

static int gpu_run(const char* in, const char* out1, const char* out2) {
  std::ifstream f(in, std::ios::binary);
  int w, h, n, method, mode;
  f.read(reinterpret_cast<char*>(&w), 4);
  f.read(reinterpret_cast<char*>(&h), 4);
  f.read(reinterpret_cast<char*>(&n), 4);
  f.read(reinterpret_cast<char*>(&method), 4);
  f.read(reinterpret_cast<char*>(&mode), 4);
  std::vector<ev::Frame> frames;
  for (int k = 0; k < n; ++k) {
    ev::Frame fr(w, h, 0);
    f.read(reinterpret_cast<char*>(fr.pixels.data()), (std::streamsize)fr.pixels.size());
    frames.push_back(std::move(fr));
  }
  for (int k = 0; k < n; ++k) f.read(reinterpret_cast<char*>(&frames[k].timestamp), 8);
  auto cfg = ev::SimulatorConfig::defaults(static_cast<ev::Method>(method));
  cfg.contrast_mode = static_cast<ev::ContrastMode>(mode);
  ev::Simulator a(cfg), b(cfg);
  ev::EventStream s1{w, h, {}};
  for (const auto& fr : frames) s1.append(a.push_frame(fr));
  const ev::EventStream s2 = b.push_frames(frames);
  // push_frame error semantics (simulate.cpp:307-318), state untouched
  EXPECT(throws_msg<std::invalid_argument>([&] { a.push_frame(frames.back()); }) ==
         "push_frame: timestamps must be strictly increasing");
  std::ofstream o1(out1, std::ios::binary), o2(out2, std::ios::binary);
  o1.write(reinterpret_cast<const char*>(s1.events.data()), (std::streamsize)(s1.events.size() * sizeof(ev::Event)));
  o2.write(reinterpret_cast<const char*>(s2.events.data()), (std::streamsize)(s2.events.size() * sizeof(ev::Event)));
  // io / metrics mirrors on the device: accumulate of the stream's own events
  // classifies every pixel that received an event in the window
  if (!s1.events.empty()) {
    const auto acc = ev::accumulate(s1, s1.events.front().t, s1.events.back().t + 1);
    std::size_t n_set = 0;
    for (auto c : acc.classes) n_set += c != ev::PixelClass::none;
    EXPECT(n_set > 0);
    const auto st = ev::events_per_pixel_second(s1, 1.0);
    EXPECT(st.total_events == s1.events.size() && st.mean_rate > 0.0);
  }
  const ev::Frame small = ev::resize_bilinear(frames[0], 17, 11);
  EXPECT(small.width == 17 && small.height == 11 && small.pixels.size() == 187);
  std::printf("gpu run ok: %zu / %zu events\n", s1.events.size(), s2.events.size());
  return fails ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "cpu") return cpu_checks();
  if (argc >= 5 && std::string(argv[1]) == "gpu") return gpu_run(argv[2], argv[3], argv[4]);
  std::fprintf(stderr, "usage: wrapper_check cpu | gpu IN OUT1 OUT2\n");
  return 2;
}
