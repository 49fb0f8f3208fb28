// evsim_gpu.cu — host side of the B200 event-simulation path: the C-ABI of
// include/evsim_gpu.h, the per-handle device state and the launch sequence.
//
// Mirrors evsim::Simulator (/root/reference/proj/include/evsim/simulate.hpp:60-94,
// src/simulate.cpp:306-347): same validation order and messages, same
// warm-up semantics, failed pushes leave the state untouched.  A push of F
// frames (push_frames; push_frame is F = 1) runs one launch sequence over the
// F frame pairs; frames live in a device ring, so the previous frame and its
// pyramid stay resident.  All device memory comes from the stream-ordered
// pool (cudaMallocAsync) with an unbounded release threshold, so a fresh
// handle per timed pass (the reference's bench_method, src/bench.cpp:53-64)
// reuses cached memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <thread>
#include <atomic>
#include <mutex>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>
#include <exception>

#include "evsim_gpu.h"
#include "kernels.h"

using namespace evsim_gpu;

namespace {

thread_local std::string g_err;

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] void invalid(const std::string& m) { throw ApiError{EVSIM_GPU_INVALID_ARGUMENT, m}; }
[[noreturn, maybe_unused]] void runtime(const std::string& m) { throw ApiError{EVSIM_GPU_RUNTIME, m}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ApiError{EVSIM_GPU_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) ck((x), #x)
#define CK_LAUNCH(what) ck(cudaGetLastError(), what)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return EVSIM_GPU_OK;
  } catch (const ApiError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return EVSIM_GPU_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EVSIM_GPU_RUNTIME;
  }
}

// ------------------------------------------------------------------ config

struct Preset {
  int levels, iters, radius;
};

Preset resolve_preset(const evsim_gpu_config& c) {
  if (c.pyramid_levels || c.iterations_per_level || c.patch_radius)
    return {c.pyramid_levels, c.iterations_per_level, c.patch_radius};
  // flow_preset(q)  include/evsim/flow.hpp:57-59
  return c.flow_preset == EVSIM_FLOW_HIGH_QUALITY ? Preset{5, 16, 6} : Preset{3, 2, 4};
}

void validate_preset(const Preset& p) {
  // FlowPreset::validate  include/evsim/flow.hpp:50-54
  if (p.levels < 1 || p.iters < 1 || p.radius < 1) invalid("FlowPreset: all fields must be >= 1");
  if (p.levels > kMaxLevels) invalid("FlowPreset: pyramid_levels above 8 are not supported");
}

void validate_config(const evsim_gpu_config& c) {
  // SimulatorConfig::validate  include/evsim/types.hpp:126-130
  if (c.c_pos <= 0) invalid("SimulatorConfig: c_pos must be > 0");
  if (c.c_neg >= 0) invalid("SimulatorConfig: c_neg must be < 0");
  if (c.n_interp < 0) invalid("SimulatorConfig: n_interp must be >= 0");
  if (c.contrast_mode != EVSIM_CONTRAST_LINEAR && c.contrast_mode != EVSIM_CONTRAST_LOG)
    invalid("SimulatorConfig: unknown contrast_mode");
  if (c.contrast_mode == EVSIM_CONTRAST_LOG) {
    if (!(c.c_pos_log > 0.0f)) invalid("SimulatorConfig: c_pos_log must be > 0");
    if (!(c.c_neg_log < 0.0f)) invalid("SimulatorConfig: c_neg_log must be < 0");
    if (c.events_per_crossing == EVSIM_EVENTS_MAGNITUDE) {
      // per-(pixel, link) counts are stored as u16: floor(|dL| / C) must fit
      const double span = std::log(1.0 + 1e-3) - std::log(1e-3);
      if (span / std::min<double>(c.c_pos_log, -c.c_neg_log) > 65535.0)
        invalid("SimulatorConfig: log contrast threshold too small for magnitude mode");
    }
  }
  if (c.method < EVSIM_METHOD_DIFFERENCE_ONLY || c.method > EVSIM_METHOD_DIFFERENCE_INTERP)
    invalid("SimulatorConfig: unknown method");
  if (c.method == EVSIM_METHOD_DIFFERENCE_INTERP && c.contrast_mode == EVSIM_CONTRAST_LOG)
    invalid("SimulatorConfig: difference_interp has no log contrast mode");
}

// The log rule as per-level thresholds for the dense chain:
// for every reference level r, pos <=> v > hi[r] and neg <=> v < lo[r], with
// the rule's own fp32 subtraction and comparisons (fsub(L[v], L[r]) is
// monotone in v, checked here).  Stored biased by kChainBias like the chain's
// values, with the level's own value: th[4r..4r+3] = (bias + hi, bias + lo,
// bits of L[r], 0).
void log_thresholds(const float* L, float c_pos, float c_neg, int32_t* th) {
  for (int r = 0; r < 256; ++r) {
    int hi = -1, lo = 256;
    bool seen_pos = false, seen_nonneg = false;
    for (int v = 0; v < 256; ++v) {
      const float d = L[v] - L[r];
      const bool pos = d > c_pos, neg = d < c_neg;
      if (pos) seen_pos = true;
      else if (seen_pos) runtime("log thresholds: rule not monotone");
      if (!pos) hi = v;
      if (!neg) seen_nonneg = true;
      else if (seen_nonneg) runtime("log thresholds: rule not monotone");
      if (!neg && lo == 256) lo = v;
    }
    th[4 * r] = kChainBias + hi;
    th[4 * r + 1] = kChainBias + lo;
    std::memcpy(&th[4 * r + 2], &L[r], 4);
    th[4 * r + 3] = 0;
  }
}

void log_lut(float* lut) {
  // L[i] = logf(i / 255 + 1e-3), evaluated once on the host so
  // every consumer (device kernels, CPU oracle) sees the same 256 floats.
  for (int i = 0; i < 256; ++i) lut[i] = std::log(static_cast<float>(i) / 255.0f + 1e-3f);
}

int64_t sub_interval_end(int64_t t0, int64_t t1, int k, int n) {
  // include/evsim/simulate.hpp:15-19
  const int64_t dt = t1 - t0;
  return t0 + (static_cast<int64_t>(k) * dt + n - 1) / n;
}

// ------------------------------------------------------------------ memory

void init_pool(int device) {
  static std::mutex m;
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(m);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // grow the pool once up front: the buffers of a handle / a stateless
    // call are then carved from reserved memory instead of mapping new pages
    // on the first call at a size (measured ~1 ms at 640x480)
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    void* p = nullptr;
    if (cudaMallocAsync(&p, (size_t)512 << 20, 0) == cudaSuccess) {
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    } else {
      cudaGetLastError();
    }
    cudaSetDevice(cur);
  }
  done[device] = true;
}

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t bytes, cudaStream_t st, bool zero = false) {
    if (bytes <= n && p) return;
    release();
    s = st;
    const size_t b = std::max<size_t>(bytes, 16);
    CK(cudaMallocAsync(&p, b, st));
    n = b;
    if (zero) CK(cudaMemsetAsync(p, 0, b, st));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ------------------------------------------------------------------ geometry

int effective_levels(int requested, int w, int h) {
  // flow.cpp:75-79 (kMinPyramidExtent = 8)
  int levels = std::max(1, requested);
  while (levels > 1 && (std::min(w, h) >> (levels - 1)) < 8) --levels;
  return levels;
}

std::vector<int> patch_centers(int extent, int radius, int stride) {
  // flow.cpp:97-107
  std::vector<int> c;
  if (extent <= 2 * radius + 1) {
    c.push_back((extent - 1) / 2);
    return c;
  }
  const int last = extent - 1 - radius;
  for (int v = radius; v <= last; v += stride) c.push_back(v);
  if (c.back() != last) c.push_back(last);
  return c;
}

void interp_table(const std::vector<int>& centers, int extent, std::vector<int>& idx, std::vector<float>& wgt) {
  // flow.cpp:111-128
  idx.assign(extent, 0);
  wgt.assign(extent, 0.0f);
  if (centers.size() < 2) return;
  int j = 0;
  for (int x = 0; x < extent; ++x) {
    if (x <= centers.front()) continue;
    if (x >= centers.back()) {
      idx[x] = static_cast<int>(centers.size()) - 2;
      wgt[x] = 1.0f;
      continue;
    }
    while (j + 2 < static_cast<int>(centers.size()) && centers[j + 1] <= x) ++j;
    idx[x] = j;
    wgt[x] = static_cast<float>(x - centers[j]) / static_cast<float>(centers[j + 1] - centers[j]);
  }
}

// Device-resident flow machinery for one resolution + preset: the pyramid
// ring (R frame slots), per-level patch grids (per pair) and static tables.
struct FlowEngine {
  int w = 0, h = 0;
  Preset preset{};
  int levels = 0;
  int R = 0, pairs = 0;
  LevelDims dims[kMaxLevels]{};
  DevBuf pyr[kMaxLevels];     // fp32 level images, R slots
  DevBuf qpyr[kMaxLevels];    // float4 quad images (4 bilinear taps per pixel), R slots
  DevBuf tex[kMaxLevels];     // sparse: float4 (value, gx, gy, 0) per pixel, R slots
  DevBuf tex8;                // sparse, level 0 from u8: packed texels (4 B per pixel), R slots
  bool texels = false;
  // dense with the warp-form solver at level 0: level 0 is read from the u8
  // frame / quad rings, so its fp32 image and float4 quads are not written
  bool u8_level0 = false;
  DevBuf tables[kMaxLevels];  // cx | cy | ix | wx | iy | wy
  DevBuf grid[kMaxLevels];    // per pair: pu | pv
  GridGeom geom[kMaxLevels]{};
  int jrange[kMaxLevels][2]{};  // patch rows solved per level (row bands; else the full grid)

  void setup(int w_, int h_, Preset p, bool want_texels, cudaStream_t s) {
    w = w_;
    h = h_;
    preset = p;
    texels = want_texels;
    levels = effective_levels(p.levels, w, h);
    dims[0] = {w, h};
    for (int l = 1; l < levels; ++l) dims[l] = {(dims[l - 1].w + 1) / 2, (dims[l - 1].h + 1) / 2};
    const int r = p.radius, stride = std::max(1, r);
    for (int l = 0; l < levels; ++l) {
      const int lw = dims[l].w, lh = dims[l].h;
      const auto cxs = patch_centers(lw, r, stride), cys = patch_centers(lh, r, stride);
      std::vector<int> ix, iy;
      std::vector<float> wx, wy;
      interp_table(cxs, lw, ix, wx);
      interp_table(cys, lh, iy, wy);
      const size_t ncx = cxs.size(), ncy = cys.size();
      std::vector<char> host((ncx + ncy + 2 * (size_t)lw + 2 * (size_t)lh) * 4);
      char* q = host.data();
      auto put = [&](const void* src, size_t bytes) {
        std::memcpy(q, src, bytes);
        q += bytes;
      };
      put(cxs.data(), ncx * 4);
      put(cys.data(), ncy * 4);
      put(ix.data(), (size_t)lw * 4);
      put(wx.data(), (size_t)lw * 4);
      put(iy.data(), (size_t)lh * 4);
      put(wy.data(), (size_t)lh * 4);
      tables[l].ensure(host.size(), s);
      CK(cudaMemcpyAsync(tables[l].p, host.data(), host.size(), cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));  // host vector goes out of scope
      GridGeom& g = geom[l];
      g.w = lw;
      g.h = lh;
      g.ncx = (int)ncx;
      g.ncy = (int)ncy;
      const int* base = tables[l].as<int>();
      g.cx = base;
      g.cy = base + ncx;
      g.ix = base + ncx + ncy;
      g.wx = reinterpret_cast<const float*>(base + ncx + ncy + lw);
      g.iy = base + ncx + ncy + 2 * lw;
      g.wy = reinterpret_cast<const float*>(base + ncx + ncy + 2 * lw + lh);
      g.pair_stride = 2 * ncx * ncy;
      jrange[l][0] = 0;
      jrange[l][1] = (int)ncy;
    }
    R = pairs = 0;
  }

  // Row band: the patch rows each level must solve so that the level-0 flow
  // of event rows [y0, y1) is identical to the full-frame solve.  Level 0:
  // densification reads grid rows iy[y], iy[y]+1 (flow.cpp:224-245); level
  // l+1: each needed level-l centre cy seeds from the densified coarse field
  // at sy = (cy + 0.5) * ry - 0.5 (flow.cpp:130-147), rows trunc(clamp(sy))
  // and +1, i.e. grid rows iy'[row], +1.  Solving a patch reads only the
  // (full) level images, so this is the whole dependency set.  Mirrors
  // parallel.band_plan.
  void plan_band(int y0, int y1) {
    const int r = preset.radius, stride = std::max(1, r);
    std::vector<std::vector<int>> cys(levels), iys(levels);
    for (int l = 0; l < levels; ++l) {
      cys[l] = patch_centers(dims[l].h, r, stride);
      std::vector<float> wy;
      interp_table(cys[l], dims[l].h, iys[l], wy);
    }
    std::vector<int> lo(levels, INT32_MAX), hi(levels, -1);
    auto add = [&](int l, int j) {
      j = std::min(j, (int)cys[l].size() - 1);
      lo[l] = std::min(lo[l], j);
      hi[l] = std::max(hi[l], j);
    };
    for (int y = y0; y < y1; ++y) {
      add(0, iys[0][y]);
      add(0, iys[0][y] + 1);
    }
    for (int l = 0; l + 1 < levels; ++l) {
      const int hf = dims[l].h, hc = dims[l + 1].h;
      const volatile float ry = (float)hc / (float)hf;
      for (int j = lo[l]; j <= hi[l]; ++j) {
        const volatile float t0 = (float)cys[l][j] + 0.5f;
        const volatile float t1 = t0 * ry;
        float sy = t1 - 0.5f;
        sy = std::min(std::max(sy, 0.0f), (float)(hc - 1));
        const int rr0 = (int)sy, rr1 = std::min(rr0 + 1, hc - 1);
        for (int rr : {rr0, rr1}) {
          add(l + 1, iys[l + 1][rr]);
          add(l + 1, iys[l + 1][rr] + 1);
        }
      }
    }
    for (int l = 0; l < levels; ++l) {
      jrange[l][0] = hi[l] >= 0 ? lo[l] : 0;
      jrange[l][1] = hi[l] >= 0 ? hi[l] + 1 : 0;
    }
  }

  void ensure(int R_, int pairs_, cudaStream_t s) {
    if (R_ > R) {
      for (int l = 0; l < levels; ++l) {
        const size_t pl = (size_t)dims[l].w * dims[l].h;
        pyr[l].release();
        qpyr[l].release();
        pyr[l].ensure((size_t)R_ * pl * sizeof(float), s);
        qpyr[l].ensure((size_t)R_ * pl * sizeof(float4), s);
        if (texels) {
          tex[l].release();
          tex[l].ensure((size_t)R_ * pl * sizeof(float4), s);
        }
      }
      if (texels) {
        tex8.release();
        tex8.ensure((size_t)R_ * dims[0].w * dims[0].h * sizeof(uint32_t), s);
      }
      R = R_;
    }
    if (pairs_ > pairs) {
      for (int l = 0; l < levels; ++l) {
        // zeroed: with row bands, tiles past the planned rows read seeds
        // from rows never solved (their results are never used)
        grid[l].ensure((size_t)pairs_ * geom[l].pair_stride * sizeof(float), s, true);
        geom[l].pu = grid[l].as<float>();
        geom[l].pv = grid[l].as<float>() + geom[l].pair_stride / 2;
      }
      pairs = pairs_;
    }
  }

  PyramidParams pyramid_params(const uint8_t* frames, size_t P, uint32_t* quad_u8, int slot0) const {
    PyramidParams p{};
    p.levels = levels;
    for (int l = 0; l < levels; ++l) {
      const size_t pl = (size_t)dims[l].w * dims[l].h;
      p.dims[l] = dims[l];
      p.pyr[l] = Ring<float>{pyr[l].as<float>(), pl};
      p.qpyr[l] = Ring<float4>{qpyr[l].as<float4>(), pl};
      p.tex[l] = Ring<float4>{texels ? tex[l].as<float4>() : nullptr, pl};
    }
    p.u8_level0 = (u8_level0 || texels) && quad_u8 != nullptr;
    if (texels && p.u8_level0) {
      // sparse: level 0 as the u8 quad + packed texels (the sparse solver
      // decodes them exactly), no fp32 level-0 images
      p.tex[0].base = nullptr;
      p.tex8 = Ring<uint32_t>{tex8.as<uint32_t>(), P};
    }
    p.frames = Ring<const uint8_t>{frames, P};
    p.quad_u8 = Ring<uint32_t>{quad_u8, P};
    p.R = R;
    p.slot0 = slot0;
    return p;
  }

  // estimate_dense_flow's level loop, flow.cpp:268-275, for n_pairs pairs;
  // result = per-pair level-0 patch grids
  // frames8 / quads8: the u8 frame and u8 quad rings (level 0 when u8_level0)
  // pair_off: the pairs' first grid slot (sub-batches of one launch)
  int solve(int r0, int n_pairs, const uint8_t* frames8, const uint32_t* quads8, cudaStream_t s, int pair_off = 0) {
    for (int l = levels - 1; l >= 0; --l) {
      DenseLKParams p{};
      if (l == 0 && u8_level0) {
        p.u8 = 1;
        p.prev8 = Ring<const uint8_t>{frames8, (size_t)w * h};
        p.qcurr8 = Ring<const uint32_t>{quads8, (size_t)w * h};
      }
      p.g = geom[l];
      p.g.pu += (size_t)pair_off * geom[l].pair_stride;
      p.g.pv += (size_t)pair_off * geom[l].pair_stride;
      p.has_coarse = l != levels - 1;
      if (p.has_coarse) {
        p.coarse = geom[l + 1];
        p.coarse.pu += (size_t)pair_off * geom[l + 1].pair_stride;
        p.coarse.pv += (size_t)pair_off * geom[l + 1].pair_stride;
      }
      const size_t pl = (size_t)dims[l].w * dims[l].h;
      p.prev = Ring<const float>{pyr[l].as<float>(), pl};
      p.qcurr = Ring<const float4>{qpyr[l].as<float4>(), pl};
      p.R = R;
      p.r0 = r0;
      p.radius = preset.radius;
      p.iterations = preset.iters;
      p.jt0 = jrange[l][0];
      p.jt1 = jrange[l][1];
      if (p.jt1 > p.jt0) launch_dense_lk(p, n_pairs, s);
    }
    CK_LAUNCH("dense_lk");
    return levels;
  }

  // quads8: the u8 quad ring the pyramid pass wrote (level 0 then comes
  // from it and the packed texels), or null (fp32 level 0)
  SparseLKParams sparse_params(int r0, const uint32_t* quads8) const {
    SparseLKParams p{};
    p.levels = levels;
    for (int l = 0; l < levels; ++l) {
      const size_t pl = (size_t)dims[l].w * dims[l].h;
      p.dims[l] = dims[l];
      p.tex[l] = Ring<const float4>{tex[l].as<float4>(), pl};
      p.qcurr[l] = Ring<const float4>{qpyr[l].as<float4>(), pl};
    }
    p.R = R;
    p.r0 = r0;
    p.w0 = w;
    p.h0 = h;
    p.radius = preset.radius;
    p.iterations = preset.iters;
    p.pair_stride = (size_t)w * h;
    p.u8_level0 = quads8 != nullptr;
    if (p.u8_level0) {
      p.tex8 = Ring<const uint32_t>{tex8.as<uint32_t>(), (size_t)w * h};
      p.qcurr8 = Ring<const uint32_t>{quads8, (size_t)w * h};
    }
    return p;
  }
};

// Chain / offsets / emit buffers for one resolution, links per pair and
// number of pairs.
struct EventEngine {
  int w = 0, h = 0, wpr = 0;
  int64_t n_words = 0;
  int wpb = 0, n_blocks = 0;
  int words_per_warp = 2;  // dense chain kernel
  int max_links = 0;  // links of a launch (pairs * per-pair links)
  bool magnitude = false;
  DevBuf masks, counts, prefix, link_total, segtab, segbase, seg_out, events, mcount, wcount, base, sched;
  DevBuf wplanes, wpol, wlinks, wbit;  // wire format of a streamed call (wire_kernels.cu)
  int64_t capacity = 0;

  // fine = true (dense): one word per warp, 8 words per block on frames up
  // to 1080p — finer tasks balance the few waves of a small frame (measured:
  // c2 chain 16.4 -> 15.0 us/frame; 1080p c4 124 -> 112)
  // tile = true (the tile-staged dense chain, csrc/event_kernels.cu): one
  // count block per tile row of kTileWords words
  static constexpr int kTileWords = 4, kTileRows = 8;
  void geometry(int w_, int h_, bool fine = false, bool tile = false) {
    w = w_;
    h = h_;
    wpr = (w + 31) / 32;
    n_words = (int64_t)h * wpr;
    if (tile) {
      words_per_warp = 1;
      wpb = kTileWords;
      n_blocks = (int)(n_words / wpb);
      max_links = 0;
      capacity = 0;
      return;
    }
    // ~8 resident blocks of 256 threads on each of the 148 SMs
    const int64_t target = 148 * 8;
    int64_t per = (n_words + target - 1) / target;
    per = std::max<int64_t>(kWarpsPerBlock, (per + kWarpsPerBlock - 1) / kWarpsPerBlock * kWarpsPerBlock);
    // a power of two (down): whole chain blocks tile the emit's 256-word
    // tiles without idle threads (stacked c1 x64: 160 -> 128-word blocks)
    {
      int64_t p2 = kWarpsPerBlock;
      while (p2 * 2 <= per) p2 *= 2;
      per = p2;
    }
    if (const char* e = std::getenv("EVSIM_WPB")) {  // A/B of the non-dense block size
      const int v = std::atoi(e);
      if (v >= kWarpsPerBlock && !fine) per = v;
    }
    words_per_warp = 2;
    if (fine) {
      // one-word warp tasks; 8-word blocks up to 8192 blocks, beyond that
      // ~45 blocks per SM (4K c5: 40-word blocks; chain 782 -> 707 and emit
      // 220 -> 201 µs/frame against 224-word blocks of two-word tasks)
      words_per_warp = 1;
      if ((n_words + 7) / 8 <= 8192) {
        per = 8;
      } else {
        const int64_t t = 148 * 45;
        per = (n_words + t - 1) / t;
        per = std::max<int64_t>(kWarpsPerBlock, (per + kWarpsPerBlock - 1) / kWarpsPerBlock * kWarpsPerBlock);
      }
    }
    wpb = (int)per;
    n_blocks = (int)((n_words + wpb - 1) / wpb);
    max_links = 0;
    capacity = 0;
  }

  void ensure(int links, bool mag, int64_t event_cap, cudaStream_t s) {
    links = std::max(links, 1);
    if (links > max_links || mag != magnitude) {
      max_links = links;
      magnitude = mag;
      masks.ensure((size_t)max_links * n_words * sizeof(uint2), s);
      counts.ensure((size_t)max_links * n_blocks * sizeof(uint32_t), s);
      prefix.ensure((size_t)max_links * n_blocks * sizeof(int64_t), s);
      link_total.ensure((size_t)max_links * sizeof(int64_t), s);
      segtab.ensure(16 + (size_t)max_links * (2 * sizeof(int) + sizeof(int64_t)), s);
      segbase.ensure((size_t)max_links * sizeof(int64_t), s);
      seg_out.ensure((3 + 2 * (size_t)max_links) * sizeof(int64_t), s);
      base.ensure(sizeof(int64_t), s);
      sched.ensure(sizeof(unsigned int), s);
      if (mag) {
        mcount.ensure((size_t)max_links * n_words * 32 * sizeof(uint16_t), s);
        wcount.ensure((size_t)max_links * n_words * sizeof(uint32_t), s);
      }
    }
    grow(event_cap, s);
  }

  void grow(int64_t cap, cudaStream_t s) {
    if (cap <= capacity) return;
    events.ensure((size_t)std::max<int64_t>(cap, 1) * sizeof(uint32_t), s);
    capacity = cap;
  }

  SegTable seg() const {
    SegTable t;
    char* b = static_cast<char*>(segtab.p);
    t.n_segs = reinterpret_cast<int*>(b);
    t.seg_t = reinterpret_cast<int64_t*>(b + 16);
    t.seg_first = reinterpret_cast<int*>(b + 16 + (size_t)max_links * 8);
    t.seg_nlinks = reinterpret_cast<int*>(b + 16 + (size_t)max_links * 12);
    return t;
  }
};

// Largest batch whose link count fits the kernels' shared-memory tables
// (chain: 4 B per link, emit: 8 B per segment, both <= 96 KB).
// Also keeps the per-launch event buffer + masks (12 B per link-pixel in
// single mode) within ~6 GB of the 180 GB HBM (24 GB for 4K and larger
// frames, so a push still holds several pairs: c5 669 -> 714 frames/s).
int max_batch_for(int links_per_pair, int64_t pixels) {
  const int L = std::max(links_per_pair, 1);
  const int by_links = 12000 / L;
  // (4K and larger frames: 24 GB, so a push holds several pairs and the
  // flow / chain overlap has sub-batches to work with)
  const int64_t budget = pixels >= ((int64_t)1 << 22) ? (int64_t)24e9 : (int64_t)6e9;
  const int64_t by_mem = budget / std::max<int64_t>(1, (int64_t)L * std::max<int64_t>(pixels, 1) * 12);
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::min(kMaxBatch, by_links), by_mem));
}

// Frames per wire call (evsim_gpu_push_frames_wire): its launches are
// chunks of <= max_batch_for pairs, so only the frame ring, the flow grids
// and the call's planes + polarity bits grow with F (~12 B per pixel per
// frame + 2 bits per pixel-link), kept within ~24 GB.
int max_wire_frames(int links_per_pair, int64_t pixels) {
  const int64_t L = std::max(links_per_pair, 1);
  const int64_t per_frame = std::max<int64_t>(pixels, 1) * 12 + L * std::max<int64_t>(pixels, 1) / 4;
  return (int)std::max<int64_t>(1, std::min<int64_t>(kMaxBatch, (int64_t)24e9 / per_frame));
}

}  // namespace

// ====================================================================== handle

struct evsim_gpu_sim {
  evsim_gpu_config cfg{};
  Preset preset{};
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;

  // stream state
  bool has_prev = false;
  int n_seen = 0;  // frames pushed since the stream start (difference_interp needs 2 before it emits)
  int w = 0, h = 0;
  int64_t prev_t = 0;
  int rhead = 0;  // ring slot of the previous frame
  int R = 0;      // ring slots allocated
  int pair_cap = 0;
  int launch_cap = 0;
  int band_y0 = 0, band_y1 = 0;  // row band of the events (0, 0 = the whole frame)

  DevBuf frames, quads, mags, lut, lthr, ref, consts, place_tab;
  std::vector<float4> h_kc;  // host copy of the chain constants kc (ChainParams::kcp)
  // dense method: the level-0 lerp quads of every ring slot, the dense
  // chain's gather source (no byte unpack, FFMA lerps)
  DevBuf quadf;
  // the dense chain's gather image: 0 = the u8 quads, 1 = fp32 lerp quads
  // (16 B/pixel, default), 2 = bf16 lerp quads (8 B/pixel: c5 log chain 604
  // -> 627 us/frame, L1 81 -> 52 % but +16 % instructions, issue 66 -> 75 %);
  // EVSIM_CHAIN_QUAD=u8|f4|bf16 selects (A/B and tests)
  // 3 = the top pairs (a00, a10 - a00) (8 B/pixel) staged per (tile, pair) in
  // shared memory by chain_dense_tile_kernel (single mode, even width,
  // 128-pixel tile columns).  Measured equal to the fp32 quads on c5 / c4
  // (the chain is issue-bound either way and the 4-word
  // count blocks cost the offsets scan 24 us/frame), so it is opt-in:
  // EVSIM_CHAIN_QUAD=tile selects it wherever the geometry allows
  int quad_req = [] {
    const char* e = std::getenv("EVSIM_CHAIN_QUAD");
    if (e && std::string(e) == "u8") return 0;
    if (e && std::string(e) == "f4") return 1;
    if (e && std::string(e) == "bf16") return 2;
    if (e && std::string(e) == "tile") return 3;
    return -1;
  }();
  int quad_kind = 1;
  // staging rows / resident blocks per SM of the tile kernel (EVSIM_TILE_BLOCKS=3|4)
  int tile_min_blocks = [] {
    const char* e = std::getenv("EVSIM_TILE_BLOCKS");
    return e && e[0] == '4' ? 4 : 3;
  }();
  bool tile_possible() const {
    return dense_flow() && !magnitude() && n_interp_eff() + 2 <= kMaxParamK && w % 2 == 0 &&
           ((w + 31) / 32) % EventEngine::kTileWords == 0;
  }
  void choose_quad_kind(int grid_h) {
    quad_kind = quad_req < 0 ? 1 : quad_req;
    if (quad_req == 3 && !tile_possible()) quad_kind = 1;
    if (quad_kind == 1 && w > kLerpQuadMaxW) quad_kind = 2;  // fp32 quads' tap-relative constants stay exact up to there
    (void)grid_h;
  }
  bool use_quadf() const { return dense_flow() && quad_kind != 0; }
  size_t quad_bytes() const { return quad_kind == 1 ? sizeof(float4) : sizeof(uint2); }
  void launch_quads(int slot0, int n, cudaStream_t st) {
    const size_t P = (size_t)w * h;
    const Ring<const uint8_t> fr{frames.as<uint8_t>(), P};
    if (quad_kind == 1) launch_lerp_quads(fr, Ring<float4>{quadf.as<float4>(), P}, w, h, R, slot0, n, st);
    else if (quad_kind == 3) launch_lerp_quads_f2(fr, Ring<float2>{quadf.as<float2>(), P}, w, h, R, slot0, n, st);
    else launch_lerp_quads_bf16(fr, Ring<uint2>{quadf.as<uint2>(), P}, w, h, R, slot0, n, st);
  }
  FlowEngine flow;
  EventEngine ev;
  // sparse (per pair)
  DevBuf sel_masks, sel_counts, sel_prefix, sel_total, points, n_points, disp, status, claims, touched, svals, dvals;

  // last result
  int64_t* h_seg_out = nullptr;  // pinned
  size_t h_seg_cap = 0;
  std::vector<int64_t> seg_t, seg_off;
  int64_t n_events = 0;
  bool pending = false;
  EmitParams last_emit{};

  // dense flow / chain pipeline of one push: the flow of sub-batch b+1 runs
  // on s_flow while the chain of sub-batch b runs on `stream` (the chain's
  // per-pixel state orders the chains; the flows are independent)
  cudaStream_t s_flow = nullptr;
  // dense: the chain's lerp quads of a push's frames are built on s_quad
  // beside the pyramid and flow (HBM-bound next to compute-bound work); the
  // chain waits for ev_qdone
  cudaStream_t s_quad = nullptr;
  cudaEvent_t ev_qin = nullptr, ev_qdone = nullptr;
  std::vector<cudaEvent_t> pipe_ev;  // [0]: inputs ready; [1 + b]: flow of sub-batch b done
  // streamed call (dense): a chunk's pyramid and flow also run on s_flow,
  // after its upload, so they overlap the previous chunk's chain and emit;
  // each chunk's pairs use their own grid slots from pair_base
  bool xchunk = false;
  int pair_base = 0;

  // wire format (evsim_gpu_push_frames_wire): the chain masks of each launch
  // become planes + polarity bits instead of packed events
  bool wire_on = false;
  // EVSIM_EMIT_LEGACY=1: the general (segment, word) emit for every launch
  // (A/B measurement and tests of both paths)
  bool emit_legacy = [] {
    const char* e = std::getenv("EVSIM_EMIT_LEGACY");
    return e && e[0] == '1';
  }();
  int64_t wire_link0 = 0;                // links of the call before this launch
  int64_t* wire_host_links = nullptr;    // pinned: this launch's (bit[G], count[G])
  std::vector<int64_t> wire_t;           // timestamps of the call's links
  int64_t* h_wl[2] = {nullptr, nullptr};
  size_t h_wl_cap = 0;

  // per-stage CUDA-event timing (evsim_gpu_set_profiling)
  using EvGroup = std::array<cudaEvent_t, EVSIM_N_STAGES + 1>;
  bool profiling = false;
  std::vector<EvGroup> ev_pool, ev_pending;
  EvGroup* cur_group = nullptr;
  int next_mark = 0;
  double stage_ms[EVSIM_N_STAGES] = {};
  int64_t timed_pushes = 0;

  ~evsim_gpu_sim() {
    if (stream) cudaStreamSynchronize(stream);
    if (h_seg_out) cudaFreeHost(h_seg_out);
    for (auto& b : h_seg2)
      if (b) cudaFreeHost(b);
    for (auto& b : h_wl)
      if (b) cudaFreeHost(b);
    if (s_flow) cudaStreamSynchronize(s_flow), cudaStreamDestroy(s_flow);
    if (s_quad) cudaStreamSynchronize(s_quad), cudaStreamDestroy(s_quad);
    if (ev_qin) cudaEventDestroy(ev_qin);
    if (ev_qdone) cudaEventDestroy(ev_qdone);
    for (auto e : pipe_ev) cudaEventDestroy(e);
    if (s_in) cudaStreamSynchronize(s_in), cudaStreamDestroy(s_in);
    if (s_out) cudaStreamSynchronize(s_out), cudaStreamDestroy(s_out);
    for (auto& g : ev_pool)
      for (auto e : g) cudaEventDestroy(e);
    for (auto& g : ev_pending)
      for (auto e : g) cudaEventDestroy(e);
  }

  // ---- profiling -----------------------------------------------------------
  void begin_group() {
    if (!profiling) return;
    EvGroup g;
    if (!ev_pool.empty()) {
      g = ev_pool.back();
      ev_pool.pop_back();
    } else {
      for (auto& e : g) CK(cudaEventCreate(&e));
    }
    ev_pending.push_back(g);
    cur_group = &ev_pending.back();
    next_mark = 0;
  }
  // record stage boundary i (and any skipped ones) at the current stream position
  void mark(int i) {
    if (!cur_group) return;
    for (; next_mark <= i; ++next_mark) CK(cudaEventRecord((*cur_group)[next_mark], stream));
  }
  void end_group() {
    if (!cur_group) return;
    mark(EVSIM_N_STAGES);
    cur_group = nullptr;
  }
  void collect() {
    for (auto& g : ev_pending) {
      CK(cudaEventSynchronize(g[EVSIM_N_STAGES]));
      for (int i = 0; i < EVSIM_N_STAGES; ++i) {
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, g[i], g[i + 1]));
        stage_ms[i] += ms;
      }
      ++timed_pushes;
      ev_pool.push_back(g);
    }
    ev_pending.clear();
  }

  // ---- configuration -------------------------------------------------------
  int n_interp_eff() const { return cfg.method == EVSIM_METHOD_DIFFERENCE_ONLY ? 0 : cfg.n_interp; }
  bool dense_flow() const { return cfg.method == EVSIM_METHOD_DENSE && n_interp_eff() > 0; }
  bool sparse_flow() const { return cfg.method == EVSIM_METHOD_SPARSE && n_interp_eff() > 0; }
  bool diff_interp() const { return cfg.method == EVSIM_METHOD_DIFFERENCE_INTERP; }
  bool di_flow() const { return diff_interp() && n_interp_eff() > 0; }
  bool splats() const { return sparse_flow() || di_flow(); }  // point selection + sparse LK + splat
  bool uses_flow() const { return dense_flow() || splats(); }
  // frames a push keeps besides its own: prev, and for difference_interp the
  // frame before it (the previous difference frame, simulate.cpp:334-341)
  int kept_frames() const { return diff_interp() ? 2 : 1; }
  bool log_mode() const { return cfg.contrast_mode == EVSIM_CONTRAST_LOG; }
  bool magnitude() const { return cfg.events_per_crossing == EVSIM_EVENTS_MAGNITUDE; }

  // chain_pipeline (simulate.cpp:57-69): which chain frames the links join
  ChainDesc desc() const {
    const int N = n_interp_eff();
    if (cfg.method == EVSIM_METHOD_DIFFERENCE_ONLY) return ChainDesc{0, 1, 1};
    // difference_interp: warped difference frames 1..N, then d2 (endpoints)
    if (diff_interp()) return ChainDesc{0, 1, N + (cfg.include_endpoints ? 1 : 0)};
    if (N == 0) return ChainDesc{0, 1, cfg.include_endpoints ? 1 : 0};
    if (cfg.include_endpoints) return ChainDesc{0, 1, N + 1};
    return ChainDesc{1, 1, std::max(0, N - 1)};
  }

  // ---- allocation ----------------------------------------------------------
  void allocate(int w_, int h_) {
    if (band_y1 > h_) invalid("set_row_band: the band lies outside the frame");
    w = w_;
    h = h_;
    R = 0;
    pair_cap = 0;
    launch_cap = 0;
    rhead = 0;
    const bool band = band_y1 > 0;
    if (uses_flow()) {
      flow.setup(w, h, preset, splats(), stream);
      {
        const int r = preset.radius;
        flow.u8_level0 = dense_flow() && (r == 4 || r == 6) && w > 2 * r + 1 && h > 2 * r + 1;
      }
      if (band && dense_flow()) flow.plan_band(band_y0, band_y1);
    }
    if (log_mode()) ref.ensure((size_t)w * h * sizeof(float), stream);
    choose_quad_kind(band ? band_y1 - band_y0 : h);
    ev.geometry(w, band ? band_y1 - band_y0 : h, dense_flow(), dense_flow() && quad_kind == 3);
    // interpolation constants, interpolate_frames simulate.cpp:97-100
    const int N = n_interp_eff();
    const int K = N + 2;
    std::vector<char> host((size_t)K * (16 + 8 + 8 + 4 + 4 + 4 + 4 + 8));
    float* kc = reinterpret_cast<float*>(host.data());  // K float4 first (16-byte aligned)
    double* alpha = reinterpret_cast<double*>(kc + 4 * K);
    double* oma = alpha + K;
    float* fwd = reinterpret_cast<float*>(oma + K);
    float* bwd = fwd + K;
    float* alpha_f = bwd + K;
    float* oma_f = alpha_f + K;
    float* nfb = oma_f + K;  // K float2, 8-byte aligned (K*8*2 + K*4*4 bytes before it)
    for (int k = 0; k < K; ++k) {
      const double a = static_cast<double>(k) / static_cast<double>(N + 1);
      alpha[k] = a;
      oma[k] = 1.0 - a;
      fwd[k] = static_cast<float>(a);
      bwd[k] = static_cast<float>(1.0 - a);
      alpha_f[k] = static_cast<float>(a);
      oma_f[k] = static_cast<float>(1.0 - a);
      nfb[2 * k] = -fwd[k];
      nfb[2 * k + 1] = bwd[k];
      kc[4 * k + 0] = -fwd[k];
      kc[4 * k + 1] = bwd[k];
      kc[4 * k + 2] = oma_f[k];
      kc[4 * k + 3] = alpha_f[k];
    }
    h_kc.assign(reinterpret_cast<const float4*>(kc), reinterpret_cast<const float4*>(kc) + K);
    consts.ensure(host.size(), stream);
    CK(cudaMemcpyAsync(consts.p, host.data(), host.size(), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
  }

  // room for `pairs` pairs in one call (ring of pairs + kept_frames() slots,
  // flow grids per pair) whose launches hold at most `launch_pairs` pairs
  // (chain masks, tables, splat buffers; 0 = pairs) and whose events need
  // `event_cap` device records (-1 = every link-pixel of the call)
  void ensure_capacity(int pairs, int launch_pairs = 0, int64_t event_cap = -1) {
    if (launch_pairs <= 0) launch_pairs = pairs;
    const size_t P = (size_t)w * h;
    const int keep = kept_frames();
    const int need_R = pairs + keep;
    if (need_R > R) {
      // grow the ring; the kept frames move to slots 0 .. keep-1 (prev last)
      const int have = std::min(n_seen, keep);  // kept frames that exist
      DevBuf nf;
      nf.ensure((size_t)need_R * P + 16, stream);
      for (int j = 0; j < have; ++j) {
        const int src = (rhead - (have - 1 - j) + R) % std::max(R, 1);
        CK(cudaMemcpyAsync(nf.as<uint8_t>() + (size_t)(keep - have + j) * P, frames.as<uint8_t>() + (size_t)src * P,
                           P, cudaMemcpyDeviceToDevice, stream));
      }
      std::swap(frames.p, nf.p);
      std::swap(frames.n, nf.n);
      std::swap(frames.s, nf.s);
      if (uses_flow()) {  // u8 quads of level 0 (dense: frames; sparse / difference_interp: the pyramid source)
        DevBuf nq;
        nq.ensure((size_t)need_R * P * 4, stream);
        if (has_prev)
          CK(cudaMemcpyAsync(nq.as<uint32_t>() + (size_t)(keep - 1) * P, quads.as<uint32_t>() + (size_t)rhead * P,
                             P * 4, cudaMemcpyDeviceToDevice, stream));
        std::swap(quads.p, nq.p);
        std::swap(quads.n, nq.n);
        std::swap(quads.s, nq.s);
      }
      if (use_quadf()) {  // (prev's lerp quads are rebuilt below)
        quadf.release();
        quadf.ensure((size_t)need_R * P * quad_bytes(), stream);
      }
      if (diff_interp()) {
        DevBuf nm;
        nm.ensure((size_t)need_R * P + 16, stream);
        if (n_seen >= 2)
          CK(cudaMemcpyAsync(nm.as<uint8_t>() + (size_t)(keep - 1) * P, mags.as<uint8_t>() + (size_t)rhead * P, P,
                             cudaMemcpyDeviceToDevice, stream));
        std::swap(mags.p, nm.p);
        std::swap(mags.n, nm.n);
        std::swap(mags.s, nm.s);
      }
      if (uses_flow()) {
        // pyramid of prev (difference_interp: of prev's difference magnitude)
        // rebuilt from the image below (cheap, exact)
        flow.ensure(need_R, std::max(pairs, 1), stream);
      }
      rhead = keep - 1;
      R = need_R;
      if (uses_flow() && has_prev && (!diff_interp() || n_seen >= 2)) {
        const uint8_t* src = diff_interp() ? mags.as<uint8_t>() : frames.as<uint8_t>();
        PyramidParams pp = flow.pyramid_params(src, P, quads.as<uint32_t>(), rhead);
        launch_pyramid(pp, 1, stream);
        CK_LAUNCH("pyramid");
        if (use_quadf()) {
          launch_quads(rhead, 1, stream);
          CK_LAUNCH("lerp_quads");
        }
      }
    }
    if (pairs > pair_cap) {
      if (uses_flow()) flow.ensure(R, pairs, stream);
      pair_cap = pairs;
    }
    const int L = desc().n_links;
    if (launch_pairs > launch_cap) {
      ev.ensure(L * launch_pairs, magnitude(), 0, stream);
      const int pairs = launch_pairs;
      if (splats()) {
        const int N = n_interp_eff();
        sel_masks.ensure((size_t)pairs * ev.n_words * 4, stream);
        sel_counts.ensure((size_t)pairs * ev.n_blocks * 4, stream);
        sel_prefix.ensure((size_t)pairs * ev.n_blocks * 8, stream);
        sel_total.ensure((size_t)pairs * 8, stream);
        points.ensure((size_t)pairs * P * 4, stream);
        n_points.ensure((size_t)pairs * sizeof(int), stream, true);
        disp.ensure((size_t)pairs * P * sizeof(float2), stream);
        status.ensure((size_t)pairs * P, stream);
        claims.release();
        claims.ensure((size_t)pairs * N * P * 4, stream, true);
        if (diff_interp()) {
          dvals.release();
          dvals.ensure((size_t)pairs * N * P * 2, stream);
        } else {
          svals.release();
          svals.ensure((size_t)pairs * N * P, stream);
        }
        touched.release();
        touched.ensure((size_t)pairs * ((N + 31) / 32) * P * 4, stream, true);
      }
      const size_t seg_need = (3 + 2 * (size_t)ev.max_links) * sizeof(int64_t);
      if (seg_need > h_seg_cap) {
        if (h_seg_out) cudaFreeHost(h_seg_out);
        h_seg_out = nullptr;
        CK(cudaHostAlloc((void**)&h_seg_out, seg_need, cudaHostAllocDefault));
        h_seg_cap = seg_need;
      }
      launch_cap = launch_pairs;
    }
    if (event_cap < 0) event_cap = (int64_t)std::max(L, 1) * pairs * (int64_t)P;
    // (magnitude mode grows the buffer on demand, finish())
    if (!magnitude() || ev.capacity == 0) ev.grow(event_cap, stream);
  }

  // ---- chain params --------------------------------------------------------
  ChainParams chain_params(int r0, int n_pairs) {
    ChainParams c{};
    const int N = n_interp_eff();
    const size_t P = (size_t)w * h;
    c.w = w;
    c.h = h;
    c.row0 = band_y1 > 0 ? band_y0 : 0;
    c.wpr = ev.wpr;
    c.n_words = ev.n_words;
    c.words_per_block = ev.wpb;
    c.n_blocks = ev.n_blocks;
    c.words_per_warp = ev.words_per_warp;
    c.n_interp = N;
    c.n_pairs = n_pairs;
    c.R = R;
    c.r0 = r0;
    c.frames = Ring<const uint8_t>{frames.as<uint8_t>(), P};
    c.quads = Ring<const uint32_t>{quads.as<uint32_t>(), P};
    c.quadf = Ring<const float4>{use_quadf() && quad_kind == 1 ? quadf.as<float4>() : nullptr, P};
    c.quadh = Ring<const uint2>{use_quadf() && quad_kind == 2 ? quadf.as<uint2>() : nullptr, P};
    c.quadt = Ring<const float2>{use_quadf() && quad_kind == 3 ? quadf.as<float2>() : nullptr, P};
    // staging rows: what 3 (4) resident blocks per SM leave of the 227 KB
    // after the kernel's static shared memory (~8 KB) and the per-block reserve
    c.tile_min_blocks = tile_min_blocks;
    c.tile_cap_rows = tile_min_blocks >= 4 ? 42 : 58;
    {
      // gather index of the dense chain: TY_bits * w + TX_bits with TX =
      // 2^23 + x, TY = 2^23 + m_y + y (fp32 bits); it equals y * w + x +
      // qshift without wrapping when qshift + P <= 2^32.  m_y = 0 almost
      // always; otherwise the smallest m_y that wraps qshift below w (it
      // exists for every frame the size checks accept)
      const uint64_t M = 0x4B000000ull, w64 = (uint64_t)w;
      uint64_t m = 0, K = (M * w64 + M) & 0xFFFFFFFFull;
      // EVSIM_TEST_MAGIC_Y=1 forces the m_y > 0 form (tested on small frames)
      const char* force = std::getenv("EVSIM_TEST_MAGIC_Y");
      const uint64_t m_wrap = ((1ull << 32) - K + w64 - 1) / w64;
      if (K + P > (1ull << 32) || (force && force[0] == '1' && m_wrap + (uint64_t)h <= (1ull << 23))) {
        m = m_wrap;
        K = (K + m * w64) & 0xFFFFFFFFull;
      }
      if (m + (uint64_t)h > (1ull << 23) || K + P > (1ull << 32)) runtime("push_frame: no gather bias for this frame size");
      c.magic_y = (float)(8388608ull + m);
      c.qshift = (uint32_t)K;
    }
    const int K = N + 2;
    c.kc = consts.as<float4>();
    for (int k = 0; k < std::min(K, kMaxParamK); ++k) c.kcp[k] = h_kc[k];
    c.alpha = reinterpret_cast<const double*>(c.kc + K);
    c.oma = c.alpha + K;
    c.fwd = reinterpret_cast<const float*>(c.alpha + 2 * K);
    c.bwd = c.fwd + K;
    c.alpha_f = c.bwd + K;
    c.oma_f = c.alpha_f + K;
    c.nfb = reinterpret_cast<const float2*>(c.oma_f + K);
    c.P = P;
    c.d = desc();
    c.log_mode = log_mode();
    c.magnitude = magnitude();
    c.c_pos = cfg.c_pos;
    c.c_neg = cfg.c_neg;
    c.c_pos_log = cfg.c_pos_log;
    c.c_neg_log = cfg.c_neg_log;
    c.lut = lut.as<float>();
    c.lthr = lthr.as<int4>();
    c.ref = ref.as<float>();
    c.masks = ev.masks.as<uint2>();
    c.mcount = ev.mcount.as<uint16_t>();
    c.wcount = ev.wcount.as<uint32_t>();
    c.counts = ev.counts.as<uint32_t>();
    c.masks_cap = (size_t)ev.max_links * (size_t)ev.n_words;
    c.counts_cap = (size_t)ev.max_links * (size_t)ev.n_blocks;
    c.sched = ev.sched.as<unsigned int>();
    return c;
  }

  // segments -> chain -> offsets -> segbase + emit, then the segment-table
  // readback.  ts: n_pairs + 1 frame timestamps.
  // continue_call: this launch's events follow those of the previous launch of
  // the same call (streamed chunks); otherwise they start at offset 0.
  // sub: sub-batch boundaries (pairs) when the flow is pipelined (empty: one
  // chain launch); the chain of sub-batch b waits for pipe_ev[1 + b]
  void run_events(ChainParams& c, int provider, const int64_t* ts, int64_t* h_seg, bool continue_call = false,
                  const std::vector<int>& sub = {}) {
    const int G = c.d.n_links * c.n_pairs;
    const int L = c.d.n_links;
    if (!continue_call) CK(cudaMemsetAsync(ev.base.p, 0, sizeof(int64_t), stream));
    SegParams sp{};
    sp.d = c.d;
    sp.n_pairs = c.n_pairs;
    sp.n_interp = c.n_interp;
    sp.seg = ev.seg();
    for (int i = 0; i <= c.n_pairs; ++i) sp.ts[i] = ts[i];
    launch_segments(sp, stream);
    CK_LAUNCH("segments");
    EmitParams ep{};
    ep.w = w;
    ep.h = h;
    ep.row0 = c.row0;
    ep.wpr = ev.wpr;
    ep.wdiv = FastDiv::make((uint32_t)ev.wpr);
    ep.n_words = ev.n_words;
    ep.words_per_block = ev.wpb;
    ep.n_blocks = ev.n_blocks;
    ep.n_links = G;
    ep.seg = ev.seg();
    ep.prefix = ev.prefix.as<int64_t>();
    ep.counts = ev.counts.as<uint32_t>();
    ep.link_total = ev.link_total.as<int64_t>();
    ep.seg_out = ev.seg_out.as<int64_t>();
    ep.base = ev.base.as<int64_t>();
    ep.magnitude = c.magnitude;
    ep.masks = ev.masks.as<uint2>();
    ep.mcount = ev.mcount.as<uint16_t>();
    ep.wcount = ev.wcount.as<uint32_t>();
    ep.capacity = ev.capacity;
    ep.out = ev.events.as<uint32_t>();
    // offsets + segment bases + emit of links [g0, g1) (segments = links when
    // every link has its own timestamp)
    // every link its own timestamp (no finalize() run spans two links) and
    // one event per crossing: segment g = link g, tile-staged emit
    bool single = !c.magnitude;
    {
      const int K = c.n_interp + 1;
      int64_t tp = 0;
      for (int g = 0; single && g < G; ++g) {
        const int i = g / L, l = g % L;
        const int k = c.d.start + (l + 1) * c.d.step;
        const int64_t t = k == K ? ts[i + 1] : sub_interval_end(ts[i], ts[i + 1], k, K);
        if (g > 0 && t == tp) single = false;
        tp = t;
      }
    }
    auto emit_links = [&](int g0, int g1, bool range) {
      OffsetParams op{g1 - g0, ev.n_blocks, ev.counts.as<uint32_t>() + (size_t)g0 * ev.n_blocks,
                      ev.prefix.as<int64_t>() + (size_t)g0 * ev.n_blocks, ev.link_total.as<int64_t>() + g0};
      launch_offsets(op, stream);
      CK_LAUNCH("offsets");
      mark(EVSIM_STAGE_EMIT);
      EmitParams e = ep;
      e.seg_lo = range ? g0 : 0;
      e.seg_hi = range ? g1 : 0;
      if (wire_on) {
        // wire format: segment table as usual, then planes + polarity bits
        // of links [0, G) instead of packed events (called once per launch)
        launch_segbase(e, ev.segbase.as<int64_t>(), stream);
        CK_LAUNCH("segbase");
        WireParams wp{};
        wp.n_links = G;
        wp.n_words = ev.n_words;
        wp.words_per_block = ev.wpb;
        wp.n_blocks = ev.n_blocks;
        wp.blocks_per_tile = std::max(1, 256 / std::max(1, ev.wpb));
        wp.masks = ev.masks.as<uint2>();
        wp.prefix = ev.prefix.as<int64_t>();
        wp.link_total = ev.link_total.as<int64_t>();
        wp.link_bit = ev.wlinks.as<int64_t>() + wire_link0;
        wp.link_count = ev.wlinks.as<int64_t>() + (ev.wlinks.n / 16) + wire_link0;
        wp.bit_base = ev.wbit.as<int64_t>();
        wp.planes = ev.wplanes.as<uint32_t>() + (size_t)wire_link0 * ev.n_words;
        wp.pol = ev.wpol.as<uint32_t>();
        launch_wire(wp, stream);
        CK_LAUNCH("wire");
        CK(cudaMemcpyAsync(wire_host_links, wp.link_bit, (size_t)G * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(wire_host_links + G, wp.link_count, (size_t)G * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           stream));
        launches += 1;  // segbase + linkbase + wire vs segbase + emit
        return;
      }
      if (!(single && !emit_legacy && launch_emit_single(e, ev.segbase.as<int64_t>(), g0, g1, stream)))
        launch_emit(e, ev.segbase.as<int64_t>(), stream);
      CK_LAUNCH("emit");
    };
    if (wire_on) {
      const int K = c.n_interp + 1;
      for (int g = 0; g < G; ++g) {
        const int i = g / L, l = g % L;
        const int k = c.d.start + (l + 1) * c.d.step;
        wire_t.push_back(k == K ? ts[i + 1] : sub_interval_end(ts[i], ts[i + 1], k, K));
      }
    }
    if (sub.empty()) {
      launch_chain(c, provider, stream);
      CK_LAUNCH("chain");
      mark(EVSIM_STAGE_SCAN);
      emit_links(0, G, false);
    } else {
      // every link its own timestamp (no collisions, one event per
      // crossing): sub-batch b's events are emitted right after its chain —
      // a link's output offset only needs the totals of the links before it.
      // The emit runs on `stream` before the next sub-batch's chain, so it
      // fills the time that chain would wait for its flow on s_flow (the
      // flows run ahead on s_flow; the chains and emits stay in order)
      // (not in the streamed call: its chunks already overlap the emit with
      // the next chunk's flow, and per-sub-batch emits measured slower there)
      const bool split = single && !continue_call && !wire_on;
      for (size_t b = 0; b + 1 < sub.size(); ++b) {
        const int off = sub[b], nb = sub[b + 1] - sub[b];
        CK(cudaStreamWaitEvent(stream, pipe_ev[1 + b], 0));
        ChainParams cb = c;
        cb.r0 = c.r0 + off;
        cb.n_pairs = nb;
        cb.g0.pu += (size_t)off * c.g0.pair_stride;
        cb.g0.pv += (size_t)off * c.g0.pair_stride;
        cb.masks += (size_t)off * L * ev.n_words;
        cb.counts += (size_t)off * L * ev.n_blocks;
        if (c.magnitude) {
          cb.mcount += (size_t)off * L * ev.n_words * 32;
          cb.wcount += (size_t)off * L * ev.n_words;
        }
        launch_chain(cb, provider, stream);
        CK_LAUNCH("chain");
        if (split) emit_links(off * L, (off + nb) * L, true);
      }
      launches += (int64_t)sub.size() - 2;
      if (split) launches += 3 * ((int64_t)sub.size() - 2);
      mark(EVSIM_STAGE_SCAN);
      if (!split) emit_links(0, G, false);
    }
    launches += 6;
    if (wire_on) wire_link0 += G;
    CK(cudaMemcpyAsync(h_seg, ev.seg_out.p, (3 + 2 * (size_t)G) * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    last_emit = ep;
    pending = true;
  }

  // ---- push ----------------------------------------------------------------
  // Simulator::push_frame (src/simulate.cpp:306-347) applied to F frames in
  // order; the whole batch is validated first and rejected atomically.
  void validate_batch(const uint8_t* pixels, int F, int fw, int fh, const int64_t* ts, bool wire = false,
                      bool custom_push = false) const {
    if (custom && has_prev && !custom_push) invalid(kCustomMsg);
    if (F < 1) invalid("push_frames: n_frames must be >= 1");
    if (fw <= 0 || fh <= 0 || !pixels || !ts) invalid("push_frame: malformed frame");
    if (has_prev) {
      if (fw != w || fh != h) invalid("push_frame: frame dimensions changed mid-stream");
      if (ts[0] <= prev_t) invalid("push_frame: timestamps must be strictly increasing");
    }
    for (int j = 1; j < F; ++j)
      if (ts[j] <= ts[j - 1]) invalid("push_frame: timestamps must be strictly increasing");
    if (fh > 32768 || fw > 65536) invalid("push_frame: frame larger than 65536 x 32768 is not supported");
    if ((int64_t)fw * fh >= (int64_t)1 << 24 && cfg.method == EVSIM_METHOD_SPARSE)
      invalid("push_frame: frames of 2^24 pixels or more are not supported by the sparse method");
    if ((int64_t)fw * fh >= (int64_t)1 << 31) invalid("push_frame: frame too large");
    const int L = desc().n_links;
    const int fmax = wire ? max_wire_frames(L, (int64_t)fw * fh) : max_batch_for(L, (int64_t)fw * fh);
    if (F > fmax) invalid("push_frames: batch too large (max " + std::to_string(fmax) + ")");
  }

  // device state for F more frames of one call (launches of <= launch_pairs
  // pairs, event_cap device event records; see ensure_capacity)
  void prepare(int F, int fw, int fh, int launch_pairs = 0, int64_t event_cap = -1) {
    CK(cudaSetDevice(device));
    // A queued single-mode result is superseded (stream order keeps the
    // device buffers consistent); magnitude mode may need a re-emit.
    if (pending) {
      if (magnitude()) finish();
      else pending = false;
    }
    if (!has_prev && (fw != w || fh != h)) allocate(fw, fh);
    const int n_pairs = has_prev ? F : F - 1;
    ensure_capacity(std::max(n_pairs, 1), launch_pairs, event_cap);
  }

  // ring slot of the first frame of the next push
  int next_slot() const { return has_prev ? (rhead + 1) % R : rhead; }

  // Upload F frames into the ring from slot `base` (at most two contiguous runs).
  void upload(const uint8_t* pixels, int F, int base, bool on_device, cudaStream_t s) {
    const size_t P = (size_t)w * h;
    const int first = std::min(F, R - base);
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(frames.as<uint8_t>() + (size_t)base * P, pixels, (size_t)first * P, kind, s));
    if (first < F)
      CK(cudaMemcpyAsync(frames.as<uint8_t>(), pixels + (size_t)first * P, (size_t)(F - first) * P, kind, s));
  }

  void push(const uint8_t* pixels, int F, int fw, int fh, const int64_t* ts, bool on_device) {
    validate_batch(pixels, F, fw, fh, ts);
    prepare(F, fw, fh);
    enqueue(pixels, F, ts, on_device, nullptr, h_seg_out, false);
  }

  // ---- push with caller-supplied flow ---------------------------------------
  // Simulator::push_frame with the flow from a caller's DenseFlowEstimator /
  // SparseFlowEstimator (include/evsim/simulate.hpp:68-77): the handle keeps
  // the stream's state (prev frame, log reference state) exactly as for its
  // own flow; only the flow comes from the caller — the dense field of
  // (prev, frame), or the tracks of the points the reference selects
  // (simulate.cpp:150-157, scan order).  A handle fed this way takes only
  // such pushes until reset() (its frames get no pyramids).
  bool custom = false;
  static constexpr const char* kCustomMsg =
      "push_frame: this simulator is fed caller-supplied flow (push_frame_with_flow); reset() first";
  DevBuf field;
  void push_custom(const uint8_t* pixels, int fw, int fh, int64_t t, const float* du, const float* dv,
                   const int32_t* pts, int64_t n_pts, const float* disp, const uint8_t* st) {
    validate_batch(pixels, 1, fw, fh, &t, false, true);
    if (diff_interp()) invalid("Simulator: custom flow estimators are not supported for difference_interp");
    const size_t P = (size_t)fw * fh;
    std::vector<uint32_t> idx;
    if (has_prev && sparse_flow()) {
      if (n_pts < 0 || (n_pts > 0 && (!pts || !disp || !st))) invalid("push_frame_with_tracks: malformed tracks");
      if ((uint64_t)n_pts > P) invalid("push_frame_with_tracks: more points than pixels");
      idx.resize((size_t)std::max<int64_t>(n_pts, 1));
      for (int64_t i = 0; i < n_pts; ++i) {
        const int x = pts[2 * i], y = pts[2 * i + 1];
        if (x < 0 || x >= fw || y < 0 || y >= fh) invalid("simulate_sparse: point outside frame bounds");
        idx[i] = (uint32_t)y * (uint32_t)fw + (uint32_t)x;
        if (i && idx[i] <= idx[i - 1]) invalid("push_frame_with_tracks: points must be in scan order");
      }
    }
    if (has_prev && dense_flow() && (!du || !dv)) invalid("push_frame_with_flow: null flow field");
    prepare(1, fw, fh);
    custom = true;
    const int base = next_slot();
    upload(pixels, 1, base, false, stream);
    if (dense_flow()) {  // the u8 quads the field-form interpolation samples
      launch_build_quad(frames.as<uint8_t>() + (size_t)base * P, quads.as<uint32_t>() + (size_t)base * P, w, h, stream);
      CK_LAUNCH("build_quad");
      ++launches;
    }
    if (!has_prev) {  // warm-up frame
      if (log_mode()) {
        launch_init_ref(frames.as<uint8_t>() + (size_t)base * P, lut.as<float>(), ref.as<float>(), (int64_t)P, stream);
        CK_LAUNCH("init_ref");
        ++launches;
      }
      seg_t.clear();
      seg_off.assign(1, 0);
      n_events = 0;
      pending = false;
    } else {
      ChainParams c = chain_params(rhead, 1);
      c.quadf = Ring<const float4>{nullptr, P};
      c.quadh = Ring<const uint2>{nullptr, P};
      int provider = kProvNone;
      if (dense_flow()) {
        field.ensure(P * 8, stream);
        CK(cudaMemcpyAsync(field.p, du, P * 4, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(field.as<float>() + P, dv, P * 4, cudaMemcpyHostToDevice, stream));
        c.du = field.as<float>();
        c.dv = field.as<float>() + P;
        provider = kProvDenseField;
      } else if (sparse_flow()) {
        const int np = (int)n_pts;
        if (np > 0) {
          CK(cudaMemcpyAsync(points.p, idx.data(), (size_t)np * 4, cudaMemcpyHostToDevice, stream));
          CK(cudaMemcpyAsync(this->disp.p, disp, (size_t)np * 8, cudaMemcpyHostToDevice, stream));
          CK(cudaMemcpyAsync(this->status.p, st, (size_t)np, cudaMemcpyHostToDevice, stream));
        }
        CK(cudaMemcpyAsync(n_points.p, &np, sizeof np, cudaMemcpyHostToDevice, stream));
        splat_stage(rhead, 1, c);
        launches += 2;
        provider = kProvSparse;
      }
      const int64_t ts2[2] = {prev_t, t};
      run_events(c, provider, ts2, h_seg_out);
      CK(cudaStreamSynchronize(stream));  // (the host staging above must outlive its copies)
    }
    rhead = base;
    prev_t = t;
    has_prev = true;
    n_seen += 1;
  }


  // Everything of one push after validation: upload (unless `uploaded` says
  // the frames are already in the ring), pyramid, flow, chain, emit.
  void enqueue(const uint8_t* pixels, int F, const int64_t* ts, bool on_device, cudaEvent_t uploaded, int64_t* h_seg,
               bool continue_call) {
    const size_t P = (size_t)w * h;
    const int base = next_slot();  // ring slot of frame 0 of the batch
    const int n_pairs = has_prev ? F : F - 1;
    const bool xc = xchunk && dense_flow() && uploaded && !profiling && s_flow;
    cudaStream_t ps = xc ? s_flow : stream;  // upload wait + pyramid
    begin_group();
    mark(EVSIM_STAGE_UPLOAD);
    // difference_only from device memory: the chain reads the caller's frames
    // in place and only the last one is kept in the ring (the next push's prev)
    const bool direct = on_device && !uploaded && !profiling && cfg.method == EVSIM_METHOD_DIFFERENCE_ONLY &&
                        !magnitude() && n_interp_eff() == 0;
    if (uploaded) CK(cudaStreamWaitEvent(ps, uploaded, 0));
    else if (!direct) upload(pixels, F, base, on_device, stream);
    mark(EVSIM_STAGE_PYRAMID);
    bool quad_side = false;
    if (use_quadf()) {
      if (profiling) {
        launch_quads(base, F, ps);  // (stage timing: serialised, counted as pyramid)
      } else {
        if (!s_quad) {
          int lo = 0, hi = 0;
          CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          CK(cudaStreamCreateWithPriority(&s_quad, cudaStreamNonBlocking, hi));
          CK(cudaEventCreateWithFlags(&ev_qin, cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&ev_qdone, cudaEventDisableTiming));
        }
        quad_side = true;  // launched after the pyramid (below)
      }
      ++launches;
    }
    // the lerp quads on s_quad, after the pyramid (beside the LK solve;
    // starting them beside the pyramid measured the same on c2 / c5)
    auto side_quads = [&]() {
      CK(cudaEventRecord(ev_qin, ps));
      CK(cudaStreamWaitEvent(s_quad, ev_qin, 0));
      launch_quads(base, F, s_quad);
      CK(cudaEventRecord(ev_qdone, s_quad));
      CK_LAUNCH("lerp_quads");
    };
    if (diff_interp()) {
      // difference magnitudes of the new frames that have a predecessor, and
      // (for the sparse solver) their pyramids
      const int j0 = n_seen == 0 ? 1 : 0;
      const int slot0 = (base + j0) % R;
      if (F - j0 > 0) {
        launch_mags(Ring<const uint8_t>{frames.as<uint8_t>(), P}, Ring<uint8_t>{mags.as<uint8_t>(), P}, R, slot0,
                    F - j0, P, stream);
        CK_LAUNCH("mags");
        ++launches;
        if (uses_flow()) {
          PyramidParams pp = flow.pyramid_params(mags.as<uint8_t>(), P, quads.as<uint32_t>(), slot0);
          launch_pyramid(pp, F - j0, stream);
          CK_LAUNCH("pyramid");
          launches += flow.levels;
        }
      }
    } else if (uses_flow()) {
      PyramidParams pp = flow.pyramid_params(frames.as<uint8_t>(), P, quads.as<uint32_t>(), base);
      launch_pyramid(pp, F, ps);
      CK_LAUNCH("pyramid");
      launches += flow.levels;
    }
    if (quad_side) side_quads();
    if (!has_prev && log_mode()) {
      // warm-up frame: ref := L(frame0)
      if (xc) CK(cudaStreamWaitEvent(stream, uploaded, 0));
      launch_init_ref(direct ? pixels : frames.as<uint8_t>() + (size_t)base * P, lut.as<float>(), ref.as<float>(),
                      (int64_t)P, stream);
      CK_LAUNCH("init_ref");
      ++launches;
    }
    mark(EVSIM_STAGE_FLOW);
    const int r0 = has_prev ? rhead : base;
    std::vector<int64_t> pts(n_pairs + 1);
    if (has_prev) {
      pts[0] = prev_t;
      for (int j = 0; j < F; ++j) pts[j + 1] = ts[j];
    } else {
      for (int j = 0; j < F; ++j) pts[j] = ts[j];
    }
    if (n_pairs > 0) {
      ChainParams c = chain_params(r0, n_pairs);
      if (direct) {
        c.dprev = has_prev ? frames.as<uint8_t>() + (size_t)rhead * P : pixels;
        c.dcurr = has_prev ? pixels : pixels + P;
      }
      int provider = kProvNone;
      std::vector<int> sub;
      if (dense_flow()) {
        // simulate_dense -> PyramidalPatchFlow -> dense_events_with_flow (simulate.cpp:130-143)
        c.g0 = flow.geom[0];
        const int pb = xc ? pair_base : 0;  // this call's grid slots of the chunk
        c.g0.pu += (size_t)pb * c.g0.pair_stride;
        c.g0.pv += (size_t)pb * c.g0.pair_stride;
        provider = kProvDenseGrid;
        // sub-batches of >= 8 pairs, at most 4; stage timing serialises
        // (measured on c2: 2, 4, 8 sub-batches within 1 %; 4 + the stream
        // priority: 33.2k -> 34.1k frames/s)
        // (4K pushes of 7 pairs in sub-batches of 1-2: 714 -> 710 frames/s, so
        // sub-batches stay >= 8 pairs)
        const int nsb = profiling ? 1 : std::min(4, n_pairs / 8);
        if (nsb < 2 && !xc) {
          launches += flow.solve(r0, n_pairs, frames.as<uint8_t>(), quads.as<uint32_t>(), stream);
        } else {
          const int ns = std::max(nsb, 1);
          if (!s_flow) CK(cudaStreamCreateWithFlags(&s_flow, cudaStreamNonBlocking));
          while ((int)pipe_ev.size() < ns + 1) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            pipe_ev.push_back(e);
          }
          if (!xc) {  // (xc: the pyramid already ran on s_flow)
            CK(cudaEventRecord(pipe_ev[0], stream));
            CK(cudaStreamWaitEvent(s_flow, pipe_ev[0], 0));
          }
          for (int b = 0; b <= ns; ++b) sub.push_back((int)((int64_t)n_pairs * b / ns));
          for (int b = 0; b < ns; ++b) {
            launches += flow.solve(r0 + sub[b], sub[b + 1] - sub[b], frames.as<uint8_t>(), quads.as<uint32_t>(),
                                   s_flow, pb + sub[b]);
            CK(cudaEventRecord(pipe_ev[1 + b], s_flow));
          }
        }
      } else if (sparse_flow()) {
        sparse_stage(r0, n_pairs, c);
        provider = kProvSparse;
      } else if (diff_interp()) {
        // difference_interp_events (simulate.cpp:212-285); pair 0 has no
        // previous difference frame while the stream holds < 2 frames
        c.skip_first = n_seen < 2;
        if (di_flow()) sparse_stage(r0, n_pairs, c);
        provider = kProvDiffInterp;
      }
      mark(EVSIM_STAGE_CHAIN);
      if (quad_side) CK(cudaStreamWaitEvent(stream, ev_qdone, 0));
      run_events(c, provider, pts.data(), h_seg, continue_call, sub);
    } else {
      // (no chain: the handle's stream still orders after the quad build, so
      // a later ring growth never frees the quads under it)
      if (quad_side) CK(cudaStreamWaitEvent(stream, ev_qdone, 0));
      if (!continue_call) {
        seg_t.clear();
        seg_off.assign(1, 0);
        n_events = 0;
      }
      pending = false;
    }
    if (direct)  // the last frame into its ring slot (the next push's prev)
      CK(cudaMemcpyAsync(frames.as<uint8_t>() + (size_t)((base + F - 1) % R) * P, pixels + (size_t)(F - 1) * P, P,
                         cudaMemcpyDeviceToDevice, stream));
    end_group();
    rhead = (base + F - 1) % R;
    prev_t = ts[F - 1];
    has_prev = true;
    n_seen += F;
  }

  // ---- streamed push: host frames in, host events out ---------------------
  // F frames in chunks of `chunk`: the upload of chunk j+1 (copy-in stream)
  // and the download of chunk j-1's events (copy-out stream) overlap the
  // compute of chunk j.  Events land contiguously, exactly as one push of
  // all F frames would leave them (segbase continues the call's offset).
  // Single-event mode only (the output bound L*pairs*P is exact there).
  cudaStream_t s_in = nullptr, s_out = nullptr;
  int64_t* h_seg2[2] = {nullptr, nullptr};
  size_t h_seg2_cap = 0;
  bool host_short = false;

  void push_streamed(const uint8_t* pixels, int F, int fw, int fh, const int64_t* ts, int chunk, uint32_t* host_dst,
                     int64_t capacity, evsim_gpu_wire* wire = nullptr) {
    if (magnitude()) invalid("push_frames_streamed: magnitude mode is not supported (use push_frames)");
    if (!wire && !host_dst && capacity > 0) invalid("push_frames_streamed: null destination");
    if (wire && ((!wire->planes && wire->planes_capacity > 0) || (!wire->polarity && wire->polarity_capacity > 0) ||
                 (wire->link_capacity > 0 && (!wire->link_t || !wire->link_events || !wire->link_bit))))
      invalid("push_frames_wire: null destination");
    validate_batch(pixels, F, fw, fh, ts, wire != nullptr);
    // a wire call may hold more frames than one launch: its chunks are
    // launches of <= max_batch_for pairs
    if (wire) chunk = std::min(chunk > 0 ? chunk : 64, max_batch_for(desc().n_links, (int64_t)fw * fh));
    if (chunk <= 0) chunk = std::max(1, std::min(F, 64));  // c2 e2e: 32 -> 27.7k, 48 -> 28.3k, 64 -> 29.1k frames/s
    // chunk sizes: a quarter-size first chunk (its upload is not overlapped)
    // and a quarter-size last one (its download is not), full ones between
    std::vector<int> cfirst, csize;
    {
      const int c4 = std::max(1, chunk / 4);
      int rem = F, at = 0;
      auto add = [&](int n) {
        cfirst.push_back(at);
        csize.push_back(n);
        at += n;
        rem -= n;
      };
      if (rem > chunk) add(c4);
      while (rem > chunk + c4) add(chunk);
      if (rem > c4 && rem > 1) {
        add(rem - c4);
        add(c4);
      } else {
        add(rem);
      }
    }
    prepare(F, fw, fh, *std::max_element(csize.begin(), csize.end()), wire ? 0 : -1);
    if (!s_in) {
      CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    }
    const size_t seg_need = (3 + 2 * (size_t)ev.max_links) * sizeof(int64_t);
    if (seg_need > h_seg2_cap) {
      for (auto& b : h_seg2) {
        if (b) cudaFreeHost(b);
        b = nullptr;
        CK(cudaHostAlloc((void**)&b, seg_need, cudaHostAllocDefault));
      }
      h_seg2_cap = seg_need;
    }
    const size_t P = (size_t)w * h;
    const int n_chunks = (int)csize.size();
    std::vector<cudaEvent_t> up(n_chunks), done(n_chunks);
    for (int j = 0; j < n_chunks; ++j) {
      CK(cudaEventCreateWithFlags(&up[j], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&done[j], cudaEventDisableTiming));
    }
    // the copy-in stream must not overwrite slots still read by earlier work
    cudaEvent_t start;
    CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CK(cudaEventRecord(start, stream));
    CK(cudaStreamWaitEvent(s_in, start, 0));
    CK(cudaStreamWaitEvent(s_out, start, 0));
    // dense: chunk j+1's pyramid + flow on s_flow overlap chunk j's chain
    xchunk = dense_flow() && !profiling;
    if (xchunk) {
      if (!s_flow) CK(cudaStreamCreateWithFlags(&s_flow, cudaStreamNonBlocking));
      CK(cudaStreamWaitEvent(s_flow, start, 0));
    }
    pair_base = 0;
    // ring slots of every chunk, as the pushes will assign them
    std::vector<int> slot(n_chunks);
    {
      int sl = next_slot();
      for (int j = 0; j < n_chunks; ++j) {
        slot[j] = sl;
        sl = (sl + csize[j]) % R;
      }
    }
    auto enqueue_upload = [&](int j) {
      const int a = cfirst[j], nf = csize[j];
      upload(pixels + (size_t)a * P, nf, slot[j], false, s_in);
      CK(cudaEventRecord(up[j], s_in));
    };
    seg_t.clear();
    seg_off.clear();
    n_events = 0;
    host_short = false;
    int64_t copied = 0;
    // wire format: the call's planes / polarity / link tables on the device
    const int L = desc().n_links;
    const int64_t call_links = (int64_t)L * (has_prev ? F : F - 1);
    std::vector<int64_t> chunk_link0(n_chunks + 1, 0);
    struct WireReset {  // the wire path ends with the call, also on errors
      bool& f;
      ~WireReset() { f = false; }
    } wire_reset{wire_on};
    if (wire) {
      const int max_chunk = *std::max_element(csize.begin(), csize.end());
      ev.wplanes.ensure((size_t)std::max<int64_t>(call_links, 1) * ev.n_words * 4, stream);
      ev.wpol.ensure(((size_t)std::max<int64_t>(call_links, 1) * P + 31) / 32 * 4 + 8 * ((size_t)n_chunks + 2), stream);
      ev.wlinks.ensure(16 * (size_t)std::max<int64_t>(call_links, 1), stream);
      ev.wbit.ensure(sizeof(int64_t), stream);
      CK(cudaMemsetAsync(ev.wpol.p, 0, ev.wpol.n, stream));
      CK(cudaMemsetAsync(ev.wbit.p, 0, sizeof(int64_t), stream));
      const size_t need = 2 * (size_t)L * max_chunk * sizeof(int64_t);
      if (need > h_wl_cap) {
        for (auto& b : h_wl) {
          if (b) cudaFreeHost(b);
          b = nullptr;
          CK(cudaHostAlloc((void**)&b, need, cudaHostAllocDefault));
        }
        h_wl_cap = need;
      }
      wire_on = true;
      wire_link0 = 0;
      wire_t.clear();
      wire->n_links = call_links;
      wire->words_per_row = ev.wpr;
      wire->row0 = band_y1 > 0 ? band_y0 : 0;
      wire->rows = (int32_t)(ev.n_words / ev.wpr);
      wire->width = w;
      wire->words_per_link = ev.n_words;
      wire->n_events = 0;
      wire->polarity_words = 0;
      if (call_links > wire->link_capacity) host_short = true;
    }
    int64_t wire_words = 0;  // polarity words downloaded so far (the call's end)
    auto drain = [&](int j) {  // chunk j's segment table and events to the host
      CK(cudaEventSynchronize(done[j]));
      const int64_t* hs = h_seg2[j & 1];
      const int S = (int)hs[0];
      const int64_t lo = copied, hi = hs[1 + 2 * S];
      for (int q = 0; q < S; ++q) {
        const int64_t a = hs[1 + S + q], b = hs[2 + S + q];
        if (b > a) {
          seg_t.push_back(hs[1 + q]);
          seg_off.push_back(a);
        }
      }
      if (wire) {
        // chunk j's links: planes, then the polarity words its bits span
        const int64_t g0 = chunk_link0[j], G = chunk_link0[j + 1] - g0;
        if (G > 0 && !host_short) {
          const int64_t* bits = h_wl[j & 1];
          const int64_t* cnts = bits + G;
          const int64_t wlo = bits[0] >> 5;  // chunk starts are u32-aligned
          const int64_t whi = (bits[G - 1] + cnts[G - 1] + 31) >> 5;
          const int64_t pw = (g0 + G) * ev.n_words;
          if (pw > wire->planes_capacity || whi > wire->polarity_capacity) {
            host_short = true;
          } else {
            for (int64_t g = 0; g < G; ++g) {
              wire->link_bit[g0 + g] = bits[g];
              wire->link_events[g0 + g] = cnts[g];
            }
            CK(cudaStreamWaitEvent(s_out, done[j], 0));
            CK(cudaMemcpyAsync(wire->planes + g0 * ev.n_words, ev.wplanes.as<uint32_t>() + g0 * ev.n_words,
                               (size_t)G * ev.n_words * 4, cudaMemcpyDeviceToHost, s_out));
            if (whi > wlo)
              CK(cudaMemcpyAsync(wire->polarity + wlo, ev.wpol.as<uint32_t>() + wlo, (size_t)(whi - wlo) * 4,
                                 cudaMemcpyDeviceToHost, s_out));
            wire_words = std::max(wire_words, whi);
          }
        }
        copied = hi;
        return;
      }
      if (hi > lo) {
        if (hi <= capacity && !host_short) {
          CK(cudaStreamWaitEvent(s_out, done[j], 0));
          CK(cudaMemcpyAsync(host_dst + lo, ev.events.as<uint32_t>() + lo, (size_t)(hi - lo) * 4,
                             cudaMemcpyDeviceToHost, s_out));
        } else {
          host_short = true;
        }
      }
      copied = hi;
    };
    CK(cudaMemsetAsync(ev.base.p, 0, sizeof(int64_t), stream));
    enqueue_upload(0);
    for (int j = 0; j < n_chunks; ++j) {
      if (j + 1 < n_chunks) enqueue_upload(j + 1);
      const int a = cfirst[j], nf = csize[j];
      const bool had_prev = has_prev;
      if (!had_prev && nf == 1) {  // a warm-up chunk of one frame: no pairs, no segment table
        h_seg2[j & 1][0] = 0;
        h_seg2[j & 1][1] = 0;
      }
      wire_host_links = h_wl[j & 1];
      enqueue(nullptr, nf, ts + a, false, up[j], h_seg2[j & 1], true);
      pair_base += had_prev ? nf : nf - 1;
      chunk_link0[j + 1] = chunk_link0[j] + (int64_t)L * (had_prev ? nf : nf - 1);
      CK(cudaEventRecord(done[j], stream));
      pending = false;
      if (j > 0) drain(j - 1);
    }
    drain(n_chunks - 1);
    xchunk = false;
    pair_base = 0;
    if (wire) {
      wire_on = false;
      if (!host_short)
        for (int64_t g = 0; g < call_links; ++g) wire->link_t[g] = wire_t[(size_t)g];
      wire->n_events = copied;
      wire->polarity_words = wire_words;
    }
    seg_off.push_back(copied);
    n_events = copied;
    CK(cudaStreamSynchronize(s_out));
    CK(cudaStreamSynchronize(stream));
    // the call's merged segment table on the device (for a later unpack)
    {
      std::vector<int64_t> t(3 + 2 * seg_t.size());
      const int S = (int)seg_t.size();
      t[0] = S;
      for (int q = 0; q < S; ++q) t[1 + q] = seg_t[q], t[1 + S + q] = seg_off[q];
      t[1 + 2 * S] = copied;
      // (the call may hold more segments than one launch's table)
      if ((3 + 2 * (size_t)S) * sizeof(int64_t) > ev.seg_out.n) ev.seg_out.ensure((3 + 2 * (size_t)S) * sizeof(int64_t), stream);
      CK(cudaMemcpy(ev.seg_out.p, t.data(), (2 + 2 * (size_t)S) * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
    for (int j = 0; j < n_chunks; ++j) {
      cudaEventDestroy(up[j]);
      cudaEventDestroy(done[j]);
    }
    cudaEventDestroy(start);
    if (host_short && wire) invalid("push_frames_wire: destination too small");
    if (host_short) invalid("push_frames_streamed: destination too small (events stay on the device; see copy_events)");
  }

  // simulate_sparse up to the intermediates (simulate.cpp:145-199), all pairs
  void sparse_stage(int r0, int n_pairs, ChainParams& c) {
    const int N = n_interp_eff();
    const size_t P = (size_t)w * h;
    SelectParams sp{};
    sp.w = w;
    sp.h = h;
    sp.wpr = ev.wpr;
    sp.n_words = ev.n_words;
    sp.words_per_block = ev.wpb;
    sp.n_blocks = ev.n_blocks;
    sp.R = R;
    sp.r0 = r0;
    sp.frames = Ring<const uint8_t>{frames.as<uint8_t>(), P};
    sp.log_mode = log_mode();
    sp.sel = cfg.selection_threshold > 0 ? cfg.selection_threshold : cfg.c_pos;  // types.hpp:122-124
    sp.sel_log = cfg.sel_log > 0.0f ? cfg.sel_log : cfg.c_pos_log;
    sp.lut = lut.as<float>();
    sp.diff_mode = diff_interp();
    sp.c_pos = cfg.c_pos;
    sp.c_neg = cfg.c_neg;
    sp.skip_first = c.skip_first;
    sp.masks = sel_masks.as<uint32_t>();
    sp.counts = sel_counts.as<uint32_t>();
    sp.prefix = sel_prefix.as<int64_t>();
    sp.total = sel_total.as<int64_t>();
    sp.points = points.as<uint32_t>();
    sp.n_points = n_points.as<int>();
    sp.P = P;
    launch_select(sp, n_pairs, stream);
    CK_LAUNCH("select");
    // estimate_sparse_flow (flow.cpp:278-381)
    SparseLKParams lk = flow.sparse_params(r0, quads.as<uint32_t>());
    lk.points = points.as<uint32_t>();
    lk.n_points = n_points.as<int>();
    lk.disp = disp.as<float2>();
    lk.status = status.as<uint8_t>();
    launch_sparse_lk(lk, (int)std::min<size_t>(P, INT32_MAX), n_pairs, stream);
    CK_LAUNCH("sparse_lk");
    splat_stage(r0, n_pairs, c);
    launches += 6;  // select mask + offsets + emit, sparse LK, splat, resolve
    (void)N;
  }

  void splat_stage(int r0, int n_pairs, ChainParams& c) {
    const int N = n_interp_eff();
    const size_t P = (size_t)w * h;
    SplatParams spl{};
    spl.w = w;
    spl.h = h;
    spl.n_interp = N;
    spl.R = R;
    spl.r0 = r0;
    spl.frames = Ring<const uint8_t>{frames.as<uint8_t>(), P};
    spl.points = points.as<uint32_t>();
    spl.n_points = n_points.as<int>();
    spl.disp = disp.as<float2>();
    spl.status = status.as<uint8_t>();
    spl.claims = claims.as<uint32_t>();
    spl.touched = touched.as<uint32_t>();
    spl.P = P;
    spl.svals = svals.as<uint8_t>();
    spl.diff_mode = diff_interp();
    spl.dvals = dvals.as<int16_t>();
    launch_splat(spl, (int)std::min<int64_t>((int64_t)P * N, INT32_MAX), n_pairs, stream);
    CK_LAUNCH("splat");
    c.svals = svals.as<uint8_t>();
    c.dvals = dvals.as<int16_t>();
    c.claims = claims.as<uint32_t>();
    c.touched = touched.as<uint32_t>();
    c.points = points.as<uint32_t>();
    c.n_points = n_points.as<int>();
    // chain_pipeline(prev, curr, {}) when nothing was selected
    // (simulate.cpp:161-163) equals the full chain over copies of prev,
    // except in log mode without endpoints, where it emits nothing
    //
    c.skip_empty = log_mode() && !cfg.include_endpoints;
  }

  // Complete the queued push: wait, read the segment table, re-emit when the
  // (magnitude-mode) event buffer was too small.
  void finish() {
    if (!pending) return;
    pending = false;
    CK(cudaStreamSynchronize(stream));
    int S = (int)h_seg_out[0];
    int64_t total = h_seg_out[1 + 2 * S];
    if (total > ev.capacity) {
      ev.grow(total + total / 4, stream);
      last_emit.capacity = ev.capacity;
      last_emit.out = ev.events.as<uint32_t>();
      CK(cudaMemsetAsync(ev.base.p, 0, sizeof(int64_t), stream));
      launch_emit(last_emit, ev.segbase.as<int64_t>(), stream);
      CK_LAUNCH("emit");
      launches += 2;
      CK(cudaStreamSynchronize(stream));
    }
    // report only the segments that hold events
    seg_t.clear();
    seg_off.clear();
    for (int s = 0; s < S; ++s) {
      const int64_t a = h_seg_out[1 + S + s], b = h_seg_out[2 + S + s];
      if (b > a) {
        seg_t.push_back(h_seg_out[1 + s]);
        seg_off.push_back(a);
      }
    }
    seg_off.push_back(total);
    n_events = total;
  }

  void fill_out(evsim_gpu_events* out) const {
    if (!out) return;
    out->width = w;
    out->height = h;
    out->n_events = n_events;
    out->n_segments = (int32_t)seg_t.size();
    out->seg_t = seg_t.data();
    out->seg_offset = seg_off.data();
    out->d_packed = ev.events.as<uint32_t>();
  }
};

// ====================================================================== wire unpack
// Expands evsim_gpu_wire (include/evsim_gpu.h) into the reference's event
// stream.  Runs of links with equal timestamps form one segment, ordered
// (y, x, p) with duplicates (finalize's stable sort, src/simulate.cpp:36-40):
// per pixel the segment's negative events, then its positive ones.  Segments
// are independent, so threads take segments (long single-link segments are
// split into word ranges, their event offsets from per-range popcounts).
namespace {

struct WireOut {
  int format;
  void* out;
  void put(int64_t i, uint32_t x, uint32_t y, bool neg, int64_t t) const {
    if (format == 0) {
      static_cast<uint32_t*>(out)[i] = x | (y << 16) | (neg ? 0x80000000u : 0u);
    } else {
      evsim_event& e = static_cast<evsim_event*>(out)[i];
      e.x = (uint16_t)x;
      e.y = (uint16_t)y;
      e.t = t;
      e.p = neg ? -1 : 1;
    }
  }
};

inline bool pol_bit(const uint32_t* pol, int64_t b) { return (pol[b >> 5] >> (b & 31)) & 1u; }

}  // namespace

void wire_unpack(const evsim_gpu_wire& wr, int format, void* out, int threads) {
  const int64_t G = wr.n_links, W = wr.words_per_link;
  const int wpr = wr.words_per_row;
  const WireOut o{format, out};
  // segments: runs of equal link_t
  std::vector<int64_t> seg_first, ev_base;
  int64_t tot = 0;
  for (int64_t g = 0; g < G; ++g) {
    if (g == 0 || wr.link_t[g] != wr.link_t[g - 1]) {
      seg_first.push_back(g);
      ev_base.push_back(tot);
    }
    tot += wr.link_events[g];
  }
  seg_first.push_back(G);
  ev_base.push_back(tot);
  // work items: (segment, word range); single-link segments in ranges of
  // ~64k words with their own event offsets
  struct Item {
    int64_t seg, w0, w1, base, bit;
  };
  std::vector<Item> items;
  const int64_t span = 1 << 16;
  for (size_t sgi = 0; sgi + 1 < seg_first.size(); ++sgi) {
    const int64_t g0 = seg_first[sgi], g1 = seg_first[sgi + 1];
    if (g1 - g0 > 1 || W <= span) {
      items.push_back({(int64_t)sgi, 0, W, ev_base[sgi], wr.link_bit[g0]});
      continue;
    }
    const uint32_t* pl = wr.planes + g0 * W;
    int64_t base = ev_base[sgi], bit = wr.link_bit[g0];
    for (int64_t w0 = 0; w0 < W; w0 += span) {
      const int64_t w1 = std::min(W, w0 + span);
      items.push_back({(int64_t)sgi, w0, w1, base, bit});
      int64_t c = 0;
      for (int64_t w = w0; w < w1; ++w) c += __builtin_popcount(pl[w]);
      base += c;
      bit += c;
    }
  }
  auto run = [&](const Item& it) {
    const int64_t g0 = seg_first[(size_t)it.seg], g1 = seg_first[(size_t)it.seg + 1];
    const int64_t t = wr.link_t[g0];
    int64_t i = it.base;
    if (g1 - g0 == 1) {
      const uint32_t* pl = wr.planes + g0 * W;
      int64_t b = it.bit;
      for (int64_t w = it.w0; w < it.w1; ++w) {
        uint32_t m = pl[w];
        if (!m) continue;
        const uint32_t y = (uint32_t)(wr.row0 + w / wpr), x0 = (uint32_t)(32 * (w % wpr));
        while (m) {
          const int bitpos = __builtin_ctz(m);
          m &= m - 1;
          o.put(i++, x0 + (uint32_t)bitpos, y, pol_bit(wr.polarity, b++), t);
        }
      }
      return;
    }
    // several links share the timestamp: per pixel, negatives then positives
    std::vector<int64_t> cur(g1 - g0);
    for (int64_t g = g0; g < g1; ++g) cur[g - g0] = wr.link_bit[g];
    for (int64_t w = 0; w < W; ++w) {
      uint32_t any = 0;
      for (int64_t g = g0; g < g1; ++g) any |= wr.planes[g * W + w];
      if (!any) continue;
      int nneg[32] = {}, npos[32] = {};
      for (int64_t g = g0; g < g1; ++g) {
        uint32_t m = wr.planes[g * W + w];
        while (m) {
          const int bitpos = __builtin_ctz(m);
          m &= m - 1;
          if (pol_bit(wr.polarity, cur[g - g0]++)) ++nneg[bitpos];
          else ++npos[bitpos];
        }
      }
      const uint32_t y = (uint32_t)(wr.row0 + w / wpr), x0 = (uint32_t)(32 * (w % wpr));
      for (int b = 0; b < 32; ++b) {
        for (int q = 0; q < nneg[b]; ++q) o.put(i++, x0 + (uint32_t)b, y, true, t);
        for (int q = 0; q < npos[b]; ++q) o.put(i++, x0 + (uint32_t)b, y, false, t);
      }
    }
  };
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::min<int64_t>(T, (int64_t)items.size());
  if (T <= 1) {
    for (const auto& it : items) run(it);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (int k = 0; k < T; ++k)
    th.emplace_back([&] {
      for (size_t j; (j = next.fetch_add(1)) < items.size();) run(items[j]);
    });
  for (auto& x : th) x.join();
}

// ====================================================================== C-ABI

namespace {

void make_sim(evsim_gpu_sim* s, const evsim_gpu_config& cfg, int device) {
  s->cfg = cfg;
  s->preset = resolve_preset(cfg);
  s->device = device;
  // the handle's stream carries the chain (the sequential critical path of a
  // push): highest priority, so its blocks dispatch ahead of the pipelined
  // flow of the next sub-batch (s_flow, default priority), which fills in
  int lo_prio = 0, hi_prio = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  CK(cudaStreamCreateWithPriority(&s->stream, cudaStreamNonBlocking, hi_prio));
  float h_lut[256];
  log_lut(h_lut);
  s->lut.ensure(sizeof h_lut, s->stream);
  CK(cudaMemcpyAsync(s->lut.p, h_lut, sizeof h_lut, cudaMemcpyHostToDevice, s->stream));
  int32_t h_th[1024];
  log_thresholds(h_lut, s->cfg.c_pos_log, s->cfg.c_neg_log, h_th);
  s->lthr.ensure(sizeof h_th, s->stream);
  CK(cudaMemcpyAsync(s->lthr.p, h_th, sizeof h_th, cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
}

}  // namespace

extern "C" {

const char* evsim_gpu_last_error(void) { return g_err.c_str(); }

void evsim_gpu_config_defaults(int32_t method, evsim_gpu_config* out) {
  // SimulatorConfig::defaults  include/evsim/types.hpp:101-120
  evsim_gpu_config c{};
  c.method = method;
  c.c_pos = 2;
  c.c_neg = -2;
  c.n_interp = 0;
  c.flow_preset = EVSIM_FLOW_LOW_QUALITY;
  c.selection_threshold = 0;
  c.events_per_crossing = EVSIM_EVENTS_SINGLE;
  c.include_endpoints = 1;
  c.contrast_mode = EVSIM_CONTRAST_LINEAR;
  c.c_pos_log = 0.2f;
  c.c_neg_log = -0.2f;
  switch (method) {
    case EVSIM_METHOD_DENSE: c.n_interp = 10; break;
    case EVSIM_METHOD_SPARSE:
      c.c_pos = 10, c.c_neg = -10, c.n_interp = 10, c.selection_threshold = 10;
      break;
    case EVSIM_METHOD_DIFFERENCE_INTERP: c.c_pos = 20, c.c_neg = -20, c.n_interp = 10; break;
    default: break;
  }
  *out = c;
}

int evsim_gpu_config_validate(const evsim_gpu_config* cfg) {
  return guarded([&] {
    if (!cfg) invalid("config must not be null");
    validate_config(*cfg);
  });
}

int evsim_gpu_create(const evsim_gpu_config* cfg, int device, evsim_gpu_sim** out) {
  return guarded([&] {
    if (!cfg || !out) invalid("evsim_gpu_create: null argument");
    validate_config(*cfg);
    validate_preset(resolve_preset(*cfg));
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) invalid("evsim_gpu_create: no such CUDA device");
    CK(cudaSetDevice(device));
    init_pool(device);
    auto s = std::make_unique<evsim_gpu_sim>();
    make_sim(s.get(), *cfg, device);
    *out = s.release();
  });
}

int evsim_gpu_push_frame(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width, int32_t height, int64_t t_us,
                         int32_t pixels_on_device, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frame: null simulator");
    sim->push(pixels, 1, width, height, &t_us, pixels_on_device != 0);
    sim->finish();
    sim->fill_out(out);
  });
}

int evsim_gpu_push_frames(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames, int32_t width,
                          int32_t height, const int64_t* t_us, int32_t pixels_on_device, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frames: null simulator");
    sim->push(pixels, n_frames, width, height, t_us, pixels_on_device != 0);
    sim->finish();
    sim->fill_out(out);
  });
}

int evsim_gpu_push_frame_async(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width, int32_t height,
                               int64_t t_us, int32_t pixels_on_device) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frame_async: null simulator");
    sim->push(pixels, 1, width, height, &t_us, pixels_on_device != 0);
  });
}

int evsim_gpu_push_frames_async(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames, int32_t width,
                                int32_t height, const int64_t* t_us, int32_t pixels_on_device) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frames_async: null simulator");
    sim->push(pixels, n_frames, width, height, t_us, pixels_on_device != 0);
  });
}

int evsim_gpu_push_frames_batched(evsim_gpu_sim* const* sims, int32_t n_sims, const uint8_t* const* pixels,
                                  int32_t n_frames, int32_t width, int32_t height, const int64_t* const* t_us,
                                  int32_t pixels_on_device, evsim_gpu_events* outs) {
  return guarded([&] {
    if (n_sims < 0 || (n_sims > 0 && (!sims || !pixels || !t_us))) invalid("push_frames_batched: null argument");
    for (int i = 0; i < n_sims; ++i) {
      if (!sims[i]) invalid("push_frames_batched: null simulator");
      for (int j = 0; j < i; ++j)
        if (sims[j] == sims[i]) invalid("push_frames_batched: a simulator appears twice");
    }
    // every batch is validated before any is enqueued (all-or-nothing)
    for (int i = 0; i < n_sims; ++i) sims[i]->validate_batch(pixels[i], n_frames, width, height, t_us[i]);
    for (int i = 0; i < n_sims; ++i) {
      sims[i]->prepare(n_frames, width, height);
      sims[i]->enqueue(pixels[i], n_frames, t_us[i], pixels_on_device != 0, nullptr, sims[i]->h_seg_out, false);
    }
    for (int i = 0; i < n_sims; ++i) {
      CK(cudaSetDevice(sims[i]->device));
      sims[i]->finish();
      if (outs) sims[i]->fill_out(outs + i);
    }
  });
}

int evsim_gpu_push_frames_streamed(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames, int32_t width,
                                   int32_t height, const int64_t* t_us, int32_t chunk, uint32_t* host_events,
                                   int64_t capacity, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frames_streamed: null simulator");
    try {
      sim->push_streamed(pixels, n_frames, width, height, t_us, chunk, host_events, capacity);
    } catch (...) {
      sim->fill_out(out);
      throw;
    }
    sim->fill_out(out);
  });
}

int evsim_gpu_push_frames_wire(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames, int32_t width,
                               int32_t height, const int64_t* t_us, int32_t chunk, evsim_gpu_wire* wire,
                               evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frames_wire: null simulator");
    if (!wire) invalid("evsim_gpu_push_frames_wire: null wire descriptor");
    try {
      sim->push_streamed(pixels, n_frames, width, height, t_us, chunk, nullptr, 0, wire);
    } catch (...) {
      sim->fill_out(out);
      throw;
    }
    sim->fill_out(out);
  });
}

int evsim_gpu_wire_unpack(const evsim_gpu_wire* wire, int32_t format, void* out, int64_t capacity, int32_t threads) {
  return guarded([&] {
    if (!wire || (!out && capacity > 0)) invalid("evsim_gpu_wire_unpack: null argument");
    if (format != 0 && format != 1) invalid("evsim_gpu_wire_unpack: format must be 0 (packed) or 1 (evsim_event)");
    if (capacity < wire->n_events) invalid("evsim_gpu_wire_unpack: destination too small");
    wire_unpack(*wire, format, out, threads);
  });
}

int evsim_gpu_place_events(evsim_gpu_sim* sim, uint32_t* dst, const int64_t* dst_offset, int32_t n_segments) {
  return guarded([&] {
    if (!sim || (!dst && n_segments > 0) || (!dst_offset && n_segments > 0))
      invalid("evsim_gpu_place_events: null argument");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    const int S = (int)sim->seg_t.size();
    if (n_segments != S) invalid("evsim_gpu_place_events: n_segments must equal the last push's segment count");
    if (S == 0) return;
    {  // a peer GPU's buffer in this process: enable P2P (IPC mappings are opened with it)
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
          at.device != sim->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    }
    std::vector<int64_t> tab(2 * (size_t)S + 1);
    int64_t max_len = 0;
    for (int q = 0; q <= S; ++q) tab[q] = sim->seg_off[q];
    for (int q = 0; q < S; ++q) {
      tab[S + 1 + q] = dst_offset[q];
      max_len = std::max(max_len, sim->seg_off[q + 1] - sim->seg_off[q]);
    }
    sim->place_tab.ensure(tab.size() * sizeof(int64_t), sim->stream);
    CK(cudaMemcpyAsync(sim->place_tab.p, tab.data(), tab.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                       sim->stream));
    const int64_t* d = sim->place_tab.as<int64_t>();
    launch_place(sim->ev.events.as<uint32_t>(), d, d + S + 1, S, max_len, dst, sim->stream);
    CK_LAUNCH("place");
    ++sim->launches;
    CK(cudaStreamSynchronize(sim->stream));  // tab is a stack buffer of this call
  });
}

int evsim_gpu_ipc_handle(const void* dptr, void* handle64) {
  return guarded([&] {
    if (!dptr || !handle64) invalid("evsim_gpu_ipc_handle: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int evsim_gpu_ipc_open(int32_t device, const void* handle64, void** dptr) {
  return guarded([&] {
    if (!handle64 || !dptr) invalid("evsim_gpu_ipc_open: null argument");
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int evsim_gpu_ipc_close(int32_t device, void* dptr) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    if (dptr) CK(cudaIpcCloseMemHandle(dptr));
  });
}

int evsim_gpu_set_row_band(evsim_gpu_sim* sim, int32_t y0, int32_t y1) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_set_row_band: null simulator");
    if (sim->has_prev) invalid("set_row_band: only at the start of a stream (before the first push or after reset)");
    if (sim->cfg.method == EVSIM_METHOD_SPARSE || sim->cfg.method == EVSIM_METHOD_DIFFERENCE_INTERP)
      invalid("set_row_band: only the dense and difference_only methods (sparse splats cross band borders)");
    if (!(y0 == 0 && y1 == 0) && (y0 < 0 || y1 <= y0)) invalid("set_row_band: need 0 <= y0 < y1");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    sim->band_y0 = y0;
    sim->band_y1 = y1;
    sim->w = sim->h = 0;  // geometry is rebuilt at the next push
  });
}

int evsim_gpu_max_batch(const evsim_gpu_sim* sim, int32_t width, int32_t height) {
  if (!sim) return 0;
  return max_batch_for(sim->desc().n_links, (int64_t)width * height);
}

int evsim_gpu_sync(evsim_gpu_sim* sim, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_sync: null simulator");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    CK(cudaStreamSynchronize(sim->stream));
    sim->fill_out(out);
  });
}

int evsim_gpu_copy_events(evsim_gpu_sim* sim, void* host_dst, int64_t capacity, int32_t format) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_copy_events: null simulator");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    const int64_t n = sim->n_events;
    if (capacity < n) invalid("evsim_gpu_copy_events: destination too small");
    if (n == 0) return;
    if (format == 0) {
      CK(cudaMemcpyAsync(host_dst, sim->ev.events.p, (size_t)n * 4, cudaMemcpyDeviceToHost, sim->stream));
    } else if (format == 1) {
      DevBuf tmp;
      tmp.ensure((size_t)n * 24, sim->stream);
      launch_unpack_events(sim->ev.events.as<uint32_t>(), sim->ev.seg_out.as<int64_t>(), n, tmp.p, sim->stream);
      CK_LAUNCH("unpack");
      CK(cudaMemcpyAsync(host_dst, tmp.p, (size_t)n * 24, cudaMemcpyDeviceToHost, sim->stream));
      CK(cudaStreamSynchronize(sim->stream));
    } else if (format == 2) {
      DevBuf tmp;
      tmp.ensure((size_t)n * 13, sim->stream);
      launch_evs_records(sim->ev.events.as<uint32_t>(), sim->ev.seg_out.as<int64_t>(), n, tmp.as<uint8_t>(),
                         sim->stream);
      CK_LAUNCH("evs");
      CK(cudaMemcpyAsync(host_dst, tmp.p, (size_t)n * 13, cudaMemcpyDeviceToHost, sim->stream));
      CK(cudaStreamSynchronize(sim->stream));
    } else {
      invalid("evsim_gpu_copy_events: unknown format");
    }
    CK(cudaStreamSynchronize(sim->stream));
  });
}

// ---- data formats either side of the path ------------------

namespace {
struct TmpStream {
  cudaStream_t s = nullptr;
  TmpStream() { CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~TmpStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};
[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
  throw ApiError{EVSIM_GPU_RUNTIME, "'" + path + "': " + what};
}
}  // namespace

int evsim_gpu_ingest_frames(const uint8_t* src, int32_t channels, int32_t w, int32_t h, int32_t n_frames,
                            int32_t tw, int32_t th, uint8_t* dst) {
  return guarded([&] {
    if (!src || !dst || w <= 0 || h <= 0 || n_frames < 0) invalid("ingest_frames: malformed input");
    if (channels != 1 && channels != 3) invalid("ingest_frames: channels must be 1 or 3");
    const bool resize = !(tw == 0 && th == 0) && (tw != w || th != h);
    if (resize && (tw <= 0 || th <= 0)) invalid("resize_bilinear: target must be positive");  // io.cpp:46-48
    if (n_frames == 0) return;
    CK(cudaSetDevice(0));
    init_pool(0);
    TmpStream ts;
    const size_t P = (size_t)w * h, Q = resize ? (size_t)tw * th : P;
    DevBuf in, gray, out;
    in.ensure((size_t)n_frames * P * channels, ts.s);
    CK(cudaMemcpyAsync(in.p, src, (size_t)n_frames * P * channels, cudaMemcpyHostToDevice, ts.s));
    const uint8_t* g = in.as<uint8_t>();
    if (channels == 3) {  // load_frames: luma of every pixel (io.cpp:86-90)
      gray.ensure((size_t)n_frames * P, ts.s);
      launch_luma(in.as<uint8_t>(), gray.as<uint8_t>(), (int64_t)(n_frames * P), ts.s);
      CK_LAUNCH("luma");
      g = gray.as<uint8_t>();
    }
    if (resize) {  // then resize_bilinear to the target (io.cpp:92-95)
      out.ensure((size_t)n_frames * Q, ts.s);
      launch_resize(g, w, h, out.as<uint8_t>(), tw, th, n_frames, ts.s);
      CK_LAUNCH("resize");
      g = out.as<uint8_t>();
    }
    CK(cudaMemcpyAsync(dst, g, (size_t)n_frames * Q, cudaMemcpyDeviceToHost, ts.s));
    CK(cudaStreamSynchronize(ts.s));
  });
}

int evsim_gpu_write_events_binary(evsim_gpu_sim* sim, const char* path) {
  return guarded([&] {
    if (!sim || !path) invalid("write_events_binary: null argument");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    const int64_t n = sim->n_events;
    std::vector<uint8_t> buf(16 + (size_t)n * 13);
    std::memcpy(buf.data(), "EVS1", 4);  // io.cpp:152-156
    const uint16_t w16 = (uint16_t)sim->w, h16 = (uint16_t)sim->h;
    const uint64_t cnt = (uint64_t)n;
    for (int b = 0; b < 2; ++b) buf[4 + b] = (uint8_t)(w16 >> (8 * b)), buf[6 + b] = (uint8_t)(h16 >> (8 * b));
    for (int b = 0; b < 8; ++b) buf[8 + b] = (uint8_t)(cnt >> (8 * b));
    if (n) {
      DevBuf tmp;
      tmp.ensure((size_t)n * 13, sim->stream);
      launch_evs_records(sim->ev.events.as<uint32_t>(), sim->ev.seg_out.as<int64_t>(), n, tmp.as<uint8_t>(),
                         sim->stream);
      CK_LAUNCH("evs");
      CK(cudaMemcpyAsync(buf.data() + 16, tmp.p, (size_t)n * 13, cudaMemcpyDeviceToHost, sim->stream));
      CK(cudaStreamSynchronize(sim->stream));
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) io_fail(path, "cannot open for writing");
    const size_t wrote = std::fwrite(buf.data(), 1, buf.size(), f);
    const bool ok = std::fclose(f) == 0 && wrote == buf.size();
    if (!ok) io_fail(path, "write failed");
  });
}

int evsim_gpu_write_events_text(evsim_gpu_sim* sim, const char* path) {
  return guarded([&] {
    if (!sim || !path) invalid("write_events_text: null argument");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    const int64_t n = sim->n_events;
    std::vector<evsim_event> ev((size_t)n);
    if (n) {
      DevBuf tmp;
      tmp.ensure((size_t)n * 24, sim->stream);
      launch_unpack_events(sim->ev.events.as<uint32_t>(), sim->ev.seg_out.as<int64_t>(), n, tmp.p, sim->stream);
      CK_LAUNCH("unpack");
      CK(cudaMemcpyAsync(ev.data(), tmp.p, (size_t)n * 24, cudaMemcpyDeviceToHost, sim->stream));
      CK(cudaStreamSynchronize(sim->stream));
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) io_fail(path, "cannot open for writing");
    std::string line;  // io.cpp:105-126: "x,y,t,p\n", p as 1 / -1
    bool ok = true;
    for (const auto& e : ev) {
      line = std::to_string(e.x) + ',' + std::to_string(e.y) + ',' + std::to_string(e.t) + ',' +
             (e.p > 0 ? "1" : "-1") + '\n';
      ok = ok && std::fwrite(line.data(), 1, line.size(), f) == line.size();
    }
    ok = std::fclose(f) == 0 && ok;
    if (!ok) io_fail(path, "write failed");
  });
}

int evsim_gpu_events_per_pixel_second(const evsim_event* ev, int64_t n, int32_t w, int32_t h, double duration,
                                      double* mean, double* stddev, uint64_t* total) {
  return guarded([&] {
    // metrics.cpp:7-39
    if (!(duration > 0.0)) invalid("events_per_pixel_second: duration must be > 0");
    if (w <= 0 || h <= 0) invalid("events_per_pixel_second: stream resolution unknown");
    if (n < 0 || (n > 0 && !ev)) invalid("events_per_pixel_second: malformed events");
    CK(cudaSetDevice(0));
    init_pool(0);
    TmpStream ts;
    const size_t P = (size_t)w * h;
    std::vector<uint32_t> counts(P, 0);
    if (n > 0) {
      DevBuf dev, dc;
      dev.ensure((size_t)n * sizeof(evsim_event), ts.s);
      dc.ensure(P * 4, ts.s, true);
      CK(cudaMemcpyAsync(dev.p, ev, (size_t)n * sizeof(evsim_event), cudaMemcpyHostToDevice, ts.s));
      launch_event_counts(dev.as<evsim_event>(), n, w, dc.as<uint32_t>(), ts.s);
      CK_LAUNCH("counts");
      CK(cudaMemcpyAsync(counts.data(), dc.p, P * 4, cudaMemcpyDeviceToHost, ts.s));
      CK(cudaStreamSynchronize(ts.s));
    }
    // the reduction keeps the reference's sequential fp64 order (it is not exact)
    double sum = 0.0, sum_sq = 0.0;
    for (size_t i = 0; i < P; ++i) {
      const double rate = static_cast<double>(counts[i]) / duration;
      sum += rate;
      sum_sq += rate * rate;
    }
    const double np = static_cast<double>(P);
    const double m = sum / np;
    const double var = std::max(0.0, sum_sq / np - m * m);
    if (mean) *mean = m;
    if (stddev) *stddev = std::sqrt(var);
    if (total) *total = (uint64_t)n;
  });
}

int evsim_gpu_accumulate(const evsim_event* ev, int64_t n, int32_t w, int32_t h, int64_t t_start, int64_t t_end,
                         uint8_t* classes) {
  return guarded([&] {
    // metrics.cpp:41-69
    if (t_start >= t_end) invalid("accumulate: window must satisfy t_start < t_end");
    if (w <= 0 || h <= 0) invalid("accumulate: stream resolution unknown");
    if (n < 0 || (n > 0 && !ev) || !classes) invalid("accumulate: malformed events");
    CK(cudaSetDevice(0));
    init_pool(0);
    TmpStream ts;
    const size_t P = (size_t)w * h;
    DevBuf dev, bits, out;
    bits.ensure(P * 4, ts.s, true);
    out.ensure(P, ts.s);
    if (n > 0) {
      dev.ensure((size_t)n * sizeof(evsim_event), ts.s);
      CK(cudaMemcpyAsync(dev.p, ev, (size_t)n * sizeof(evsim_event), cudaMemcpyHostToDevice, ts.s));
    }
    launch_accumulate(n > 0 ? dev.as<evsim_event>() : nullptr, n, w, t_start, t_end, bits.as<uint32_t>(),
                      out.as<uint8_t>(), (int64_t)P, ts.s);
    CK_LAUNCH("accumulate");
    CK(cudaMemcpyAsync(classes, out.p, P, cudaMemcpyDeviceToHost, ts.s));
    CK(cudaStreamSynchronize(ts.s));
  });
}

int evsim_gpu_difference_frame(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h, int16_t* values) {
  return guarded([&] {
    // core.cpp:5-19
    if (!prev || !curr || !values || w <= 0 || h <= 0) invalid("difference_frame: malformed frames");
    CK(cudaSetDevice(0));
    init_pool(0);
    TmpStream ts;
    const size_t P = (size_t)w * h;
    DevBuf f, out;
    f.ensure(2 * P, ts.s);
    out.ensure(2 * P, ts.s);
    CK(cudaMemcpyAsync(f.p, prev, P, cudaMemcpyHostToDevice, ts.s));
    CK(cudaMemcpyAsync(f.as<uint8_t>() + P, curr, P, cudaMemcpyHostToDevice, ts.s));
    launch_difference(f.as<uint8_t>(), f.as<uint8_t>() + P, out.as<int16_t>(), (int64_t)P, ts.s);
    CK_LAUNCH("difference");
    CK(cudaMemcpyAsync(values, out.p, 2 * P, cudaMemcpyDeviceToHost, ts.s));
    CK(cudaStreamSynchronize(ts.s));
  });
}

int evsim_gpu_threshold_events(const int16_t* values, int32_t w, int32_t h, const evsim_gpu_config* cfg,
                               int64_t event_time, evsim_event* events, int64_t capacity, int64_t* n_events) {
  return guarded([&] {
    // core.cpp:21-46 (config.validate() first, core.cpp:23)
    if (!cfg || !n_events) invalid("threshold_events: null argument");
    validate_config(*cfg);
    if (w < 0 || h < 0 || ((int64_t)w * h > 0 && !values)) invalid("threshold_events: malformed difference frame");
    const int64_t P = (int64_t)w * h;
    *n_events = 0;
    if (P == 0) return;
    CK(cudaSetDevice(0));
    init_pool(0);
    TmpStream ts;
    const int64_t T = threshold_tiles(P);
    const int mag = cfg->events_per_crossing == EVSIM_EVENTS_MAGNITUDE ? 1 : 0;
    DevBuf dv, tiles;
    dv.ensure((size_t)P * 2, ts.s);
    tiles.ensure((size_t)T * 8, ts.s);
    CK(cudaMemcpyAsync(dv.p, values, (size_t)P * 2, cudaMemcpyHostToDevice, ts.s));
    launch_threshold_count(dv.as<int16_t>(), P, cfg->c_pos, cfg->c_neg, mag, tiles.as<int64_t>(), ts.s);
    CK_LAUNCH("threshold_count");
    std::vector<int64_t> off((size_t)T);
    CK(cudaMemcpyAsync(off.data(), tiles.p, (size_t)T * 8, cudaMemcpyDeviceToHost, ts.s));
    CK(cudaStreamSynchronize(ts.s));
    int64_t total = 0;
    for (auto& o : off) {  // exclusive prefix of the tile totals
      const int64_t c = o;
      o = total;
      total += c;
    }
    *n_events = total;
    if (!events || capacity < total || total == 0) return;
    DevBuf dout;
    dout.ensure((size_t)total * sizeof(evsim_event), ts.s);
    CK(cudaMemcpyAsync(tiles.p, off.data(), (size_t)T * 8, cudaMemcpyHostToDevice, ts.s));
    launch_threshold_emit(dv.as<int16_t>(), P, w, cfg->c_pos, cfg->c_neg, mag, event_time, tiles.as<int64_t>(),
                          dout.as<evsim_event>(), ts.s);
    CK_LAUNCH("threshold_emit");
    CK(cudaMemcpyAsync(events, dout.p, (size_t)total * sizeof(evsim_event), cudaMemcpyDeviceToHost, ts.s));
    CK(cudaStreamSynchronize(ts.s));
  });
}

void evsim_gpu_log_lut(float* lut256) {
  if (lut256) log_lut(lut256);
}

int evsim_gpu_push_frame_with_flow(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width, int32_t height,
                                   int64_t t_us, const float* du, const float* dv, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frame_with_flow: null simulator");
    CK(cudaSetDevice(sim->device));
    if (sim->cfg.method == EVSIM_METHOD_SPARSE && sim->n_interp_eff() > 0)
      invalid("push_frame_with_flow: a sparse simulator takes tracks (evsim_gpu_push_frame_with_tracks)");
    sim->push_custom(pixels, width, height, t_us, du, dv, nullptr, 0, nullptr, nullptr);
    sim->finish();
    sim->fill_out(out);
  });
}

int evsim_gpu_push_frame_with_tracks(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width, int32_t height,
                                     int64_t t_us, const int32_t* points_xy, int64_t n_points, const float* disp,
                                     const uint8_t* status, evsim_gpu_events* out) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_push_frame_with_tracks: null simulator");
    CK(cudaSetDevice(sim->device));
    if (sim->cfg.method == EVSIM_METHOD_DENSE && sim->n_interp_eff() > 0)
      invalid("push_frame_with_tracks: a dense simulator takes a flow field (evsim_gpu_push_frame_with_flow)");
    sim->push_custom(pixels, width, height, t_us, nullptr, nullptr, points_xy, n_points, disp, status);
    sim->finish();
    sim->fill_out(out);
  });
}

void* evsim_gpu_stream(evsim_gpu_sim* sim) { return sim ? (void*)sim->stream : nullptr; }

int evsim_gpu_reset(evsim_gpu_sim* sim) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_reset: null simulator");
    CK(cudaSetDevice(sim->device));
    sim->finish();
    // Simulator::reset  include/evsim/simulate.hpp:83-86
    sim->has_prev = false;
    sim->custom = false;
    sim->n_seen = 0;
    sim->n_events = 0;
    sim->seg_t.clear();
    sim->seg_off.assign(1, 0);
  });
}

void evsim_gpu_destroy(evsim_gpu_sim* sim) {
  if (!sim) return;
  cudaSetDevice(sim->device);
  cudaStreamSynchronize(sim->stream);
  cudaStream_t s = sim->stream;
  delete sim;  // DevBufs free on the stream (pool)
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

int64_t evsim_gpu_kernel_launches(const evsim_gpu_sim* sim) { return sim ? sim->launches : 0; }

int evsim_gpu_set_profiling(evsim_gpu_sim* sim, int32_t enable) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_set_profiling: null simulator");
    CK(cudaSetDevice(sim->device));
    sim->collect();
    sim->profiling = enable != 0;
    for (double& v : sim->stage_ms) v = 0.0;
    sim->timed_pushes = 0;
  });
}

int evsim_gpu_stage_times(evsim_gpu_sim* sim, double* ms, int32_t n_stages, int64_t* n_pushes) {
  return guarded([&] {
    if (!sim) invalid("evsim_gpu_stage_times: null simulator");
    CK(cudaSetDevice(sim->device));
    sim->collect();
    for (int i = 0; i < n_stages && i < EVSIM_N_STAGES; ++i) ms[i] = sim->stage_ms[i];
    if (n_pushes) *n_pushes = sim->timed_pushes;
  });
}

// ------------------------------------------------------------ stateless entry points

namespace {

// Scratch simulator for the free functions: one (prev, curr) pair in ring
// slots 0 and 1.
// Stateless entry points (estimate_dense_flow, interpolate_frames, the
// *_events_with_flow functions) run on a scratch simulator.  Idle scratch
// simulators are kept per thread (up to 4, keyed by config and frame size)
// and reused, so a repeated call costs its uploads, kernels and downloads
// only — not a stream, pinned buffers and device allocations each time.
struct ScratchCache {
  struct Entry {
    evsim_gpu_config cfg;
    int w, h;
    evsim_gpu_sim* s;
  };
  std::vector<Entry> idle;
};
ScratchCache& scratch_cache() {
  // leaked on purpose: thread-exit destructors may run after the CUDA runtime is gone
  static thread_local ScratchCache* c = new ScratchCache();
  return *c;
}
void destroy_scratch(evsim_gpu_sim* s) {
  cudaStream_t st = s->stream;
  cudaStreamSynchronize(st);
  delete s;
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
}

struct Scratch {
  std::unique_ptr<evsim_gpu_sim> s;
  evsim_gpu_config key{};
  int kw = 0, kh = 0;
  Scratch(const evsim_gpu_config& cfg, int w, int h, const uint8_t* prev, const uint8_t* curr) {
    CK(cudaSetDevice(0));
    init_pool(0);
    key = cfg;
    kw = w;
    kh = h;
    auto& cache = scratch_cache().idle;
    for (size_t i = 0; i < cache.size(); ++i) {
      if (cache[i].w == w && cache[i].h == h && std::memcmp(&cache[i].cfg, &cfg, sizeof cfg) == 0) {
        s.reset(cache[i].s);
        cache.erase(cache.begin() + (long)i);
        break;
      }
    }
    if (!s) {
      s = std::make_unique<evsim_gpu_sim>();
      make_sim(s.get(), cfg, 0);
      s->allocate(w, h);
      s->ensure_capacity(1);
    }
    const size_t P = (size_t)w * h;
    CK(cudaMemcpyAsync(s->frames.p, prev, P, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->frames.as<uint8_t>() + P, curr, P, cudaMemcpyHostToDevice, s->stream));
  }
  ~Scratch() {
    if (!s) return;
    // a call that failed part-way is not reused (its buffers may be half-written)
    if (cudaStreamSynchronize(s->stream) == cudaSuccess && std::uncaught_exceptions() == 0) {
      auto& cache = scratch_cache().idle;
      if (cache.size() >= 4) {
        destroy_scratch(cache.front().s);
        cache.erase(cache.begin());
      }
      cache.push_back(ScratchCache::Entry{key, kw, kh, s.release()});
      return;
    }
    destroy_scratch(s.release());
  }
  evsim_gpu_sim* operator->() { return s.get(); }
  void pyramids() {
    PyramidParams pp = s->flow.pyramid_params(s->frames.as<uint8_t>(), (size_t)s->w * s->h,
                                              s->uses_flow() ? s->quads.as<uint32_t>() : nullptr, 0);
    launch_pyramid(pp, 2, s->stream);
    CK_LAUNCH("pyramid");
  }
};

void check_frames(const uint8_t* a, const uint8_t* b, int w, int h, const char* who) {
  if (!a || !b || w <= 0 || h <= 0) invalid(std::string(who) + ": empty frame");
}

void copy_events24(evsim_gpu_sim* s, evsim_event* events, int64_t capacity, int64_t* n_events) {
  *n_events = s->n_events;
  if (!events || capacity <= 0 || s->n_events == 0) return;
  if (capacity < s->n_events) invalid("events: destination too small");
  DevBuf tmp;
  tmp.ensure((size_t)s->n_events * 24, s->stream);
  launch_unpack_events(s->ev.events.as<uint32_t>(), s->ev.seg_out.as<int64_t>(), s->n_events, tmp.p, s->stream);
  CK_LAUNCH("unpack");
  CK(cudaMemcpyAsync(events, tmp.p, (size_t)s->n_events * 24, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
}

}  // namespace

int evsim_gpu_dense_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h, int32_t levels,
                         int32_t iterations, int32_t radius, float* du, float* dv) {
  return guarded([&] {
    validate_preset(Preset{levels, iterations, radius});
    check_frames(prev, curr, w, h, "estimate_dense_flow");
    evsim_gpu_config cfg;
    evsim_gpu_config_defaults(EVSIM_METHOD_DENSE, &cfg);
    cfg.pyramid_levels = levels;
    cfg.iterations_per_level = iterations;
    cfg.patch_radius = radius;
    Scratch s(cfg, w, h, prev, curr);
    s.pyramids();
    s->flow.solve(0, 1, s->frames.as<uint8_t>(), s->quads.as<uint32_t>(), s->stream);
    DevBuf field;
    field.ensure((size_t)w * h * 8, s->stream);
    launch_densify(s->flow.geom[0], field.as<float>(), field.as<float>() + (size_t)w * h, s->stream);
    CK_LAUNCH("densify");
    CK(cudaMemcpyAsync(du, field.p, (size_t)w * h * 4, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(dv, field.as<float>() + (size_t)w * h, (size_t)w * h * 4, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int evsim_gpu_sparse_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h, int32_t levels,
                          int32_t iterations, int32_t radius, const int32_t* pts, int64_t n_points, float* disp,
                          uint8_t* status) {
  return guarded([&] {
    validate_preset(Preset{levels, iterations, radius});
    check_frames(prev, curr, w, h, "estimate_sparse_flow");
    std::vector<uint32_t> idx((size_t)std::max<int64_t>(n_points, 1));
    for (int64_t i = 0; i < n_points; ++i) {
      const int x = pts[2 * i], y = pts[2 * i + 1];
      if (x < 0 || x >= w || y < 0 || y >= h) invalid("estimate_sparse_flow: point outside frame bounds");
      idx[i] = (uint32_t)y * (uint32_t)w + (uint32_t)x;
    }
    for (int64_t i = 0; i < n_points; ++i) {
      disp[2 * i] = disp[2 * i + 1] = 0.0f;
      status[i] = 0;
    }
    if (n_points == 0) return;
    evsim_gpu_config cfg;
    evsim_gpu_config_defaults(EVSIM_METHOD_SPARSE, &cfg);
    cfg.n_interp = 1;
    cfg.pyramid_levels = levels;
    cfg.iterations_per_level = iterations;
    cfg.patch_radius = radius;
    Scratch s(cfg, w, h, prev, curr);
    s.pyramids();
    DevBuf dpts, ddisp, dst;
    dpts.ensure((size_t)n_points * 4, s->stream);
    ddisp.ensure((size_t)n_points * 8, s->stream);
    dst.ensure((size_t)n_points, s->stream);
    CK(cudaMemcpyAsync(dpts.p, idx.data(), (size_t)n_points * 4, cudaMemcpyHostToDevice, s->stream));
    SparseLKParams lk = s->flow.sparse_params(0, s->quads.as<uint32_t>());
    lk.points = dpts.as<uint32_t>();
    lk.n_points = nullptr;
    lk.n_points_host = n_points;
    lk.disp = ddisp.as<float2>();
    lk.status = dst.as<uint8_t>();
    launch_sparse_lk(lk, (int)std::min<int64_t>(n_points, INT32_MAX), 1, s->stream);
    CK_LAUNCH("sparse_lk");
    CK(cudaMemcpyAsync(disp, ddisp.p, (size_t)n_points * 8, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(status, dst.p, (size_t)n_points, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int evsim_gpu_interpolate_frames(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h, int64_t t_prev,
                                 int64_t t_curr, const float* du, const float* dv, int32_t n, uint8_t* out,
                                 int64_t* out_t) {
  return guarded([&] {
    check_frames(prev, curr, w, h, "interpolate_frames");
    if (n < 0) invalid("interpolate_frames: n must be >= 0");  // simulate.cpp:97
    for (int k = 1; k <= n; ++k) out_t[k - 1] = sub_interval_end(t_prev, t_curr, k, n + 1);
    if (n == 0) return;
    evsim_gpu_config cfg;
    evsim_gpu_config_defaults(EVSIM_METHOD_DENSE, &cfg);
    cfg.n_interp = n;
    Scratch s(cfg, w, h, prev, curr);
    const size_t P = (size_t)w * h;
    launch_build_quad(s->frames.as<uint8_t>(), s->quads.as<uint32_t>(), w, h, s->stream);
    launch_build_quad(s->frames.as<uint8_t>() + P, s->quads.as<uint32_t>() + P, w, h, s->stream);
    DevBuf field, dout;
    field.ensure(P * 8, s->stream);
    dout.ensure(P * n, s->stream);
    CK(cudaMemcpyAsync(field.p, du, P * 4, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(field.as<float>() + P, dv, P * 4, cudaMemcpyHostToDevice, s->stream));
    ChainParams c = s->chain_params(0, 1);
    c.du = field.as<float>();
    c.dv = field.as<float>() + P;
    launch_interp_frames(c, dout.as<uint8_t>(), s->stream);
    CK_LAUNCH("interp_frames");
    CK(cudaMemcpyAsync(out, dout.p, P * n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  });
}

int evsim_gpu_dense_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h, int64_t t_prev,
                                     int64_t t_curr, const float* du, const float* dv, const evsim_gpu_config* cfg_in,
                                     evsim_event* events, int64_t capacity, int64_t* n_events) {
  return guarded([&] {
    if (!cfg_in || !n_events) invalid("dense_events_with_flow: null argument");
    validate_config(*cfg_in);  // dense_events_with_flow: config.validate() (simulate.cpp:124)
    if (cfg_in->contrast_mode != EVSIM_CONTRAST_LINEAR)
      invalid("events_with_flow: stateless entry points are linear-mode only");
    check_frames(prev, curr, w, h, "dense_events_with_flow");
    evsim_gpu_config cfg = *cfg_in;
    cfg.method = EVSIM_METHOD_DENSE;
    Scratch s(cfg, w, h, prev, curr);
    const size_t P = (size_t)w * h;
    ChainParams c = s->chain_params(0, 1);
    DevBuf field;
    int provider = kProvNone;
    if (cfg.n_interp > 0) {
      launch_build_quad(s->frames.as<uint8_t>(), s->quads.as<uint32_t>(), w, h, s->stream);
      launch_build_quad(s->frames.as<uint8_t>() + P, s->quads.as<uint32_t>() + P, w, h, s->stream);
      field.ensure(P * 8, s->stream);
      CK(cudaMemcpyAsync(field.p, du, P * 4, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemcpyAsync(field.as<float>() + P, dv, P * 4, cudaMemcpyHostToDevice, s->stream));
      c.du = field.as<float>();
      c.dv = field.as<float>() + P;
      provider = kProvDenseField;
    }
    const int64_t ts[2] = {t_prev, t_curr};
    s->run_events(c, provider, ts, s->h_seg_out);
    s->finish();
    copy_events24(s.s.get(), events, capacity, n_events);
  });
}

int evsim_gpu_sparse_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                      int64_t t_prev, int64_t t_curr, const int32_t* pts, int64_t n_points,
                                      const float* disp, const uint8_t* st, const evsim_gpu_config* cfg_in,
                                      evsim_event* events, int64_t capacity, int64_t* n_events) {
  return guarded([&] {
    if (!cfg_in || !n_events) invalid("sparse_events_with_flow: null argument");
    validate_config(*cfg_in);
    if (cfg_in->contrast_mode != EVSIM_CONTRAST_LINEAR)
      invalid("events_with_flow: stateless entry points are linear-mode only");
    check_frames(prev, curr, w, h, "simulate_sparse");
    evsim_gpu_config cfg = *cfg_in;
    cfg.method = EVSIM_METHOD_SPARSE;
    const bool with_points = cfg.n_interp > 0 && n_points > 0;
    if (!with_points) cfg.n_interp = 0;  // chain_pipeline(prev, curr, {}) (simulate.cpp:161-163)
    Scratch s(cfg, w, h, prev, curr);
    ChainParams c = s->chain_params(0, 1);
    int provider = kProvNone;
    if (with_points) {
      std::vector<uint32_t> idx((size_t)n_points);
      for (int64_t i = 0; i < n_points; ++i) {
        const int x = pts[2 * i], y = pts[2 * i + 1];
        if (x < 0 || x >= w || y < 0 || y >= h) invalid("simulate_sparse: point outside frame bounds");
        idx[i] = (uint32_t)y * (uint32_t)w + (uint32_t)x;
      }
      const int np = (int)n_points;
      CK(cudaMemcpyAsync(s->points.p, idx.data(), (size_t)n_points * 4, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemcpyAsync(s->n_points.p, &np, sizeof np, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemcpyAsync(s->disp.p, disp, (size_t)n_points * 8, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemcpyAsync(s->status.p, st, (size_t)n_points, cudaMemcpyHostToDevice, s->stream));
      s->splat_stage(0, 1, c);
      provider = kProvSparse;
      CK(cudaStreamSynchronize(s->stream));  // host staging (np, idx) must outlive the copies
    }
    const int64_t ts[2] = {t_prev, t_curr};
    s->run_events(c, provider, ts, s->h_seg_out);
    s->finish();
    copy_events24(s.s.get(), events, capacity, n_events);
  });
}

}  // extern "C"
