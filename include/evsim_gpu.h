/*
 * evsim_gpu.h — C-ABI of the B200-native event-simulation hot path.
 *
 * Drop-in boundary for the reference simulator `evsim` (arXiv 2209.04634).
 * Every entry point below replaces one reference interface; the citation
 * names the reference file:line it stands in for (paths under
 * /root/reference/proj/).  Plain pointers and sizes only: no C++ or torch
 * types cross this boundary, so the reference's own C++ host (or ctypes,
 * cgo, JNI ...) can bind it directly.  See INTEGRATION.md.
 *
 * Semantics follow the reference exactly in contrast_mode LINEAR (the
 * reference's only mode): same integer thresholds, same strict
 * inequalities, same timestamps, same event order (t, y, x, p).  The LOG
 * mode is the BASELINE.json extension (log intensity + per-pixel reference
 * state); its rule is specified in DESIGN.md §3.
 *
 * Error handling mirrors the reference's exceptions: a non-zero status is
 * returned and evsim_gpu_last_error() holds the message text, which for
 * EVSIM_GPU_INVALID_ARGUMENT is the reference's exact std::invalid_argument
 * message (e.g. "push_frame: timestamps must be strictly increasing",
 * include/evsim/types.hpp + src/simulate.cpp:306-318).  A failed push leaves
 * the simulator state untouched (tests/test_simulate.cpp:66-74).
 */
#ifndef EVSIM_GPU_H_
#define EVSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EVSIM_GPU_API __attribute__((visibility("default")))
#else
#define EVSIM_GPU_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  EVSIM_GPU_OK = 0,
  EVSIM_GPU_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  EVSIM_GPU_RUNTIME = 2,          /* reference: std::runtime_error    */
  EVSIM_GPU_CUDA = 3              /* device / driver failure          */
};

/* ---- enums: same numbering as the reference's enum classes ------------- */
/* evsim::Method            include/evsim/types.hpp:82 */
enum { EVSIM_METHOD_DIFFERENCE_ONLY = 0, EVSIM_METHOD_DENSE = 1, EVSIM_METHOD_SPARSE = 2,
       EVSIM_METHOD_DIFFERENCE_INTERP = 3 };
/* evsim::FlowQuality       include/evsim/types.hpp:83 */
enum { EVSIM_FLOW_LOW_QUALITY = 0, EVSIM_FLOW_HIGH_QUALITY = 1 };
/* evsim::EventsPerCrossing include/evsim/types.hpp:86 */
enum { EVSIM_EVENTS_SINGLE = 0, EVSIM_EVENTS_MAGNITUDE = 1 };
/* extension (BASELINE.json configs): how a chain link is turned into events */
enum { EVSIM_CONTRAST_LINEAR = 0, EVSIM_CONTRAST_LOG = 1 };

/*
 * Mirrors evsim::SimulatorConfig field for field (include/evsim/types.hpp:88-131)
 * followed by the extension fields.  Zero-initialise, then call
 * evsim_gpu_config_defaults() for the reference's per-method defaults
 * (SimulatorConfig::defaults, types.hpp:101-120).
 */
typedef struct evsim_gpu_config {
  int32_t method;              /* EVSIM_METHOD_*                      */
  int32_t c_pos;               /* > 0, intensity units (linear mode)  */
  int32_t c_neg;               /* < 0                                 */
  int32_t n_interp;            /* >= 0                                */
  int32_t flow_preset;         /* EVSIM_FLOW_*                        */
  int32_t selection_threshold; /* 0 => c_pos (effective_selection_threshold) */
  int32_t events_per_crossing; /* EVSIM_EVENTS_*                      */
  int32_t include_endpoints;   /* bool                                */
  /* ---- extension ---- */
  int32_t contrast_mode;       /* EVSIM_CONTRAST_*                    */
  float c_pos_log;             /* > 0, log-intensity units (log mode) */
  float c_neg_log;             /* < 0                                 */
  float sel_log;               /* sparse selection in log mode, 0 => c_pos_log */
  /* Flow preset override (FlowPreset, include/evsim/flow.hpp:45-59); all
   * three 0 => flow_preset(flow_preset).  Used by the plug-in flow entry
   * points and by tests; the reference exposes the same knobs. */
  int32_t pyramid_levels;
  int32_t iterations_per_level;
  int32_t patch_radius;
} evsim_gpu_config;

/*
 * One event in exactly evsim::Event's in-memory layout (types.hpp:54-61):
 * x@0 (u16), y@2 (u16), t@8 (i64), p@16 (i8), sizeof 24.
 */
typedef struct evsim_event {
  uint16_t x;
  uint16_t y;
  int64_t t;
  int8_t p;
} evsim_event;

/*
 * Device-side packed event: bits 0-15 x, bits 16-30 y, bit 31 = 1 for
 * polarity -1.  Events of one push are stored contiguously in the
 * reference's output order; segment s (one distinct timestamp) covers
 * [seg_offset[s], seg_offset[s+1]).
 */
#define EVSIM_PACK_X(e) ((uint32_t)(e) & 0xFFFFu)
#define EVSIM_PACK_Y(e) (((uint32_t)(e) >> 16) & 0x7FFFu)
#define EVSIM_PACK_P(e) (((uint32_t)(e) >> 31) ? -1 : 1)

/* Result of one push; owned by the simulator, valid until the next
 * push / reset / destroy on the same handle. */
typedef struct evsim_gpu_events {
  int32_t width;
  int32_t height;
  int64_t n_events;
  int32_t n_segments;
  const int64_t* seg_t;      /* host, n_segments timestamps (strictly increasing) */
  const int64_t* seg_offset; /* host, n_segments + 1 offsets                       */
  const uint32_t* d_packed;  /* DEVICE pointer, n_events packed records            */
} evsim_gpu_events;

typedef struct evsim_gpu_sim evsim_gpu_sim;

/* Thread-local message of the last failing call on this thread. */
EVSIM_GPU_API const char* evsim_gpu_last_error(void);

/* SimulatorConfig::defaults(Method)  include/evsim/types.hpp:101-120 */
EVSIM_GPU_API void evsim_gpu_config_defaults(int32_t method, evsim_gpu_config* out);

/* SimulatorConfig::validate          include/evsim/types.hpp:126-130 */
EVSIM_GPU_API int evsim_gpu_config_validate(const evsim_gpu_config* cfg);

/* Simulator(SimulatorConfig)          include/evsim/simulate.hpp:62-77
 * device: CUDA ordinal.  Device memory is pooled per handle, so creating a
 * fresh simulator per timed pass (src/bench.cpp:53-64) stays cheap. */
EVSIM_GPU_API int evsim_gpu_create(const evsim_gpu_config* cfg, int device, evsim_gpu_sim** out);

/* Simulator::push_frame               src/simulate.cpp:306-347
 * pixels: width*height u8, row-major; on the host unless pixels_on_device.
 * Synchronous: on return `out` describes the events (device-resident). */
EVSIM_GPU_API int evsim_gpu_push_frame(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width, int32_t height,
                         int64_t t_us, int32_t pixels_on_device, evsim_gpu_events* out);

/* Batched Simulator::push_frame: n_frames consecutive frames (pixels:
 * n_frames*width*height bytes, t_us: n_frames host timestamps) in one launch
 * sequence.  Results are identical to n_frames push_frame calls with their
 * event streams concatenated (segments of all intervals, in order).  The
 * whole batch is validated first and rejected atomically (state untouched).
 * At most evsim_gpu_max_batch(sim, width, height) frames per call (bounded
 * by kernel shared-memory tables and a per-launch buffer budget of ~6 GB,
 * ~24 GB for frames of 4 Mpixel or more). */
EVSIM_GPU_API int evsim_gpu_push_frames(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames,
                                        int32_t width, int32_t height, const int64_t* t_us,
                                        int32_t pixels_on_device, evsim_gpu_events* out);
EVSIM_GPU_API int evsim_gpu_push_frames_async(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames,
                                              int32_t width, int32_t height, const int64_t* t_us,
                                              int32_t pixels_on_device);
EVSIM_GPU_API int evsim_gpu_max_batch(const evsim_gpu_sim* sim, int32_t width, int32_t height);

/* Row band (multi-GPU): this handle emits only the events of
 * frame rows [y0, y1) and solves only the flow patch rows they depend on,
 * from the full frames (every rank holds the whole frame).  Per timestamp the
 * reference orders events by (y, x), so the global stream is, per segment,
 * band 0's events, then band 1's, ...  (0, 0) = the whole frame (default).
 * Only at the start of a stream (before the first push or after reset);
 * dense and difference_only methods. */
EVSIM_GPU_API int evsim_gpu_set_row_band(evsim_gpu_sim* sim, int32_t y0, int32_t y1);

/* Several independent camera streams in one call (c4: many streams per GPU;
 * the reference runs one Simulator per thread, bench.cpp:53-64):
 * sims[i] gets the n_frames frames pixels[i] with timestamps t_us[i].  The
 * pushes are enqueued on the handles' own CUDA streams and run concurrently;
 * outs[i] (optional) is what evsim_gpu_push_frames would report for sims[i].
 * Every batch is validated before any is enqueued: one invalid batch rejects
 * the whole call and leaves every stream untouched. */
EVSIM_GPU_API int evsim_gpu_push_frames_batched(evsim_gpu_sim* const* sims, int32_t n_sims,
                                                const uint8_t* const* pixels, int32_t n_frames, int32_t width,
                                                int32_t height, const int64_t* const* t_us,
                                                int32_t pixels_on_device, evsim_gpu_events* outs);

/* Host frames in, host events out, overlapped: the frames are pushed in
 * chunks of about `chunk` frames (0 = 64; a quarter-size first and last
 * chunk); chunk j+1's upload and chunk j-1's event
 * download run on two copy streams while chunk j computes.  host_events
 * receives the packed records (format 0 of evsim_gpu_copy_events) of all
 * n_frames, in order; `out` gets the call's segment table, exactly as
 * evsim_gpu_push_frames would report it.  If capacity is too small the
 * simulation still completes, the call returns INVALID_ARGUMENT and the events
 * stay readable with evsim_gpu_copy_events.  Single-event mode only.
 * Same validation and errors as evsim_gpu_push_frames. */
EVSIM_GPU_API int evsim_gpu_push_frames_streamed(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames,
                                                 int32_t width, int32_t height, const int64_t* t_us, int32_t chunk,
                                                 uint32_t* host_events, int64_t capacity, evsim_gpu_events* out);

/* ---- compact lossless wire format ----------------------------------------
 * Replaces, for the caller that wants the events on the host, the 24-byte
 * std::vector<Event> the reference's push_frame returns
 * (include/evsim/types.hpp:54-80, src/simulate.cpp:306-347), carrying the
 * same events in ~1 bit per pixel-link + 1 bit per event.  The call's links
 * (every chain link of every frame pair, in stream order: chain_pipeline,
 * src/simulate.cpp:57-69) are numbered g = 0 .. n_links-1:
 *   link_t[g]        the link's timestamp (sub_interval_end, simulate.hpp:15-19)
 *   planes[g*words_per_link + w]  bit i set = an event of link g at pixel
 *                    x = 32*(w % words_per_row) + i, y = row0 + w / words_per_row
 *   link_events[g]   its number of events (= popcount of its plane)
 *   polarity         bit link_bit[g] + k (u32 words, LSB first) = 1 when the
 *                    k-th event of link g (plane order) has polarity -1
 * A link's events in plane order are the reference's (y, x) order; links
 * with equal timestamps form one reference segment, ordered (y, x, p)
 * (finalize's stable sort, src/simulate.cpp:36-40): evsim_gpu_wire_unpack
 * reproduces the reference's event stream exactly.  Single-event mode
 * (EVSIM_EVENTS_SINGLE) only. */
typedef struct evsim_gpu_wire {
  /* caller-owned host buffers (pinned memory lets the downloads overlap) */
  uint32_t* planes;
  int64_t planes_capacity;   /* u32 words */
  uint32_t* polarity;
  int64_t polarity_capacity; /* u32 words */
  int64_t* link_t;
  int64_t* link_events;
  int64_t* link_bit;
  int64_t link_capacity;     /* entries of each link array */
  /* filled by evsim_gpu_push_frames_wire */
  int64_t n_links;
  int32_t words_per_row;
  int32_t row0;
  int32_t rows;
  int32_t width;
  int64_t words_per_link;    /* rows * words_per_row */
  int64_t n_events;
  int64_t polarity_words;
} evsim_gpu_wire;

/* evsim_gpu_push_frames_streamed with the events delivered in the wire
 * format: host frames in, planes + polarity bits out, chunked and overlapped
 * the same way (chunk 0 = 64 frames).  Needs (links of the call) *
 * words_per_link plane words and about n_events/32 + 2*chunks polarity
 * words; too small buffers -> INVALID_ARGUMENT after the simulation
 * completed.  Same validation and errors as evsim_gpu_push_frames. */
EVSIM_GPU_API int evsim_gpu_push_frames_wire(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t n_frames,
                                             int32_t width, int32_t height, const int64_t* t_us, int32_t chunk,
                                             evsim_gpu_wire* wire, evsim_gpu_events* out);

/* Expand a wire buffer into the reference's event stream: format 0 packed u32
 * records (EVSIM_PACK_*), format 1 evsim_event (24 B), on `threads` host
 * threads (0 = all).  capacity in records. */
EVSIM_GPU_API int evsim_gpu_wire_unpack(const evsim_gpu_wire* wire, int32_t format, void* out, int64_t capacity,
                                        int32_t threads);

/* ---- multi-GPU merged output ------------------------------
 * One process per GPU; each rank's handle emits its row band (or its
 * streams).  The reference's single stream is, per timestamp, band 0's
 * events, then band 1's, ... (event order (t, y, x, p),
 * include/evsim/types.hpp:64-69, src/simulate.cpp:36-40); an all-gather of
 * per-(band, segment) counts gives every band's offset in it.
 * evsim_gpu_place_events copies the last push's segment s (the
 * evsim_gpu_events table) to dst + dst_offset[s] records — dst in this GPU's
 * or a peer GPU's memory (NVLink P2P; across processes via the CUDA IPC
 * calls below) — on the handle's stream (evsim_gpu_sync waits). */
EVSIM_GPU_API int evsim_gpu_place_events(evsim_gpu_sim* sim, uint32_t* dst, const int64_t* dst_offset,
                                         int32_t n_segments);
/* CUDA IPC of a device buffer: the 64-byte handle of dptr (cudaIpcGetMemHandle),
 * and the mapping of a peer process's buffer into this one (opened with lazy
 * peer access). */
EVSIM_GPU_API int evsim_gpu_ipc_handle(const void* dptr, void* handle64);
EVSIM_GPU_API int evsim_gpu_ipc_open(int32_t device, const void* handle64, void** dptr);
EVSIM_GPU_API int evsim_gpu_ipc_close(int32_t device, void* dptr);

/* Asynchronous variant: enqueues the push on the handle's CUDA stream and
 * returns without waiting; evsim_gpu_sync() completes it.  Validation
 * errors are still reported synchronously. */
EVSIM_GPU_API int evsim_gpu_push_frame_async(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width,
                               int32_t height, int64_t t_us, int32_t pixels_on_device);
EVSIM_GPU_API int evsim_gpu_sync(evsim_gpu_sim* sim, evsim_gpu_events* out);

/* Copy the last push's events to host memory.
 * format 0: packed u32 records (4 B each); format 1: evsim_event (24 B);
 * format 2: .evs records (13 B each: x u16, y u16, t u64, p i8, little
 * endian; src/io.cpp:158-165), formatted on the device.
 * capacity is in records; returns INVALID_ARGUMENT if too small. */
EVSIM_GPU_API int evsim_gpu_copy_events(evsim_gpu_sim* sim, void* host_dst, int64_t capacity, int32_t format);

/* ---- data formats either side of the path ------------- */
/* load_frames' pixel path (src/io.cpp:41-103): n_frames frames of w x h with
 * `channels` (1 gray, 3 RGB) -> luma_bt601 -> resize_bilinear to tw x th
 * ((0, 0) or (w, h) = no resize) -> dst (n_frames * tw * th bytes); host
 * buffers.  Errors as the reference ("resize_bilinear: target must be
 * positive"). */
EVSIM_GPU_API int evsim_gpu_ingest_frames(const uint8_t* src, int32_t channels, int32_t width, int32_t height,
                                          int32_t n_frames, int32_t target_width, int32_t target_height,
                                          uint8_t* dst);
/* write_events_binary / write_events_text (src/io.cpp:105-170) of the last
 * push's events; records formatted on the device.  I/O errors return
 * RUNTIME with the reference's message ("'<path>': cannot open for
 * writing"). */
EVSIM_GPU_API int evsim_gpu_write_events_binary(evsim_gpu_sim* sim, const char* path);
EVSIM_GPU_API int evsim_gpu_write_events_text(evsim_gpu_sim* sim, const char* path);
/* Simulator::push_frame with the flow from a caller's estimator
 * (Simulator(config, dense_flow, sparse_flow), include/evsim/simulate.hpp:68-77):
 * the handle keeps the stream's state — prev frame, the log reference state
 * (so log mode works through the plug-in seam) — and takes only the flow from
 * the caller.
 *   _with_flow   dense method: du, dv = the DenseFlowEstimator's FlowField for
 *                (prev, this frame), W*H floats each (ignored on the warm-up
 *                frame and when n_interp == 0);
 *   _with_tracks sparse method: the SparseFlowEstimator's result for the
 *                points the reference selects (|curr - prev| > selection
 *                threshold, scan order, simulate.cpp:150-157): n_points
 *                (x, y) pairs, 2*n_points displacements, n_points status.
 * difference_only handles accept either call (no flow).  A handle fed this
 * way takes only these pushes until evsim_gpu_reset.  Errors as
 * evsim_gpu_push_frame. */
EVSIM_GPU_API int evsim_gpu_push_frame_with_flow(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width,
                                                 int32_t height, int64_t t_us, const float* du, const float* dv,
                                                 evsim_gpu_events* out);
EVSIM_GPU_API int evsim_gpu_push_frame_with_tracks(evsim_gpu_sim* sim, const uint8_t* pixels, int32_t width,
                                                   int32_t height, int64_t t_us, const int32_t* points_xy,
                                                   int64_t n_points, const float* disp, const uint8_t* status,
                                                   evsim_gpu_events* out);
/* The log-intensity table of the log contrast mode:
 * lut[i] = logf(i / 255 + 1e-3), the exact fp32 values the kernels use — for
 * callers that restate the sparse selection |L[curr] - L[prev]| > sel_log on
 * the host (the flow plug-in seam, evsim_gpu_push_frame_with_tracks). */
EVSIM_GPU_API void evsim_gpu_log_lut(float* lut256);
/* difference_frame (include/evsim/core.hpp:8, src/core.cpp:5-19): values[i]
 * = curr[i] - prev[i] as int16 over w*h pixels (the caller checks that the
 * two frames have one size; the reference's message is "difference_frame:
 * incompatible input frames (WxH vs WxH)"). */
EVSIM_GPU_API int evsim_gpu_difference_frame(const uint8_t* prev, const uint8_t* curr, int32_t width, int32_t height,
                                             int16_t* values);
/* threshold_events / threshold_events_into (include/evsim/core.hpp:14-19,
 * src/core.cpp:21-52): the events of a difference frame's values, scan
 * order, every event at event_time; single or magnitude mode from the
 * config, which is validated first (INVALID with the reference's messages).
 * events == NULL (or capacity too small) only reports *n_events. */
EVSIM_GPU_API int evsim_gpu_threshold_events(const int16_t* values, int32_t width, int32_t height,
                                             const evsim_gpu_config* config, int64_t event_time, evsim_event* events,
                                             int64_t capacity, int64_t* n_events);
/* events_per_pixel_second (src/metrics.cpp:7-39): per-pixel counts on the
 * device, the fp64 reduction in the reference's pixel order on the host. */
EVSIM_GPU_API int evsim_gpu_events_per_pixel_second(const evsim_event* events, int64_t n, int32_t width,
                                                    int32_t height, double duration, double* mean_rate,
                                                    double* std_rate, uint64_t* total_events);
/* accumulate (src/metrics.cpp:41-69): PixelClass per pixel (0 none,
 * 1 positive, 2 negative, 3 both) over [t_start, t_end). */
EVSIM_GPU_API int evsim_gpu_accumulate(const evsim_event* events, int64_t n, int32_t width, int32_t height,
                                       int64_t t_start, int64_t t_end, uint8_t* classes);

/* CUDA stream (cudaStream_t) the handle enqueues on, for event timing. */
EVSIM_GPU_API void* evsim_gpu_stream(evsim_gpu_sim* sim);

/* Simulator::reset                    include/evsim/simulate.hpp:83-86 */
EVSIM_GPU_API int evsim_gpu_reset(evsim_gpu_sim* sim);
EVSIM_GPU_API void evsim_gpu_destroy(evsim_gpu_sim* sim);

/* ---- instrumentation --------------------------------------------------- */
/* Pipeline stages timed with CUDA events on the handle's stream. */
enum {
  EVSIM_STAGE_UPLOAD = 0,  /* frame H2D / D2D into the handle         */
  EVSIM_STAGE_PYRAMID = 1, /* quad image + pyramid of the new frame   */
  EVSIM_STAGE_FLOW = 2,    /* dense LK levels / sparse select+LK+splat */
  EVSIM_STAGE_CHAIN = 3,   /* interpolation + link chain + ballots    */
  EVSIM_STAGE_SCAN = 4,    /* (segment, block) offsets                */
  EVSIM_STAGE_EMIT = 5,    /* ordered event compaction                */
  EVSIM_N_STAGES = 6
};
/* enable != 0 starts per-stage event timing (and clears the totals).  While
 * enabled, a dense push runs its stages serially on the handle's stream (the
 * flow of the next sub-batch no longer overlaps the chain of the current one),
 * so stage times add up to the push time. */
EVSIM_GPU_API int evsim_gpu_set_profiling(evsim_gpu_sim* sim, int32_t enable);
/* Accumulated device milliseconds per stage and number of timed pushes
 * since profiling was enabled (waits for queued work). */
EVSIM_GPU_API int evsim_gpu_stage_times(evsim_gpu_sim* sim, double* ms, int32_t n_stages, int64_t* n_pushes);

/* Number of kernels this handle launched so far (instrumentation). */
EVSIM_GPU_API int64_t evsim_gpu_kernel_launches(const evsim_gpu_sim* sim);

/* ---- free functions / plug-in seams (stateless, synchronous) ----------- */

/* estimate_dense_flow / PyramidalPatchFlow::estimate
 *   src/flow.cpp:260-276, include/evsim/flow.hpp:64,88-97
 * du, dv: host buffers of width*height floats. */
EVSIM_GPU_API int evsim_gpu_dense_flow(const uint8_t* prev, const uint8_t* curr, int32_t width, int32_t height,
                         int32_t pyramid_levels, int32_t iterations, int32_t patch_radius,
                         float* du, float* dv);

/* estimate_sparse_flow / PyramidalLucasKanade::estimate
 *   src/flow.cpp:278-381, include/evsim/flow.hpp:69-70,100-110
 * pts: 2*M int32 (x, y); disp: 2*M float (du, dv); status: M bytes. */
EVSIM_GPU_API int evsim_gpu_sparse_flow(const uint8_t* prev, const uint8_t* curr, int32_t width, int32_t height,
                          int32_t pyramid_levels, int32_t iterations, int32_t patch_radius,
                          const int32_t* pts, int64_t n_points, float* disp, uint8_t* status);

/* interpolate_frames                  src/simulate.cpp:91-121
 * out: n*width*height bytes, out_t: n timestamps. */
EVSIM_GPU_API int evsim_gpu_interpolate_frames(const uint8_t* prev, const uint8_t* curr, int32_t width,
                                 int32_t height, int64_t t_prev, int64_t t_curr, const float* du,
                                 const float* dv, int32_t n, uint8_t* out, int64_t* out_t);

/* dense_events_with_flow              src/simulate.cpp:123-128
 * Caller-supplied flow: the seam a custom DenseFlowEstimator plugs into
 * (include/evsim/flow.hpp:74-78).  Events in evsim_event layout; the call
 * returns the count in *n_events and writes up to `capacity` records (pass
 * capacity 0 to query the size).  Linear mode only (the free function is
 * stateless). */
EVSIM_GPU_API int evsim_gpu_dense_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t width,
                                     int32_t height, int64_t t_prev, int64_t t_curr,
                                     const float* du, const float* dv,
                                     const evsim_gpu_config* cfg, evsim_event* events,
                                     int64_t capacity, int64_t* n_events);

/* simulate_sparse with caller-supplied sparse flow (a custom
 * SparseFlowEstimator, include/evsim/flow.hpp:80-85):
 * src/simulate.cpp:145-201 after the estimator call.  pts must be the
 * selection of src/simulate.cpp:149-159 in scan order. */
EVSIM_GPU_API int evsim_gpu_sparse_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t width,
                                      int32_t height, int64_t t_prev, int64_t t_curr,
                                      const int32_t* pts, int64_t n_points, const float* disp,
                                      const uint8_t* status, const evsim_gpu_config* cfg,
                                      evsim_event* events, int64_t capacity, int64_t* n_events);

#ifdef __cplusplus
}
#endif

#endif /* EVSIM_GPU_H_ */
