/*
 * evsim_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference simulator's hot
 * path (arXiv 2209.04634 reference `evsim`, /root/reference/proj), used as
 * the parity checker for the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product library never links or calls it.
 *
 * Linear mode is pinned bit-for-bit against the compiled reference
 * (oracle/_ref, tests/test_oracle_vs_ref.py) and against golden fixtures
 * generated from it (tests/golden/, tests/golden/make_golden.py).  Log mode
 * has no reference implementation: its flow / interpolation / splat stages
 * are the pinned linear-mode code, only the per-link rule is
 * new, so the log rule itself is "parity unpinned" by the reference.
 *
 * Compiled with -O2 -ffp-contract=off -fno-fast-math: like the reference's
 * own x86-64 build (no -march, SSE2 scalar), no FMA contraction.
 */
#ifndef EVSIM_ORACLE_H_
#define EVSIM_ORACLE_H_

#include <stdint.h>

#include "evsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct evsim_oracle_sim evsim_oracle_sim;

const char* evsim_oracle_last_error(void);

/* log LUT: L[i] = logf(i / 255 + 1e-3) */
void evsim_oracle_log_lut(float* lut256);

int evsim_oracle_create(const evsim_gpu_config* cfg, evsim_oracle_sim** out);
void evsim_oracle_destroy(evsim_oracle_sim* sim);
int evsim_oracle_reset(evsim_oracle_sim* sim);
/* events valid until the next push/reset/destroy */
int evsim_oracle_push_frame(evsim_oracle_sim* sim, const uint8_t* pixels, int32_t w, int32_t h,
                            int64_t t, const evsim_event** events, int64_t* n_events);
/* log-mode reference state plane (NULL in linear mode / before the first frame) */
const float* evsim_oracle_ref_state(const evsim_oracle_sim* sim);

int evsim_oracle_dense_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                            int32_t levels, int32_t iters, int32_t radius, float* du, float* dv);
int evsim_oracle_sparse_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                             int32_t levels, int32_t iters, int32_t radius, const int32_t* pts,
                             int64_t n_points, float* disp, uint8_t* status);
int evsim_oracle_interpolate_frames(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                    int64_t t_prev, int64_t t_curr, const float* du,
                                    const float* dv, int32_t n, uint8_t* out, int64_t* out_t);
/* dense_events_with_flow; *events malloc'd, caller frees with evsim_oracle_free */
int evsim_oracle_dense_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w,
                                        int32_t h, int64_t t_prev, int64_t t_curr,
                                        const float* du, const float* dv,
                                        const evsim_gpu_config* cfg, evsim_event** events,
                                        int64_t* n_events);
int evsim_oracle_sparse_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w,
                                         int32_t h, int64_t t_prev, int64_t t_curr,
                                         const int32_t* pts, int64_t n_points, const float* disp,
                                         const uint8_t* status, const evsim_gpu_config* cfg,
                                         evsim_event** events, int64_t* n_events);
void evsim_oracle_free(void* p);

#ifdef __cplusplus
}
#endif

#endif
