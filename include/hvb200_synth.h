/*
 * hvb200_synth.h — the synthetic benchmark workload, defined once.
 *
 * A counter-based generator (splitmix64 of a per-element counter), so the
 * GPU bench (device kernel), the reference CPU baseline (oracle/ref_bench.cpp)
 * and the tests all produce bit-identical datasets for any prefix or shard of
 * rows without replaying a sequential RNG.
 *
 * Shape semantics follow the reference's synthetic data (make_synth,
 * tests/support/synth.cpp:9-47): labels i % C, a per-(class, feature) centre
 * bin (c*(f+1) + 3f) mod 16, and a small jitter. The CHB-MIT label kind adds
 * the survey's imbalance: ~0.3 % positives in contiguous runs of 120 samples
 * (SURVEY.md §8d).
 */
#ifndef HVB200_SYNTH_H
#define HVB200_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define HVS_FN __host__ __device__ static inline
#else
#define HVS_FN static inline
#endif

enum { HVS_LABELS_MOD = 0, HVS_LABELS_CHBMIT = 1 };

HVS_FN uint64_t hvs_mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* label of global row i */
HVS_FN int32_t hvs_label(uint64_t i, uint32_t classes, int kind) {
  if (kind == HVS_LABELS_CHBMIT) return (i % 40000u) < 120u ? 1 : 0;
  return (int32_t)(i % classes);
}

/* bin of (row i, feature f) for a row labelled y; B bins */
HVS_FN uint32_t hvs_bin(uint64_t i, uint32_t f, uint32_t features, int32_t y, uint32_t bins,
                        uint64_t seed) {
  const uint32_t centre = (uint32_t)(((uint64_t)y * (f + 1u) + 3u * (uint64_t)f) % 16u) % bins;
  const uint64_t r = hvs_mix(seed ^ (i * (uint64_t)features + f) * 0xD6E8FEB86659FD93ULL);
  const uint32_t u = (uint32_t)(r >> 61); /* 0..7: 1/8 down, 1/8 up */
  if (u == 0 && centre > 0) return centre - 1;
  if (u == 1 && centre + 1 < bins) return centre + 1;
  return centre;
}

#endif
