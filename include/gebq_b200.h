/*
 * gebq_b200.h -- C ABI of libgebq_b200.so, the B200 (sm_100a) backend for the
 * gebq guaranteed-error-bound quantizers (LC, arXiv 2407.15037).
 *
 * The reference's operator boundary for the hot path is the set of numba
 * dispatchers in gebq._kernels (looked up by attribute at call time from
 * pipeline.py:106-109/203-206, container.py:243-305 and sweep.py:96-102).
 * Each entry point below replaces one of them; the comment names the
 * reference function (path relative to /root/reference/pkg/src/gebq/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers; calls are stream-ordered on
 *    `stream` (a cudaStream_t, NULL = legacy default stream) and return before
 *    the work completes.
 *  - Return 0 on success or a negative code; gebq_b200_last_error() gives
 *    the text (thread-local).  Kernels never fail on data: every input bit
 *    pattern has a defined output (SPEC.md: quantize is total).
 *  - Scalars are width-typed exactly as the reference derives them
 *    (quantizers.py:92-118): float for binary32 streams, double for binary64.
 *  - Counter outputs (trig4, tally15) are ACCUMULATED with device atomics:
 *    zero them before the call.  first_violation is atomically MIN-ed: set it
 *    to UINT64_MAX before the call.
 *  - lossless flags are one byte per value (numpy bool layout).
 *  - Results do not depend on grid size or partitioning: bit-identical to the
 *    reference for every input.
 */
#ifndef GEBQ_B200_H
#define GEBQ_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* exported even under -fvisibility=hidden */
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GEBQ_B200_ABI_VERSION 1

/* ---- library ------------------------------------------------------------ */
int gebq_b200_abi_version(void);
const char *gebq_b200_last_error(void);
/* SM count of the current device (a cheap probe that the CUDA backend works). */
int gebq_b200_sm_count(void);

/* ---- quantize: quantize_{abs,rel}{32,64} (_kernels.py:86-285) ------------
 * x -> (codes, lossless); trig4 += {nan, inf, guard, double_check} counts
 * (the int64[4] the reference returns, pipeline.py:155-165). NOA uses ABS.  */
int gebq_quantize_abs_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                          float eb_eff, float eb2, float inv_eb2, float thr, int unsafe,
                          unsigned long long *trig4, void *stream);
int gebq_quantize_abs_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                          double eb_eff, double eb2, double inv_eb2, double thr, int unsafe,
                          unsigned long long *trig4, void *stream);
int gebq_quantize_rel_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                          float op_eps, float w, float thr, int unsafe,
                          unsigned long long *trig4, void *stream);
int gebq_quantize_rel_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                          double op_eps, double w, double thr, int unsafe,
                          unsigned long long *trig4, void *stream);
/* NOA with constants produced on the device by gebq_noa_derive_* (no host sync):
 * consts_dev points at {eb_eff, eb2, inv_eb2, thr} in the value width.        */
int gebq_quantize_noa_dev_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                              const void *consts_dev, int unsafe, unsigned long long *trig4,
                              void *stream);
int gebq_quantize_noa_dev_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                              const void *consts_dev, int unsafe, unsigned long long *trig4,
                              void *stream);

/* ---- dequantize: reconstruct_{abs,rel}{32,64} (_kernels.py:293-354) -------
 * (codes, lossless) -> value bit patterns; derived = eb2 (ABS/NOA) or w (REL),
 * exactly the header's derived_bits (pipeline.py:202-213).                  */
int gebq_dequantize_abs_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out,
                            int64_t n, float eb2, void *stream);
int gebq_dequantize_abs_f64(const uint64_t *codes, const uint8_t *lossless, uint64_t *out,
                            int64_t n, double eb2, void *stream);
int gebq_dequantize_rel_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out,
                            int64_t n, float w, void *stream);
int gebq_dequantize_rel_f64(const uint64_t *codes, const uint8_t *lossless, uint64_t *out,
                            int64_t n, double w, void *stream);

/* ---- NOA range pass: compute_noa_range (quantizers.py:337-351) ----------
 * minmax: keys2[2] (int64, device) <- order-preserving keys of max / min over
 *   the finite values (overwritten, not accumulated).  Shards combine with
 *   ONE max-allreduce of the two int64 (ncclInt64 / torch.distributed MAX).
 * derive: keys2 -> R = max - min in the value width (+0 if no finite value),
 *   consts_out = {eb_eff = f(eb)*R, eb2, inv_eb2, thr} (quantizers.py:106-116),
 *   range_out = (double)R.  Both outputs are device pointers.                */
int gebq_noa_minmax_f32(const uint32_t *x, int64_t n, long long *keys2, void *stream);
int gebq_noa_minmax_f64(const uint64_t *x, int64_t n, long long *keys2, void *stream);
int gebq_noa_derive_f32(const long long *keys2, double eb, void *consts_out, double *range_out,
                        void *stream);
int gebq_noa_derive_f64(const long long *keys2, double eb, void *consts_out, double *range_out,
                        void *stream);

/* ---- sweeps: sweep_{abs,rel}{32,64}_on (_kernels.py:717-896) -------------
 * tally15[class*3 + outcome] += counts, classes {zero, denormal, normal, inf,
 * nan}, outcomes {quantized, lossless, violation}; first_violation <- min
 * sequence index of a violating pattern.  Constants: ABS/NOA (c0,c1,c2) =
 * (eb_eff, eb2, inv_eb2); REL (c0,c1) = (op_eps, w).
 *   _on:       patterns from a device array bits[n]
 *   _range:    pattern i = (start + i) mod 2^32 (sweep.py:165-169, exhaustive)
 *   _splitmix: pattern i = splitmix64(seed, start_index + i + 1), low 32 bits
 *              for f32 (sweep.py:194-202, sampled sweeps)                     */
int gebq_sweep_abs_f32(int source, const uint32_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, float eb_eff, float eb2, float inv_eb2, float thr,
                       int unsafe, unsigned long long *tally15,
                       unsigned long long *first_violation, void *stream);
int gebq_sweep_rel_f32(int source, const uint32_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, float op_eps, float w, float thr, int unsafe,
                       unsigned long long *tally15, unsigned long long *first_violation,
                       void *stream);
int gebq_sweep_abs_f64(int source, const uint64_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, double eb_eff, double eb2, double inv_eb2, double thr,
                       int unsafe, unsigned long long *tally15,
                       unsigned long long *first_violation, void *stream);
int gebq_sweep_rel_f64(int source, const uint64_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, double op_eps, double w, double thr, int unsafe,
                       unsigned long long *tally15, unsigned long long *first_violation,
                       void *stream);
#define GEBQ_SWEEP_SOURCE_RANGE 0
#define GEBQ_SWEEP_SOURCE_ARRAY 1
#define GEBQ_SWEEP_SOURCE_SPLITMIX 2

/* ---- device corpus generators -------------------------------------------
 * splitmix64_fill (_kernels.py:671-685): out[i] = splitmix64 number
 * start_index+i+1 for seed.  gen_mixed_f32: the C2 mixed-class recipe.     */
int gebq_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index,
                         void *stream);
int gebq_gen_mixed_f32(uint32_t *out, int64_t n, uint64_t seed, int64_t start_index,
                       void *stream);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* GEBQ_B200_H */
