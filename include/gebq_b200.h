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
/* Number of kernels this library has launched in the process (for audits). */
unsigned long long gebq_b200_launch_count(void);

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
/* The one cross-GPU exchange of the path: in place
 * ncclAllReduce(keys2, keys2, 2, ncclInt64, ncclMax, comm, stream) over the
 * two order keys of gebq_noa_minmax_* ([key(max), ~key(min)], both "larger is
 * more extreme"), so every rank then derives identical constants with
 * gebq_noa_derive_*.  `nccl_comm` is an ncclComm_t of the caller's NCCL (the
 * libnccl.so.2 loaded in the process is used; no link-time dependency).
 * Replaces the global reduction implied by compute_noa_range over the whole
 * array (quantizers.py:337-351) when the array is sharded.                  */
int gebq_noa_allreduce(long long *keys2, void *nccl_comm, void *stream);
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
/* gen_smooth: the C3 / C5-smooth field with counter-based noise (bench and
 * parity workloads; no reference counterpart -- the reference's synthetic
 * field, bench.py:357-374, draws numpy noise that a GPU cannot reproduce).
 * g = start_index + i, (ii, j, k) = digits of g in base side;
 * v = ((5*tab3[ii]) * tab3[side+j]) * tab3[2*side+k] + (s - 131070) * noise_scale
 * in binary64 (one rounding each), s = sum of the four 16-bit fields of
 * splitmix64(seed, g+1); out = v (width 64) or (float)v (width 32).  plant:
 * g=0 NaN, g=1 +Inf, g=2 -7, g=total-1 +7.  tab3 is a device array.        */
int gebq_gen_smooth(int width, void *out, int64_t n, int64_t side, const double *tab3,
                    uint64_t seed, int64_t start_index, int plant, int64_t total,
                    double noise_scale, void *stream);


/* ---- library-log REL variant: quantize_rel32_lib / reconstruct_rel32_lib
 * (_kernels.py:356-431).  Non-conforming by design (binary64 library
 * log2/exp2 instead of the bit-level approximations; GPU and host libm may
 * differ in the last ulp), bound still guaranteed by the double-check.
 * Benchmark comparisons only (bench.py:143-201 "library_log").              */
int gebq_quantize_rel_lib_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n, float op_eps,
                              float w, float thr, int unsafe, unsigned long long *trig4, void *stream);
int gebq_dequantize_rel_lib_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out, int64_t n, float w,
                                void *stream);

/* ---- verify: verify.py:88-153 on the device -------------------------------
 * rel = 1: bound = op_eps (same sign, q = |r|/|o|, q <= op_eps, q*op_eps >= 1);
 * rel = 0: bound = eb_eff (|o - r| <= eb_eff; ABS and NOA).  NaN/Inf
 * originals must match bit-exactly.  out5 = {violations (+=), special
 * mismatches (+=), first violation index (min; preset UINT64_MAX), max error
 * (|o-r| or |q-1| as binary64 bits, max; preset 0), unused}.  mask (optional,
 * n bytes): 1 violation, 2 special mismatch, 0 otherwise.                  */
int gebq_verify_f32(const uint32_t *original, const uint32_t *recon, int64_t n, int rel, float bound,
                    unsigned long long *out5, uint8_t *mask, void *stream);
int gebq_verify_f64(const uint64_t *original, const uint64_t *recon, int64_t n, int rel, double bound,
                    unsigned long long *out5, uint8_t *mask, void *stream);

/* ---- stream encode: quantize + pack into FORMAT.md in ONE pass ------------
 * Replaces quantize_* + block_sizes_* + cumsum + emit_blocks_* as driven by
 * pipeline.compress / container.encode_stream (pipeline.py:112-191,
 * container.py:235-259, _kernels.py:439-518/606-639).
 * Writes the block REGION (bitmaps + LEB128 varints) to `region` and the N
 * block offsets (u64, relative to the region start, plus base_offset) to
 * `index`; *region_len (device) receives the region byte count.  The host
 * adds the 48-byte header and the u64 block count (container.py:258).
 *   region capacity: gebq_encode_region_capacity(n, block_size, width) bytes
 *   workspace:       gebq_encode_workspace_bytes(n, block_size, width) bytes
 * base_offset lets a shard of a multi-GPU job write its part of the global
 * index directly (shard boundaries are multiples of block_size).            */
int64_t gebq_encode_region_capacity(int64_t n, int64_t block_size, int width);
size_t gebq_encode_workspace_bytes(int64_t n, int64_t block_size, int width);
int gebq_encode_abs_f32(const uint32_t *x, int64_t n, float eb_eff, float eb2, float inv_eb2,
                        float thr, int unsafe, int64_t block_size, uint8_t *region,
                        uint64_t *index, int64_t base_offset, void *ws, size_t ws_bytes,
                        unsigned long long *trig4, long long *region_len, void *stream);
int gebq_encode_abs_f64(const uint64_t *x, int64_t n, double eb_eff, double eb2, double inv_eb2,
                        double thr, int unsafe, int64_t block_size, uint8_t *region,
                        uint64_t *index, int64_t base_offset, void *ws, size_t ws_bytes,
                        unsigned long long *trig4, long long *region_len, void *stream);
int gebq_encode_rel_f32(const uint32_t *x, int64_t n, float op_eps, float w, float thr,
                        int unsafe, int64_t block_size, uint8_t *region, uint64_t *index,
                        int64_t base_offset, void *ws, size_t ws_bytes,
                        unsigned long long *trig4, long long *region_len, void *stream);
int gebq_encode_rel_f64(const uint64_t *x, int64_t n, double op_eps, double w, double thr,
                        int unsafe, int64_t block_size, uint8_t *region, uint64_t *index,
                        int64_t base_offset, void *ws, size_t ws_bytes,
                        unsigned long long *trig4, long long *region_len, void *stream);
int gebq_encode_noa_dev_f32(const uint32_t *x, int64_t n, const void *consts_dev, int unsafe,
                            int64_t block_size, uint8_t *region, uint64_t *index,
                            int64_t base_offset, void *ws, size_t ws_bytes,
                            unsigned long long *trig4, long long *region_len, void *stream);
int gebq_encode_noa_dev_f64(const uint64_t *x, int64_t n, const void *consts_dev, int unsafe,
                            int64_t block_size, uint8_t *region, uint64_t *index,
                            int64_t base_offset, void *ws, size_t ws_bytes,
                            unsigned long long *trig4, long long *region_len, void *stream);
/* encode_stream(CodedArray, header) (container.py:235-259): pack given codes */
int gebq_encode_coded_u32(const uint32_t *codes, const uint8_t *lossless, int64_t n,
                          int64_t block_size, uint8_t *region, uint64_t *index,
                          int64_t base_offset, void *ws, size_t ws_bytes, long long *region_len,
                          void *stream);
int gebq_encode_coded_u64(const uint64_t *codes, const uint8_t *lossless, int64_t n,
                          int64_t block_size, uint8_t *region, uint64_t *index,
                          int64_t base_offset, void *ws, size_t ws_bytes, long long *region_len,
                          void *stream);

/* ---- stream decode --------------------------------------------------------
 * validate_index: the index checks of decode_stream (container.py:283-291);
 *   flags3 = {first offset != 0, offsets decreasing, last offset > region_len}.
 * decode_{abs,rel}_*: unpack + reconstruct fused (decode_blocks_* then
 *   reconstruct_*, pipeline.py:195-213) straight to value bits.  Optional
 *   device-side inputs (NULL = use the scalar): region_len_dev (the encoder's
 *   *region_len, so decode can follow encode without a host round trip) and
 *   derived_dev (eb2 / w written by gebq_noa_derive_*: consts + 1 element).
 * decode_blocks_u{32,64}: decode_blocks_* (_kernels.py:642-664) to codes +
 *   lossless flags for blocks [b0, b1).
 * Errors: *err_key (device, caller sets UINT64_MAX) is atomically MIN-ed with
 *   (position << 2) | status, status 1 truncated / 2 non-canonical / 3 count
 *   mismatch (_kernels.py:33-37), position relative to the region -- the
 *   reference reports the failure with the smallest position
 *   (container.py:308-311).                                                  */
int gebq_validate_index(const int64_t *offsets, int64_t nblocks, int64_t region_len,
                        int *flags3, void *stream);
int gebq_decode_abs_f32(const uint8_t *region, int64_t region_len,
                        const long long *region_len_dev, const int64_t *offsets, int64_t nblocks,
                        int64_t count, int64_t block_size, float eb2, const void *derived_dev,
                        uint32_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_abs_f64(const uint8_t *region, int64_t region_len,
                        const long long *region_len_dev, const int64_t *offsets, int64_t nblocks,
                        int64_t count, int64_t block_size, double eb2, const void *derived_dev,
                        uint64_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_rel_f32(const uint8_t *region, int64_t region_len,
                        const long long *region_len_dev, const int64_t *offsets, int64_t nblocks,
                        int64_t count, int64_t block_size, float w, const void *derived_dev,
                        uint32_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_rel_f64(const uint8_t *region, int64_t region_len,
                        const long long *region_len_dev, const int64_t *offsets, int64_t nblocks,
                        int64_t count, int64_t block_size, double w, const void *derived_dev,
                        uint64_t *out, unsigned long long *err_key, void *stream);
/* Self-check of the production REL binary32 quantizers (the stream
 * encoder's exact-division one and the CodedArray kernel's division-free
 * filtered one) against the reference op sequence (quantize_rel32,
 * _kernels.py:165-224) for patterns [start, start+count) mod 2^32:
 * out2[0] += mismatching (code, trigger) outcomes -- must stay 0;
 * out2[1] is unused (0).                                                    */
/* Same for the production ABS/NOA binary32 quantizer (quantize_abs32,
 * _kernels.py:86-123): out2[0] += mismatching outcomes over the range.      */
int gebq_selfcheck_abs_f32(uint64_t start, int64_t count, float eb_eff, float eb2, float inv_eb2, float thr,
                           int unsafe, unsigned long long *out2, void *stream);
int gebq_selfcheck_rel_filter_f32(uint64_t start, int64_t count, float op_eps, float w, float thr,
                                  int unsafe, unsigned long long *out2, void *stream);
/* Self-check of the production binary64 quantizers (the stream encoder's and
 * CodedArray kernel's ABS op sequence and filtered REL quantizer) against the
 * reference op sequences (quantize_abs64 _kernels.py:126-162, quantize_rel64
 * :227-285) over `count` sampled patterns from splitmix64(seed): raw words,
 * moderate magnitudes, bin / double-check edges and range edges (see
 * k_check_f64).  out2[0] += mismatching (code, trigger) outcomes -- must stay
 * 0; out2[1] += patterns checked.                                           */
int gebq_selfcheck_abs_f64(uint64_t seed, int64_t count, double eb_eff, double eb2, double inv_eb2,
                           double thr, int unsafe, unsigned long long *out2, void *stream);
int gebq_selfcheck_rel_f64(uint64_t seed, int64_t count, double op_eps, double w, double thr, int unsafe,
                           unsigned long long *out2, void *stream);
/* The binary32 REL encoder's FCHK-free division against div.rn for any
 * bound w in [2^-100, 2^100] (sampled (l, w) pairs and double-check
 * quotients).  out2[0] += differing quotients; out2[1] += pairs checked.    */
int gebq_selfcheck_div_f32(uint64_t seed, int64_t count, unsigned long long *out2, void *stream);

/* decode_span_*: the fused decode restricted to blocks [b0, b1) of a stream
 * (same region / offsets / count as the whole-stream call; outputs land at
 * their absolute value positions).  Lets the host API decode early blocks
 * while later stream bytes are still being copied in.                      */
int gebq_decode_span_abs_f32(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, float eb2, int64_t b0,
                             int64_t b1, uint32_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_span_abs_f64(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, double eb2, int64_t b0,
                             int64_t b1, uint64_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_span_rel_f32(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, float w, int64_t b0,
                             int64_t b1, uint32_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_span_rel_f64(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, double w, int64_t b0,
                             int64_t b1, uint64_t *out, unsigned long long *err_key, void *stream);
int gebq_decode_blocks_u32(const uint8_t *buf, const int64_t *offsets, int64_t noffsets,
                           int64_t region_end, int64_t count, int64_t block_size, int64_t b0,
                           int64_t b1, uint32_t *codes, uint8_t *lossless,
                           unsigned long long *err_key, void *stream);
int gebq_decode_blocks_u64(const uint8_t *buf, const int64_t *offsets, int64_t noffsets,
                           int64_t region_end, int64_t count, int64_t block_size, int64_t b0,
                           int64_t b1, uint64_t *codes, uint8_t *lossless,
                           unsigned long long *err_key, void *stream);

/* ---- drop-ins for block_sizes_u{32,64} / emit_blocks_u{32,64} -------------
 * (_kernels.py:606-639): per-block encoded sizes and emission at given
 * offsets, blocks [b0, b1).                                                 */
int gebq_block_sizes_u32(const uint32_t *codes, int64_t count, int64_t block_size, int64_t b0,
                         int64_t b1, int64_t *sizes, void *stream);
int gebq_block_sizes_u64(const uint64_t *codes, int64_t count, int64_t block_size, int64_t b0,
                         int64_t b1, int64_t *sizes, void *stream);
int gebq_emit_blocks_u32(const uint32_t *codes, const uint8_t *lossless, int64_t count,
                         int64_t block_size, int64_t b0, int64_t b1, const int64_t *offsets,
                         uint8_t *out, void *stream);
int gebq_emit_blocks_u64(const uint64_t *codes, const uint8_t *lossless, int64_t count,
                         int64_t block_size, int64_t b0, int64_t b1, const int64_t *offsets,
                         uint8_t *out, void *stream);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* GEBQ_B200_H */
