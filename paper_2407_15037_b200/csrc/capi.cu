// capi.cu -- extern "C" entry points of libgebq_b200.so (include/gebq_b200.h).
// Thin: argument plumbing + error text; all work is in the kernel files.
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/gebq_b200.h"
#include "gebq_internal.cuh"


namespace gebq {

static thread_local std::string g_err;

int set_error(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return -(int)e;
}
int set_error_msg(int code, const char *msg) {
    g_err = msg;
    return code;
}
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(e, what);
    return 0;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached[dev] = v;
    }
    return cached[dev];
}
int resident_grid() { return sm_count() * (2048 / kThreads); }

}  // namespace gebq

using namespace gebq;

static inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

extern "C" {

int gebq_b200_abi_version(void) { return GEBQ_B200_ABI_VERSION; }
const char *gebq_b200_last_error(void) { return g_err.c_str(); }
int gebq_b200_sm_count(void) { return sm_count(); }

// ---- quantize ---------------------------------------------------------------
int gebq_quantize_abs_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                          float eb_eff, float eb2, float inv_eb2, float thr, int unsafe,
                          unsigned long long *trig4, void *stream) {
    Consts<float> k{eb_eff, eb2, inv_eb2, thr};
    return launch_quantize<float>(MODE_ABS, x, codes, lossless, n, k, nullptr, unsafe, trig4, S(stream));
}
int gebq_quantize_abs_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                          double eb_eff, double eb2, double inv_eb2, double thr, int unsafe,
                          unsigned long long *trig4, void *stream) {
    Consts<double> k{eb_eff, eb2, inv_eb2, thr};
    return launch_quantize<double>(MODE_ABS, x, codes, lossless, n, k, nullptr, unsafe, trig4, S(stream));
}
int gebq_quantize_rel_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                          float op_eps, float w, float thr, int unsafe,
                          unsigned long long *trig4, void *stream) {
    Consts<float> k{op_eps, w, 0.0f, thr};
    return launch_quantize<float>(MODE_REL, x, codes, lossless, n, k, nullptr, unsafe, trig4, S(stream));
}
int gebq_quantize_rel_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                          double op_eps, double w, double thr, int unsafe,
                          unsigned long long *trig4, void *stream) {
    Consts<double> k{op_eps, w, 0.0, thr};
    return launch_quantize<double>(MODE_REL, x, codes, lossless, n, k, nullptr, unsafe, trig4, S(stream));
}
int gebq_quantize_noa_dev_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n,
                              const void *consts_dev, int unsafe, unsigned long long *trig4,
                              void *stream) {
    Consts<float> k{0, 0, 0, 0};
    return launch_quantize<float>(MODE_ABS, x, codes, lossless, n, k, (const Consts<float> *)consts_dev,
                                  unsafe, trig4, S(stream));
}
int gebq_quantize_noa_dev_f64(const uint64_t *x, uint64_t *codes, uint8_t *lossless, int64_t n,
                              const void *consts_dev, int unsafe, unsigned long long *trig4,
                              void *stream) {
    Consts<double> k{0, 0, 0, 0};
    return launch_quantize<double>(MODE_ABS, x, codes, lossless, n, k, (const Consts<double> *)consts_dev,
                                   unsafe, trig4, S(stream));
}

// ---- dequantize -------------------------------------------------------------
int gebq_dequantize_abs_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out,
                            int64_t n, float eb2, void *stream) {
    return launch_reconstruct<float>(MODE_ABS, codes, lossless, out, n, eb2, S(stream));
}
int gebq_dequantize_abs_f64(const uint64_t *codes, const uint8_t *lossless, uint64_t *out,
                            int64_t n, double eb2, void *stream) {
    return launch_reconstruct<double>(MODE_ABS, codes, lossless, out, n, eb2, S(stream));
}
int gebq_dequantize_rel_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out,
                            int64_t n, float w, void *stream) {
    return launch_reconstruct<float>(MODE_REL, codes, lossless, out, n, w, S(stream));
}
int gebq_dequantize_rel_f64(const uint64_t *codes, const uint8_t *lossless, uint64_t *out,
                            int64_t n, double w, void *stream) {
    return launch_reconstruct<double>(MODE_REL, codes, lossless, out, n, w, S(stream));
}

// ---- NOA ----------------------------------------------------------------------
int gebq_noa_minmax_f32(const uint32_t *x, int64_t n, long long *keys2, void *stream) {
    return launch_noa_minmax<float>(x, n, keys2, S(stream));
}
int gebq_noa_minmax_f64(const uint64_t *x, int64_t n, long long *keys2, void *stream) {
    return launch_noa_minmax<double>(x, n, keys2, S(stream));
}
int gebq_noa_derive_f32(const long long *keys2, double eb, void *consts_out, double *range_out,
                        void *stream) {
    return launch_noa_derive<float>(keys2, eb, (Consts<float> *)consts_out, range_out, S(stream));
}
int gebq_noa_derive_f64(const long long *keys2, double eb, void *consts_out, double *range_out,
                        void *stream) {
    return launch_noa_derive<double>(keys2, eb, (Consts<double> *)consts_out, range_out, S(stream));
}

// ---- sweeps -------------------------------------------------------------------
int gebq_sweep_abs_f32(int source, const uint32_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, float eb_eff, float eb2, float inv_eb2, float thr,
                       int unsafe, unsigned long long *tally15,
                       unsigned long long *first_violation, void *stream) {
    Consts<float> k{eb_eff, eb2, inv_eb2, thr};
    return launch_sweep<float>(MODE_ABS, unsafe, source, start, count, bits, seed, k, tally15,
                               first_violation, S(stream));
}
int gebq_sweep_rel_f32(int source, const uint32_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, float op_eps, float w, float thr, int unsafe,
                       unsigned long long *tally15, unsigned long long *first_violation,
                       void *stream) {
    Consts<float> k{op_eps, w, 0.0f, thr};
    return launch_sweep<float>(MODE_REL, unsafe, source, start, count, bits, seed, k, tally15,
                               first_violation, S(stream));
}
int gebq_sweep_abs_f64(int source, const uint64_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, double eb_eff, double eb2, double inv_eb2, double thr,
                       int unsafe, unsigned long long *tally15,
                       unsigned long long *first_violation, void *stream) {
    Consts<double> k{eb_eff, eb2, inv_eb2, thr};
    return launch_sweep<double>(MODE_ABS, unsafe, source, start, count, bits, seed, k, tally15,
                                first_violation, S(stream));
}
int gebq_sweep_rel_f64(int source, const uint64_t *bits, uint64_t start, int64_t count,
                       uint64_t seed, double op_eps, double w, double thr, int unsafe,
                       unsigned long long *tally15, unsigned long long *first_violation,
                       void *stream) {
    Consts<double> k{op_eps, w, 0.0, thr};
    return launch_sweep<double>(MODE_REL, unsafe, source, start, count, bits, seed, k, tally15,
                                first_violation, S(stream));
}

// ---- generators -----------------------------------------------------------
int gebq_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index, void *stream) {
    return launch_splitmix64_fill(out, n, seed, start_index, S(stream));
}
int gebq_gen_mixed_f32(uint32_t *out, int64_t n, uint64_t seed, int64_t start_index, void *stream) {
    return launch_gen_mixed_f32(out, n, seed, start_index, S(stream));
}

}  // extern "C"
