// capi.cu -- extern "C" entry points of libgebq_b200.so (include/gebq_b200.h).
// Thin: argument plumbing + error text; all work is in the kernel files.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>

#include <dlfcn.h>

#include "../../include/gebq_b200.h"
#include "gebq_internal.cuh"
#include "gebq_stream.cuh"


namespace gebq {

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

void note_launch(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }

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
    note_launch(1);
    return 0;
}

int sm_count() {
    static std::atomic<int> cached[64];   // per device, 0 = not queried yet (idempotent fill)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cached[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}
int resident_grid() { return sm_count() * (2048 / kThreads); }

bool force_generic_kernels() {
    const char *v = getenv("GEBQ_B200_GENERIC");
    return v && v[0] == '1';
}

}  // namespace gebq

using namespace gebq;

static inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

extern "C" {

int gebq_b200_abi_version(void) { return GEBQ_B200_ABI_VERSION; }
const char *gebq_b200_last_error(void) { return g_err.c_str(); }
int gebq_b200_sm_count(void) { return sm_count(); }
unsigned long long gebq_b200_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

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

// ---- NOA cross-GPU exchange ----------------------------------------------------
// ncclAllReduce(keys2, keys2, 2, ncclInt64, ncclMax, comm, stream), resolved at
// run time from the libnccl.so.2 already loaded in the process (the one that
// created `comm`, e.g. torch's), else loaded here -- the library itself has
// no link-time NCCL dependency.
typedef int (*nccl_allreduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef const char *(*nccl_errstr_t)(int);
static nccl_allreduce_t g_nccl_allreduce = nullptr;
static nccl_errstr_t g_nccl_errstr = nullptr;
static std::once_flag g_nccl_once;

int gebq_noa_allreduce(long long *keys2, void *nccl_comm, void *stream) {
    std::call_once(g_nccl_once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        g_nccl_allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
        g_nccl_errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
    });
    if (!g_nccl_allreduce) return set_error_msg(-1, "noa_allreduce: libnccl.so.2 not available");
    if (!nccl_comm || !keys2) return set_error_msg(-1, "noa_allreduce: null communicator or keys");
    const int kInt64 = 4, kMax = 2;   // ncclInt64, ncclMax (nccl.h)
    int r = g_nccl_allreduce(keys2, keys2, 2, kInt64, kMax, nccl_comm, S(stream));
    if (r != 0) {
        std::string m = std::string("noa_allreduce: ncclAllReduce failed: ") +
                        (g_nccl_errstr ? g_nccl_errstr(r) : "unknown NCCL error");
        return set_error_msg(-1, m.c_str());
    }
    return 0;
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
int gebq_gen_smooth(int width, void *out, int64_t n, int64_t side, const double *tab3, uint64_t seed,
                    int64_t start_index, int plant, int64_t total, double noise_scale, void *stream) {
    if ((width != 32 && width != 64) || side <= 0 || n < 0) return set_error_msg(-1, "gen_smooth: bad arguments");
    return launch_gen_smooth(width, out, n, side, tab3, seed, start_index, plant, total, noise_scale, S(stream));
}
int gebq_quantize_rel_lib_f32(const uint32_t *x, uint32_t *codes, uint8_t *lossless, int64_t n, float op_eps,
                              float w, float thr, int unsafe, unsigned long long *trig4, void *stream) {
    return launch_rel32_lib_quantize(x, codes, lossless, n, op_eps, w, thr, unsafe, trig4, S(stream));
}
int gebq_dequantize_rel_lib_f32(const uint32_t *codes, const uint8_t *lossless, uint32_t *out, int64_t n, float w,
                                void *stream) {
    return launch_rel32_lib_reconstruct(codes, lossless, out, n, w, S(stream));
}
int gebq_verify_f32(const uint32_t *original, const uint32_t *recon, int64_t n, int rel, float bound,
                    unsigned long long *out5, uint8_t *mask, void *stream) {
    return launch_verify<float>(rel, original, recon, n, bound, out5, mask, S(stream));
}
int gebq_verify_f64(const uint64_t *original, const uint64_t *recon, int64_t n, int rel, double bound,
                    unsigned long long *out5, uint8_t *mask, void *stream) {
    return launch_verify<double>(rel, original, recon, n, bound, out5, mask, S(stream));
}

}  // extern "C"

// ---- stream encode / decode (FORMAT.md) ------------------------------------
extern "C" {

int64_t gebq_encode_region_capacity(int64_t n, int64_t block_size, int width) {
    return encode_region_capacity(n, block_size, width);
}
size_t gebq_encode_workspace_bytes(int64_t n, int64_t block_size, int width) {
    return encode_workspace_bytes(n, block_size, width);
}

#define ENC_CFG(MODE, SRC)                                                                \
    EncodeCfg cfg{MODE, SRC, unsafe, n, block_size, base_offset};

int gebq_encode_abs_f32(const uint32_t *x, int64_t n, float eb_eff, float eb2, float inv_eb2, float thr,
                        int unsafe, int64_t block_size, uint8_t *region, uint64_t *index,
                        int64_t base_offset, void *ws, size_t ws_bytes, unsigned long long *trig4,
                        long long *region_len, void *stream) {
    ENC_CFG(MODE_ABS, 0)
    Consts<float> k{eb_eff, eb2, inv_eb2, thr};
    return launch_encode<float>(cfg, x, nullptr, k, nullptr, region, index, ws, ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_abs_f64(const uint64_t *x, int64_t n, double eb_eff, double eb2, double inv_eb2, double thr,
                        int unsafe, int64_t block_size, uint8_t *region, uint64_t *index,
                        int64_t base_offset, void *ws, size_t ws_bytes, unsigned long long *trig4,
                        long long *region_len, void *stream) {
    ENC_CFG(MODE_ABS, 0)
    Consts<double> k{eb_eff, eb2, inv_eb2, thr};
    return launch_encode<double>(cfg, x, nullptr, k, nullptr, region, index, ws, ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_rel_f32(const uint32_t *x, int64_t n, float op_eps, float w, float thr, int unsafe,
                        int64_t block_size, uint8_t *region, uint64_t *index, int64_t base_offset,
                        void *ws, size_t ws_bytes, unsigned long long *trig4, long long *region_len,
                        void *stream) {
    ENC_CFG(MODE_REL, 0)
    Consts<float> k{op_eps, w, 0.0f, thr};
    return launch_encode<float>(cfg, x, nullptr, k, nullptr, region, index, ws, ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_rel_f64(const uint64_t *x, int64_t n, double op_eps, double w, double thr, int unsafe,
                        int64_t block_size, uint8_t *region, uint64_t *index, int64_t base_offset,
                        void *ws, size_t ws_bytes, unsigned long long *trig4, long long *region_len,
                        void *stream) {
    ENC_CFG(MODE_REL, 0)
    Consts<double> k{op_eps, w, 0.0, thr};
    return launch_encode<double>(cfg, x, nullptr, k, nullptr, region, index, ws, ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_noa_dev_f32(const uint32_t *x, int64_t n, const void *consts_dev, int unsafe,
                            int64_t block_size, uint8_t *region, uint64_t *index, int64_t base_offset,
                            void *ws, size_t ws_bytes, unsigned long long *trig4, long long *region_len,
                            void *stream) {
    ENC_CFG(MODE_ABS, 0)
    Consts<float> k{};
    return launch_encode<float>(cfg, x, nullptr, k, (const Consts<float> *)consts_dev, region, index, ws,
                                ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_noa_dev_f64(const uint64_t *x, int64_t n, const void *consts_dev, int unsafe,
                            int64_t block_size, uint8_t *region, uint64_t *index, int64_t base_offset,
                            void *ws, size_t ws_bytes, unsigned long long *trig4, long long *region_len,
                            void *stream) {
    ENC_CFG(MODE_ABS, 0)
    Consts<double> k{};
    return launch_encode<double>(cfg, x, nullptr, k, (const Consts<double> *)consts_dev, region, index, ws,
                                 ws_bytes, trig4, region_len, S(stream));
}
int gebq_encode_coded_u32(const uint32_t *codes, const uint8_t *lossless, int64_t n, int64_t block_size,
                          uint8_t *region, uint64_t *index, int64_t base_offset, void *ws,
                          size_t ws_bytes, long long *region_len, void *stream) {
    const int unsafe = 0;
    ENC_CFG(MODE_ABS, 1)
    Consts<float> k{};
    return launch_encode<float>(cfg, codes, lossless, k, nullptr, region, index, ws, ws_bytes, nullptr,
                                region_len, S(stream));
}
int gebq_encode_coded_u64(const uint64_t *codes, const uint8_t *lossless, int64_t n, int64_t block_size,
                          uint8_t *region, uint64_t *index, int64_t base_offset, void *ws,
                          size_t ws_bytes, long long *region_len, void *stream) {
    const int unsafe = 0;
    ENC_CFG(MODE_ABS, 1)
    Consts<double> k{};
    return launch_encode<double>(cfg, codes, lossless, k, nullptr, region, index, ws, ws_bytes, nullptr,
                                 region_len, S(stream));
}
#undef ENC_CFG

int gebq_validate_index(const int64_t *offsets, int64_t nblocks, int64_t region_len, int *flags3,
                        void *stream) {
    return launch_validate_index(offsets, nblocks, region_len, flags3, S(stream));
}

#define DEC_CFG(MODE, SINK) \
    DecodeCfg d{MODE, SINK, count, block_size, 0, nblocks, nblocks, region_len, region_len_dev, derived_dev};

int gebq_decode_abs_f32(const uint8_t *region, int64_t region_len, const long long *region_len_dev,
                        const int64_t *offsets, int64_t nblocks, int64_t count, int64_t block_size,
                        float eb2, const void *derived_dev, uint32_t *out, unsigned long long *err_key,
                        void *stream) {
    DEC_CFG(MODE_ABS, 1)
    return launch_decode<float>(d, region, offsets, eb2, out, nullptr, err_key, S(stream));
}
int gebq_decode_abs_f64(const uint8_t *region, int64_t region_len, const long long *region_len_dev,
                        const int64_t *offsets, int64_t nblocks, int64_t count, int64_t block_size,
                        double eb2, const void *derived_dev, uint64_t *out, unsigned long long *err_key,
                        void *stream) {
    DEC_CFG(MODE_ABS, 1)
    return launch_decode<double>(d, region, offsets, eb2, out, nullptr, err_key, S(stream));
}
int gebq_decode_rel_f32(const uint8_t *region, int64_t region_len, const long long *region_len_dev,
                        const int64_t *offsets, int64_t nblocks, int64_t count, int64_t block_size,
                        float w, const void *derived_dev, uint32_t *out, unsigned long long *err_key,
                        void *stream) {
    DEC_CFG(MODE_REL, 1)
    return launch_decode<float>(d, region, offsets, w, out, nullptr, err_key, S(stream));
}
int gebq_decode_rel_f64(const uint8_t *region, int64_t region_len, const long long *region_len_dev,
                        const int64_t *offsets, int64_t nblocks, int64_t count, int64_t block_size,
                        double w, const void *derived_dev, uint64_t *out, unsigned long long *err_key,
                        void *stream) {
    DEC_CFG(MODE_REL, 1)
    return launch_decode<double>(d, region, offsets, w, out, nullptr, err_key, S(stream));
}
#undef DEC_CFG

// span variants: blocks [b0, b1) of a stream whose bytes may still be arriving
// (the host-buffer API pipelines H2D of later blocks behind this decode)
#define SPAN_CFG(MODE) \
    DecodeCfg d{MODE, 1, count, block_size, b0, b1, nblocks, region_len, nullptr, nullptr};
int gebq_decode_span_abs_f32(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, float eb2, int64_t b0,
                             int64_t b1, uint32_t *out, unsigned long long *err_key, void *stream) {
    SPAN_CFG(MODE_ABS)
    return launch_decode<float>(d, region, offsets, eb2, out, nullptr, err_key, S(stream));
}
int gebq_decode_span_abs_f64(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, double eb2, int64_t b0,
                             int64_t b1, uint64_t *out, unsigned long long *err_key, void *stream) {
    SPAN_CFG(MODE_ABS)
    return launch_decode<double>(d, region, offsets, eb2, out, nullptr, err_key, S(stream));
}
int gebq_decode_span_rel_f32(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, float w, int64_t b0,
                             int64_t b1, uint32_t *out, unsigned long long *err_key, void *stream) {
    SPAN_CFG(MODE_REL)
    return launch_decode<float>(d, region, offsets, w, out, nullptr, err_key, S(stream));
}
int gebq_decode_span_rel_f64(const uint8_t *region, int64_t region_len, const int64_t *offsets,
                             int64_t nblocks, int64_t count, int64_t block_size, double w, int64_t b0,
                             int64_t b1, uint64_t *out, unsigned long long *err_key, void *stream) {
    SPAN_CFG(MODE_REL)
    return launch_decode<double>(d, region, offsets, w, out, nullptr, err_key, S(stream));
}
#undef SPAN_CFG

int gebq_selfcheck_abs_f32(uint64_t start, int64_t count, float eb_eff, float eb2, float inv_eb2, float thr,
                           int unsafe, unsigned long long *out2, void *stream) {
    Consts<float> k{eb_eff, eb2, inv_eb2, thr};
    return launch_check_abs_bf(start, count, k, unsafe, out2, S(stream));
}
int gebq_selfcheck_rel_filter_f32(uint64_t start, int64_t count, float op_eps, float w, float thr,
                                  int unsafe, unsigned long long *out2, void *stream) {
    Consts<float> k{op_eps, w, 0.0f, thr};
    return launch_check_rel_try(start, count, k, unsafe, out2, S(stream));
}

int gebq_selfcheck_abs_f64(uint64_t seed, int64_t count, double eb_eff, double eb2, double inv_eb2, double thr,
                           int unsafe, unsigned long long *out2, void *stream) {
    Consts<double> k{eb_eff, eb2, inv_eb2, thr};
    return launch_check_f64(MODE_ABS, seed, count, k, unsafe, out2, S(stream));
}
int gebq_selfcheck_rel_f64(uint64_t seed, int64_t count, double op_eps, double w, double thr, int unsafe,
                           unsigned long long *out2, void *stream) {
    Consts<double> k{op_eps, w, 0.0, thr};
    return launch_check_f64(MODE_REL, seed, count, k, unsafe, out2, S(stream));
}
int gebq_selfcheck_div_f32(uint64_t seed, int64_t count, unsigned long long *out2, void *stream) {
    return launch_check_div32(seed, count, out2, S(stream));
}

int gebq_decode_blocks_u32(const uint8_t *buf, const int64_t *offsets, int64_t noffsets, int64_t region_end,
                           int64_t count, int64_t block_size, int64_t b0, int64_t b1, uint32_t *codes,
                           uint8_t *lossless, unsigned long long *err_key, void *stream) {
    DecodeCfg d{MODE_ABS, 0, count, block_size, b0, b1, noffsets, region_end, nullptr, nullptr};
    return launch_decode<float>(d, buf, offsets, 0.0f, codes, lossless, err_key, S(stream));
}
int gebq_decode_blocks_u64(const uint8_t *buf, const int64_t *offsets, int64_t noffsets, int64_t region_end,
                           int64_t count, int64_t block_size, int64_t b0, int64_t b1, uint64_t *codes,
                           uint8_t *lossless, unsigned long long *err_key, void *stream) {
    DecodeCfg d{MODE_ABS, 0, count, block_size, b0, b1, noffsets, region_end, nullptr, nullptr};
    return launch_decode<double>(d, buf, offsets, 0.0, codes, lossless, err_key, S(stream));
}
int gebq_block_sizes_u32(const uint32_t *codes, int64_t count, int64_t block_size, int64_t b0, int64_t b1,
                         int64_t *sizes, void *stream) {
    return launch_block_sizes<uint32_t>(codes, count, block_size, b0, b1, sizes, S(stream));
}
int gebq_block_sizes_u64(const uint64_t *codes, int64_t count, int64_t block_size, int64_t b0, int64_t b1,
                         int64_t *sizes, void *stream) {
    return launch_block_sizes<uint64_t>(codes, count, block_size, b0, b1, sizes, S(stream));
}
int gebq_emit_blocks_u32(const uint32_t *codes, const uint8_t *lossless, int64_t count, int64_t block_size,
                         int64_t b0, int64_t b1, const int64_t *offsets, uint8_t *out, void *stream) {
    return launch_emit_blocks<uint32_t>(codes, lossless, count, block_size, b0, b1, offsets, out, S(stream));
}
int gebq_emit_blocks_u64(const uint64_t *codes, const uint8_t *lossless, int64_t count, int64_t block_size,
                         int64_t b0, int64_t b1, const int64_t *offsets, uint8_t *out, void *stream) {
    return launch_emit_blocks<uint64_t>(codes, lossless, count, block_size, b0, b1, offsets, out, S(stream));
}

}  // extern "C"
