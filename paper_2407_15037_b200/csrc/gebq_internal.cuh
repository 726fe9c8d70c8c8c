// gebq_internal.cuh -- launch geometry, error plumbing and launcher
// declarations shared by the kernel files and the C-ABI (capi.cu).
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "gebq_common.cuh"

namespace gebq {

constexpr int kThreads = 256;                  // 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kRows = 4;                       // rows of 128 values per lane-tile
constexpr int kTile = kThreads * 4 * kRows;    // 4096 values per CTA step

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// error state (thread-local text, returned codes are negative)
int set_error(cudaError_t e, const char *what);
int set_error_msg(int code, const char *msg);
int check_launch(const char *what);   // also counts one kernel launch
void note_launch(int k);                // count k further launches

// GEBQ_B200_GENERIC=1 routes block_size 4096 through the generic stream kernels
// (used by the tests to cover both code paths on the same inputs)
bool force_generic_kernels();

// SM count x resident CTAs of kThreads (queried once per device)
int sm_count();

// Raise Kern's dynamic shared memory limit to at least `smem` on the current
// device (the attribute belongs to the per-device module, so it is tracked per
// device; concurrent callers may both set it, which is harmless).  0 or the
// set_error code.
template <auto Kern>
inline int ensure_dyn_smem(int smem, const char *what) {
    static std::atomic<int> done[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    if (smem <= 48 * 1024 || done[dev].load(std::memory_order_acquire) >= smem) return 0;
    const cudaError_t e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(e, what);
    int cur = done[dev].load(std::memory_order_relaxed);
    while (cur < smem && !done[dev].compare_exchange_weak(cur, smem, std::memory_order_release)) {
    }
    return 0;
}
int resident_grid();
inline int grid_for(int64_t n) {
    int64_t tiles = (n + kTile - 1) / kTile;
    int g = resident_grid();
    if (tiles < 1) tiles = 1;
    return (int)(tiles < g ? tiles : g);
}
// grid of at most one full wave of Kern (its measured residency per SM, not the
// 2048-thread ideal): a grid-stride loop over a second, partial wave leaves SMs
// idle for a whole CTA lifetime
// Grids of the elementwise kernels, measured on B200 (C2 / C5 CodedArray stage):
// reconstruct streams best as one CTA per 4096-value tile
// (the block scheduler keeps every SM fed to the end; a resident-sized grid
// was 17 % slower), quantize best with 16 CTAs per SM oversubscribed (its
// register-limited residency is 5 CTAs; one exact wave was 6 % slower)
inline int grid_tiles(int64_t n) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    return (int)(tiles < 1 ? 1 : tiles < (1 << 30) ? tiles : (1 << 30));
}
inline int grid_per_sm(int64_t n, int per_sm) {
    int64_t tiles = (n + kTile - 1) / kTile;
    const int64_t g = (int64_t)sm_count() * per_sm;
    if (tiles < 1) tiles = 1;
    return (int)(tiles < g ? tiles : g);
}

template <typename T>
int launch_quantize(int mode, const void *x, void *codes, uint8_t *flags, int64_t n,
                    const Consts<T> &k, const Consts<T> *kdev, int unsafe,
                    unsigned long long *trig, cudaStream_t st);
template <typename T>
int launch_reconstruct(int mode, const void *codes, const uint8_t *flags, void *out, int64_t n,
                       T derived, cudaStream_t st);
template <typename T>
int launch_noa_minmax(const void *x, int64_t n, long long *keys2, cudaStream_t st);
template <typename T>
int launch_noa_derive(const long long *keys2, double eb, Consts<T> *kout, double *range_out,
                      cudaStream_t st);
template <typename T>
int launch_sweep(int mode, int unsafe, int source, uint64_t start, int64_t count, const void *bits,
                 uint64_t seed, const Consts<T> &k, unsigned long long *tally15,
                 unsigned long long *first, cudaStream_t st);
template <typename T>
int launch_verify(int rel, const void *o, const void *r, int64_t n, T bound, unsigned long long *out5,
                  uint8_t *mask, cudaStream_t st);
int launch_rel32_lib_quantize(const uint32_t *x, uint32_t *codes, uint8_t *flags, int64_t n, float op_eps, float w,
                              float thr, int unsafe, unsigned long long *trig, cudaStream_t st);
int launch_rel32_lib_reconstruct(const uint32_t *codes, const uint8_t *flags, uint32_t *out, int64_t n, float w,
                                 cudaStream_t st);
int launch_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index,
                           cudaStream_t st);
int launch_gen_smooth(int width, void *out, int64_t n, int64_t side, const double *tab, uint64_t seed,
                      int64_t start_index, int plant, int64_t total, double nz, cudaStream_t st);
int launch_gen_mixed_f32(uint32_t *out, int64_t n, uint64_t seed, int64_t start_index,
                         cudaStream_t st);

}  // namespace gebq
