// gebq_stream.cuh -- launchers for the FORMAT.md stream kernels (stream.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include "gebq_common.cuh"

namespace gebq {

// values per fused-encode tile (whole container blocks per tile)
constexpr int64_t kEncTileMax = 4096;

struct EncodeCfg {
    int mode;        // MODE_ABS / MODE_REL
    int src;         // 0 = quantize from values, 1 = pack given codes + flags
    int unsafe;
    int64_t n;
    int64_t block_size;
    int64_t base_offset;  // added to every index entry (multi-GPU shard placement)
};

int64_t encode_region_capacity(int64_t n, int64_t block_size, int width);
size_t encode_workspace_bytes(int64_t n, int64_t block_size, int width);

template <typename T>
int launch_encode(const EncodeCfg &cfg, const void *x, const uint8_t *flags_in, const Consts<T> &k,
                  const Consts<T> *kdev, uint8_t *region, uint64_t *index, void *ws,
                  size_t ws_bytes, unsigned long long *trig, long long *region_len,
                  cudaStream_t st);

// decode blocks [b0, b1) of a region; sink 0 = codes + flags, 1 = fused reconstruct
struct DecodeCfg {
    int mode;
    int sink;
    int64_t count;
    int64_t block_size;
    int64_t b0, b1;
    int64_t noffsets;
    int64_t region_end;
    const long long *region_end_dev;  // optional: region length produced on the device
    const void *derived_dev;          // optional: eb2 / w produced on the device (value width)
};

template <typename T>
int launch_decode(const DecodeCfg &cfg, const uint8_t *region, const int64_t *offsets, T derived,
                  void *out_codes, uint8_t *out_flags, unsigned long long *err_key,
                  cudaStream_t st);

size_t encode4k_workspace_bytes(int64_t n, int width);
template <typename T>
int launch_encode4k(const EncodeCfg &cfg, const void *x, const Consts<T> &k, const Consts<T> *kdev,
                    uint8_t *region, uint64_t *index, void *ws, unsigned long long *trig,
                    long long *region_len, cudaStream_t st);
template <typename T>
int launch_decode4k(const DecodeCfg &d, const uint8_t *region, const int64_t *offsets, T derived,
                    void *out_codes, uint8_t *out_flags, unsigned long long *err_key, cudaStream_t st);

int launch_check_f64(int mode, uint64_t seed, int64_t count, const Consts<double> &k, int unsafe,
                     unsigned long long *out2, cudaStream_t st);
int launch_check_div32(uint64_t seed, int64_t count, unsigned long long *out2, cudaStream_t st);
int launch_check_abs_bf(uint64_t start, int64_t count, const Consts<float> &k, int unsafe,
                        unsigned long long *out2, cudaStream_t st);
int launch_check_rel_try(uint64_t start, int64_t count, const Consts<float> &k, int unsafe,
                         unsigned long long *out2, cudaStream_t st);
int launch_validate_index(const int64_t *offsets, int64_t nblocks, int64_t region_len, int *flags3,
                          cudaStream_t st);

// drop-in container kernels (_kernels.block_sizes_* / emit_blocks_*)
template <typename U>
int launch_block_sizes(const U *codes, int64_t count, int64_t block_size, int64_t b0, int64_t b1,
                       int64_t *sizes, cudaStream_t st);
template <typename U>
int launch_emit_blocks(const U *codes, const uint8_t *flags, int64_t count, int64_t block_size,
                       int64_t b0, int64_t b1, const int64_t *offsets, uint8_t *out,
                       cudaStream_t st);

}  // namespace gebq
