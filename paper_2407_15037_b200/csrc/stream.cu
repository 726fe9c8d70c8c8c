// stream.cu -- FORMAT.md stream kernels (sm_100a).
//
// Encode (replaces block_sizes_* + cumsum + emit_blocks_* + the quantize pass,
// _kernels.py:86-285/439-518/606-639, container.py:241-258) is ONE pass over
// the input: a persistent CTA takes a tile of whole container blocks (ticket
// order), quantizes it in registers, scans the LEB128 lengths (warp shuffles
// + one CTA scan), publishes the tile's byte count and obtains its global
// offset with a decoupled look-back, then builds the tile's bytes (bitmap
// words + varints) in shared memory and streams them out with 16 B aligned
// stores.  HBM traffic = input once + output once.
//
// Decode (replaces decode_blocks_* + reconstruct_*, _kernels.py:521-603/
// 642-664/293-354) is one CTA per container block: the block's bytes are
// staged in shared memory, varint boundaries come from a CTA-wide scan of
// terminator bytes, values are parsed in parallel with the reference's exact
// canonical-form checks, and the reconstruction is fused into the store.
// Errors reduce to the minimum (position, status) key, which is exactly the
// reference's "first failure by byte position" rule (container.py:308-311).
#include <cub/device/device_scan.cuh>

#include "gebq_common.cuh"
#include "gebq_internal.cuh"
#include "gebq_stream.cuh"

namespace gebq {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_relaxed(const unsigned long long *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
        if (lane >= off) v += o;
    }
    return v;
}
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    return v;
}

// decoupled look-back (warp 0 of the CTA): returns the exclusive byte prefix
__device__ __forceinline__ uint64_t lookback(unsigned long long *tiles, int64_t tile, uint64_t total,
                                             int lane) {
    if (tile == 0) {
        if (lane == 0) st_relaxed(&tiles[0], kFlagPre | total);
        return 0;
    }
    if (lane == 0) st_relaxed(&tiles[tile], kFlagAgg | total);
    uint64_t excl = 0;
    int64_t base = tile - 1;
    for (;;) {
        int64_t j = base - lane;
        uint64_t s = kFlagPre;  // before tile 0: inclusive zero
        if (j >= 0) {
            do {
                s = ld_relaxed(&tiles[j]);
            } while ((s >> 62) == 0);
        }
        unsigned pm = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2);
        uint64_t v = s & kValMask;
        if (pm) {
            int first = __ffs(pm) - 1;
            if (lane > first) v = 0;
            excl += warp_sum_u64(v);
            break;
        }
        excl += warp_sum_u64(v);
        base -= 32;
    }
    if (lane == 0) st_relaxed(&tiles[tile], kFlagPre | (excl + total));
    return excl;
}

template <typename T>
struct EncArgs {
    using U = typename W<T>::U;
    const U *x;            // values (src 0) or codes (src 1)
    const uint8_t *fin;    // lossless flags (src 1)
    Consts<T> k;
    const Consts<T> *kdev;
    uint8_t *region;
    uint64_t *index;
    int64_t n, bs, K, V, ntiles, base_offset;
    int bmb;               // bitmap bytes of a full block
    int stage_bytes;
    int vec_ok;
    unsigned long long *tiles;
    unsigned int *ticket;
    unsigned long long *trig;
    long long *region_len;
};

// ---------------------------------------------------------------------------
// fused quantize + pack, tiles of whole container blocks (block_size <= 4096)
// ---------------------------------------------------------------------------
template <typename T, int kSrc, int kMode, bool kUnsafe>
__global__ void __launch_bounds__(kThreads) k_encode(EncArgs<T> a) {
    using X = W<T>;
    using U = typename X::U;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t *stage = smem;
    uint32_t *s_boff = reinterpret_cast<uint32_t *>(smem + a.stage_bytes);
    __shared__ uint32_t s_wsum[kWarps];
    __shared__ long long s_tile;
    __shared__ unsigned long long s_excl;

    Consts<T> k = a.k;
    if (a.kdev) k = *a.kdev;
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t out_mis = (uint32_t)((uintptr_t)a.region & 15u);
    const uint32_t bs32 = (uint32_t)a.bs;

    for (;;) {
        if (threadIdx.x == 0) s_tile = (long long)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= a.ntiles) break;
        const int64_t t0 = tile * a.V;
        const int64_t rem = a.n - t0;
        const uint32_t nv = (uint32_t)(rem < a.V ? rem : a.V);

        // ---- A: wire codes, flags and LEB128 lengths in registers ----
        U code[kRows][4];
        uint32_t lens[kRows];  // 4 x 8-bit lengths per row
        uint32_t lflag[kRows]; // 4 lossless bits per row
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            const uint32_t ti0 = warp * (kTile / kWarps) + r * 128 + 4 * lane;
            U raw[4];
            uint32_t fbytes = 0;
            if (a.vec_ok && ti0 + 3 < nv) {
                const U *p = a.x + t0 + ti0;
                if constexpr (sizeof(U) == 4) {
                    uint4 q = __ldcs(reinterpret_cast<const uint4 *>(p));
                    raw[0] = q.x; raw[1] = q.y; raw[2] = q.z; raw[3] = q.w;
                } else {
                    ulonglong2 q0 = __ldcs(reinterpret_cast<const ulonglong2 *>(p));
                    ulonglong2 q1 = __ldcs(reinterpret_cast<const ulonglong2 *>(p) + 1);
                    raw[0] = q0.x; raw[1] = q0.y; raw[2] = q1.x; raw[3] = q1.y;
                }
                if constexpr (kSrc == 1) fbytes = __ldcs(reinterpret_cast<const uint32_t *>(a.fin + t0 + ti0));
            } else {
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    raw[s] = 0;
                    if (ti0 + s < nv) {
                        raw[s] = a.x[t0 + ti0 + s];
                        if constexpr (kSrc == 1) fbytes |= (uint32_t)(a.fin[t0 + ti0 + s] != 0) << (8 * s);
                    }
                }
            }
            uint32_t lp = 0, fl = 0;
#pragma unroll
            for (int s = 0; s < 4; s++) {
                U c = raw[s];
                bool ll;
                if constexpr (kSrc == 0) {
                    int tr = quantize_one<T, kMode, kUnsafe>(raw[s], k, c);
                    ll = tr != TRIG_NONE;
                    if (ti0 + s < nv) {
                        c0 += tr == TRIG_NAN; c1 += tr == TRIG_INF; c2 += tr == TRIG_GUARD; c3 += tr == TRIG_DCHECK;
                    }
                } else {
                    ll = (fbytes >> (8 * s)) & 0xFF;
                }
                code[r][s] = c;
                const bool valid = ti0 + s < nv;
                lp |= (uint32_t)(valid ? varint_len(c) : 0) << (8 * s);
                fl |= (uint32_t)(valid && ll) << s;
            }
            lens[r] = lp;
            lflag[r] = fl;
        }

        // ---- B: byte positions (varint stream, tile-relative) ----
        uint32_t rowpre[kRows], rowoff[kRows];
        uint32_t wacc = 0;
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            uint32_t S = (lens[r] & 0xFF) + ((lens[r] >> 8) & 0xFF) + ((lens[r] >> 16) & 0xFF) + (lens[r] >> 24);
            uint32_t inc = warp_incl_scan(S, lane);
            rowpre[r] = inc - S;
            rowoff[r] = wacc;
            wacc += __shfl_sync(0xFFFFFFFFu, inc, 31);
        }
        if (lane == 0) s_wsum[warp] = wacc;
        __syncthreads();
        uint32_t wbase = 0, vtotal = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            uint32_t v = s_wsum[w];
            wbase += w < warp ? v : 0;
            vtotal += v;
        }
        const uint32_t kt = (nv + bs32 - 1) / bs32;                // blocks in this tile
        const uint32_t last_n = nv - (kt - 1) * bs32;              // values in its last block
        const uint32_t bm_last = ((last_n + 63) / 64) * 8;
        const uint32_t total = vtotal + (kt - 1) * (uint32_t)a.bmb + bm_last;
        // block start offsets inside the tile (bitmap first, then varints)
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            const uint32_t ti0 = warp * (kTile / kWarps) + r * 128 + 4 * lane;
            uint32_t p = wbase + rowoff[r] + rowpre[r];
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const uint32_t ti = ti0 + s;
                if (ti < nv && ti % bs32 == 0) {
                    const uint32_t kk = ti / bs32;
                    s_boff[kk] = p + kk * (uint32_t)a.bmb;
                }
                p += (lens[r] >> (8 * s)) & 0xFF;
            }
        }

        // ---- C: global offset of the tile (decoupled look-back) ----
        if (warp == 0) {
            uint64_t excl = lookback(a.tiles, tile, total, lane);
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        const uint64_t excl = s_excl;
        const uint32_t sh = (uint32_t)((out_mis + excl) & 15u);

        // ---- D: build the tile's bytes in shared memory ----
        {
            const uint32_t nz = (sh + total + 15) / 16;
            uint4 *z = reinterpret_cast<uint4 *>(stage);
            for (uint32_t i = threadIdx.x; i < nz; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            const uint32_t ti0 = warp * (kTile / kWarps) + r * 128 + 4 * lane;
            uint32_t p = wbase + rowoff[r] + rowpre[r];
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const uint32_t L = (lens[r] >> (8 * s)) & 0xFF;
                if (L) {
                    const uint32_t ti = ti0 + s;
                    const uint32_t kk = ti / bs32;
                    const uint32_t bmk = kk + 1 == kt ? bm_last : (uint32_t)a.bmb;
                    uint8_t *dst = stage + sh + p + kk * (uint32_t)a.bmb + bmk;
                    uint64_t c = (uint64_t)code[r][s];
                    for (uint32_t i = 0; i + 1 < L; i++) {
                        dst[i] = (uint8_t)((c & 0x7F) | 0x80);
                        c >>= 7;
                    }
                    dst[L - 1] = (uint8_t)c;
                }
                p += L;
            }
        }
        __syncthreads();
        // lossless bitmap bits (rare) and the block index entries
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            uint32_t fl = lflag[r];
            while (fl) {
                const int s = __ffs(fl) - 1;
                fl &= fl - 1;
                const uint32_t ti = warp * (kTile / kWarps) + r * 128 + 4 * lane + s;
                const uint32_t kk = ti / bs32;
                const uint32_t j = ti - kk * bs32;
                const uint32_t byte = sh + s_boff[kk] + (j >> 3);
                atomicOr(reinterpret_cast<unsigned int *>(stage + (byte & ~3u)),
                         1u << ((byte & 3u) * 8 + (j & 7u)));
            }
        }
        for (uint32_t kk = threadIdx.x; kk < kt; kk += kThreads)
            a.index[tile * a.K + kk] = (uint64_t)a.base_offset + excl + s_boff[kk];
        __syncthreads();

        // ---- E: stream the tile out (16 B aligned stores, byte-exact edges) ----
        {
            uint8_t *g = a.region + excl;
            const uint32_t head = (16 - ((out_mis + (uint32_t)(excl & 15u)) & 15u)) & 15u;
            if (head >= total) {
                for (uint32_t i = threadIdx.x; i < total; i += kThreads) g[i] = stage[sh + i];
            } else {
                const uint32_t nchunks = (total - head) / 16;
                const uint32_t tail0 = head + nchunks * 16;
                if (threadIdx.x < head) g[threadIdx.x] = stage[sh + threadIdx.x];
                if (threadIdx.x < total - tail0) g[tail0 + threadIdx.x] = stage[sh + tail0 + threadIdx.x];
                const uint4 *src = reinterpret_cast<const uint4 *>(stage + sh + head);
                uint4 *dst = reinterpret_cast<uint4 *>(g + head);
                for (uint32_t i = threadIdx.x; i < nchunks; i += kThreads) __stcs(dst + i, src[i]);
            }
        }
        if (tile == a.ntiles - 1 && threadIdx.x == 0) *a.region_len = (long long)(excl + total);
        __syncthreads();
    }
    if constexpr (kSrc == 0) {
        // trigger totals (same reduction as the elementwise quantizer)
        __shared__ unsigned long long s_trig[4];
        if (threadIdx.x < 4) s_trig[threadIdx.x] = 0;
        __syncthreads();
        c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
        c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
        c2 = __reduce_add_sync(0xFFFFFFFFu, c2);
        c3 = __reduce_add_sync(0xFFFFFFFFu, c3);
        if (lane == 0) {
            if (c0) atomicAdd(&s_trig[0], (unsigned long long)c0);
            if (c1) atomicAdd(&s_trig[1], (unsigned long long)c1);
            if (c2) atomicAdd(&s_trig[2], (unsigned long long)c2);
            if (c3) atomicAdd(&s_trig[3], (unsigned long long)c3);
        }
        __syncthreads();
        if (threadIdx.x < 4 && s_trig[threadIdx.x]) atomicAdd(&a.trig[threadIdx.x], s_trig[threadIdx.x]);
    }
}

// ---------------------------------------------------------------------------
// generic path (any block_size; also the drop-in block_sizes / emit_blocks):
// one warp per container block, 32 values per step.
// ---------------------------------------------------------------------------
template <typename T, int kSrc, int kMode, bool kUnsafe>
__device__ __forceinline__ bool gen_value(const typename W<T>::U *x, const uint8_t *fin, int64_t gi,
                                          const Consts<T> &k, typename W<T>::U &c, int &tr) {
    if constexpr (kSrc == 0) {
        tr = quantize_one<T, kMode, kUnsafe>(x[gi], k, c);
        return tr != TRIG_NONE;
    } else {
        tr = TRIG_NONE;
        c = x[gi];
        return fin[gi] != 0;
    }
}

template <typename T, int kSrc, int kMode, bool kUnsafe>
__global__ void __launch_bounds__(kThreads) k_gen_sizes(const typename W<T>::U *x, const uint8_t *fin,
                                                        Consts<T> k, const Consts<T> *kdev, int64_t n,
                                                        int64_t bs, int64_t b0, int64_t b1,
                                                        int64_t *sizes) {
    using U = typename W<T>::U;
    if (kdev) k = *kdev;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = b0 + gw; b < b1; b += nw) {
        const int64_t s = b * bs;
        const int64_t e = s + bs < n ? s + bs : n;
        uint64_t acc = 0;
        for (int64_t i = s + lane; i < e; i += 32) {
            U c;
            int tr;
            gen_value<T, kSrc, kMode, kUnsafe>(x, fin, i, k, c, tr);
            acc += varint_len(c);
        }
        acc = warp_sum_u64(acc);
        if (lane == 0) sizes[b] = (int64_t)acc + ((e - s + 63) / 64) * 8;
    }
}

template <typename T, int kSrc, int kMode, bool kUnsafe>
__global__ void __launch_bounds__(kThreads) k_gen_emit(const typename W<T>::U *x, const uint8_t *fin,
                                                       Consts<T> k, const Consts<T> *kdev, int64_t n,
                                                       int64_t bs, int64_t b0, int64_t b1,
                                                       const int64_t *offsets, uint8_t *out,
                                                       uint64_t *index, int64_t base_offset,
                                                       unsigned long long *trig) {
    using U = typename W<T>::U;
    if (kdev) k = *kdev;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    for (int64_t b = b0 + gw; b < b1; b += nw) {
        const int64_t s = b * bs;
        const int64_t e = s + bs < n ? s + bs : n;
        const int64_t off = offsets[b];
        if (index && lane == 0) index[b] = (uint64_t)(base_offset + off);
        int64_t pos = off + ((e - s + 63) / 64) * 8;
        for (int64_t c0 = s; c0 < e; c0 += 64) {
            uint64_t word = 0;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t i = c0 + 32 * h + lane;
                U c = 0;
                int tr = TRIG_NONE;
                bool ll = false;
                uint32_t L = 0;
                if (i < e) {
                    ll = gen_value<T, kSrc, kMode, kUnsafe>(x, fin, i, k, c, tr);
                    L = varint_len(c);
                    t0 += tr == TRIG_NAN; t1 += tr == TRIG_INF; t2 += tr == TRIG_GUARD; t3 += tr == TRIG_DCHECK;
                }
                word |= (uint64_t)__ballot_sync(0xFFFFFFFFu, ll) << (32 * h);
                uint32_t inc = warp_incl_scan(L, lane);
                uint8_t *dst = out + pos + (inc - L);
                uint64_t cc = (uint64_t)c;
                for (uint32_t q = 0; q + 1 < L; q++) {
                    dst[q] = (uint8_t)((cc & 0x7F) | 0x80);
                    cc >>= 7;
                }
                if (L) dst[L - 1] = (uint8_t)cc;
                pos += __shfl_sync(0xFFFFFFFFu, inc, 31);
            }
            if (lane < 8) out[off + ((c0 - s) / 64) * 8 + lane] = (uint8_t)(word >> (8 * lane));
        }
    }
    if (trig) {
        t0 = __reduce_add_sync(0xFFFFFFFFu, t0);
        t1 = __reduce_add_sync(0xFFFFFFFFu, t1);
        t2 = __reduce_add_sync(0xFFFFFFFFu, t2);
        t3 = __reduce_add_sync(0xFFFFFFFFu, t3);
        if (lane == 0) {
            if (t0) atomicAdd(&trig[0], (unsigned long long)t0);
            if (t1) atomicAdd(&trig[1], (unsigned long long)t1);
            if (t2) atomicAdd(&trig[2], (unsigned long long)t2);
            if (t3) atomicAdd(&trig[3], (unsigned long long)t3);
        }
    }
}

__global__ void k_region_len(const int64_t *offsets, const int64_t *sizes, int64_t nblocks,
                             long long *region_len) {
    *region_len = nblocks ? (long long)(offsets[nblocks - 1] + sizes[nblocks - 1]) : 0;
}

// ---------------------------------------------------------------------------
// decode
// ---------------------------------------------------------------------------
__device__ __forceinline__ void report_error(unsigned long long *err_key, int64_t pos, int status) {
    atomicMin(err_key, ((unsigned long long)pos << 2) | (unsigned long long)status);
}

template <typename T, int kSink, int kMode>
__device__ __forceinline__ void sink_put(void *out_codes, uint8_t *out_flags, int64_t gi,
                                         typename W<T>::U c, bool ll, T derived) {
    using U = typename W<T>::U;
    if constexpr (kSink == 0) {
        reinterpret_cast<U *>(out_codes)[gi] = c;
        out_flags[gi] = ll;
    } else {
        reinterpret_cast<U *>(out_codes)[gi] = reconstruct_one<T, kMode>(c, ll, derived);
    }
}

// One CTA per container block (64 <= block_size <= 4096).
template <typename T, int kSink, int kMode>
__global__ void __launch_bounds__(kThreads) k_decode_par(DecodeCfg d, const uint8_t *__restrict__ region,
                                                         const int64_t *__restrict__ offsets, T derived,
                                                         void *out_codes, uint8_t *out_flags,
                                                         unsigned long long *err_key, int buf_bytes) {
    using X = W<T>;
    using U = typename X::U;
    constexpr int MAXL = X::kMaxVarint;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t *buf = smem;
    uint16_t *tpos = reinterpret_cast<uint16_t *>(smem + buf_bytes);
    __shared__ uint32_t s_wsum[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (d.region_end_dev) d.region_end = *d.region_end_dev;
    if (d.derived_dev) derived = *reinterpret_cast<const T *>(d.derived_dev);

    for (int64_t b = d.b0 + blockIdx.x; b < d.b1; b += gridDim.x) {
        const int64_t s = b * d.block_size;
        const int64_t e = s + d.block_size < d.count ? s + d.block_size : d.count;
        const int nb = (int)(e - s);
        const int bmb = ((nb + 63) / 64) * 8;
        const int64_t start = offsets[b];
        const int64_t end = b + 1 < d.noffsets ? offsets[b + 1] : d.region_end;
        const int64_t size = end - start;
        if (size < bmb) {
            if (threadIdx.x == 0) report_error(err_key, start, DEC_TRUNCATED);
            continue;
        }
        const int64_t cap = (int64_t)bmb + (int64_t)nb * MAXL + 1;
        const int lsz = (int)(size < cap ? size : cap);
        // stage [start, start + lsz) at buf + (start & 15)
        const int boff = (int)(((uintptr_t)region + (uintptr_t)start) & 15u);
        {
            const int64_t a0 = start - boff;
            const int nch = (boff + lsz + 15) / 16;
            for (int c = threadIdx.x; c < nch; c += kThreads) {
                const int64_t g = a0 + 16 * (int64_t)c;
                if (g >= start && g + 16 <= d.region_end) {
                    *reinterpret_cast<uint4 *>(buf + 16 * c) = __ldcs(reinterpret_cast<const uint4 *>(region + g));
                } else {
                    for (int q = 0; q < 16; q++) {
                        const int64_t gq = g + q;
                        buf[16 * c + q] = (gq >= start && gq < start + lsz) ? region[gq] : 0;
                    }
                }
            }
        }
        __syncthreads();
        const uint8_t *pay = buf + boff + bmb;
        const int plen = lsz - bmb;                 // staged payload bytes
        const int64_t ptrue = size - bmb;           // true payload bytes of the block
        // terminator scan
        const int chunk = (plen + kThreads - 1) / kThreads;
        const int p0 = threadIdx.x * chunk;
        const int p1 = p0 + chunk < plen ? p0 + chunk : plen;
        uint32_t cnt = 0;
        for (int p = p0; p < p1; p++) cnt += (pay[p] & 0x80) == 0;
        uint32_t inc = warp_incl_scan(cnt, lane);
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        uint32_t wb = 0, nterm = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            wb += w < warp ? s_wsum[w] : 0;
            nterm += s_wsum[w];
        }
        uint32_t r = wb + inc - cnt;
        for (int p = p0; p < p1 && r < (uint32_t)nb; p++) {
            if ((pay[p] & 0x80) == 0) tpos[r++] = (uint16_t)p;
        }
        __syncthreads();
        // parse values in parallel
        for (int v = threadIdx.x; v < nb; v += kThreads) {
            if ((uint32_t)v > nterm) continue;  // beyond the first failure
            const int s0 = v == 0 ? 0 : tpos[v - 1] + 1;
            uint64_t val = 0;
            bool bad = false;
            if ((uint32_t)v < nterm) {
                const int ee = tpos[v];
                const int len = ee - s0 + 1;
                const int m = len < MAXL ? len : MAXL;
                for (int q = 0; q < m; q++) val |= (uint64_t)(pay[s0 + q] & 0x7F) << (7 * q);
                if constexpr (MAXL == 5) {
                    if (len > 5) { report_error(err_key, start + bmb + s0 + 5, DEC_NONCANONICAL); bad = true; }
                    else if (len > 1 && (pay[ee] & 0x7F) == 0) { report_error(err_key, start + bmb + ee, DEC_NONCANONICAL); bad = true; }
                    else if (val > 0xFFFFFFFFull) { report_error(err_key, start + bmb + ee, DEC_NONCANONICAL); bad = true; }
                } else {
                    if (len >= 10 && (pay[s0 + 9] & 0x7E) != 0) { report_error(err_key, start + bmb + s0 + 9, DEC_NONCANONICAL); bad = true; }
                    else if (len > 10) { report_error(err_key, start + bmb + s0 + 10, DEC_NONCANONICAL); bad = true; }
                    else if (len > 1 && (pay[ee] & 0x7F) == 0) { report_error(err_key, start + bmb + ee, DEC_NONCANONICAL); bad = true; }
                }
                if (!bad && v == nb - 1 && (int64_t)ee + 1 != ptrue)
                    report_error(err_key, start + bmb + ee + 1, DEC_COUNT_MISMATCH);
            } else {
                // no terminator left for this value: the sequential parse runs off the block
                const int64_t m = ptrue - s0;
                bad = true;
                if constexpr (MAXL == 5) {
                    if (m >= 6) report_error(err_key, start + bmb + s0 + 5, DEC_NONCANONICAL);
                    else report_error(err_key, end, DEC_TRUNCATED);
                } else {
                    if (m >= 10 && (pay[s0 + 9] & 0x7E) != 0) report_error(err_key, start + bmb + s0 + 9, DEC_NONCANONICAL);
                    else if (m >= 11) report_error(err_key, start + bmb + s0 + 10, DEC_NONCANONICAL);
                    else report_error(err_key, end, DEC_TRUNCATED);
                }
            }
            if (!bad) {
                const bool ll = (buf[boff + (v >> 3)] >> (v & 7)) & 1;
                sink_put<T, kSink, kMode>(out_codes, out_flags, s + v, (U)val, ll, derived);
            }
        }
        __syncthreads();
    }
}

// One thread per container block: the reference's sequential parse
// (decode_block_*, _kernels.py:521-603) for tiny or very large blocks.
template <typename T, int kSink, int kMode>
__global__ void __launch_bounds__(kThreads) k_decode_seq(DecodeCfg d, const uint8_t *__restrict__ region,
                                                         const int64_t *__restrict__ offsets, T derived,
                                                         void *out_codes, uint8_t *out_flags,
                                                         unsigned long long *err_key) {
    using X = W<T>;
    using U = typename X::U;
    constexpr int MAXL = X::kMaxVarint;
    if (d.region_end_dev) d.region_end = *d.region_end_dev;
    if (d.derived_dev) derived = *reinterpret_cast<const T *>(d.derived_dev);
    for (int64_t b = d.b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < d.b1;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = b * d.block_size;
        const int64_t e = s + d.block_size < d.count ? s + d.block_size : d.count;
        const int64_t nvals = e - s;
        int64_t pos = offsets[b];
        const int64_t endpos = b + 1 < d.noffsets ? offsets[b + 1] : d.region_end;
        const int64_t nwords = (nvals + 63) / 64;
        if (pos + nwords * 8 > endpos) { report_error(err_key, pos, DEC_TRUNCATED); continue; }
        const int64_t bm = pos;
        pos += nwords * 8;
        bool failed = false;
        for (int64_t i = 0; i < nvals && !failed; i++) {
            uint64_t val = 0;
            int shift = 0, nb = 0;
            uint8_t last = 0;
            for (;;) {
                if (pos >= endpos) { report_error(err_key, pos, DEC_TRUNCATED); failed = true; break; }
                const uint8_t byte = region[pos++];
                nb++;
                if (nb > MAXL) { report_error(err_key, pos - 1, DEC_NONCANONICAL); failed = true; break; }
                if (MAXL == 10 && nb == 10 && (byte & 0x7E) != 0) { report_error(err_key, pos - 1, DEC_NONCANONICAL); failed = true; break; }
                val |= (uint64_t)(byte & 0x7F) << shift;
                shift += 7;
                last = byte;
                if ((byte & 0x80) == 0) break;
            }
            if (failed) break;
            if (nb > 1 && (last & 0x7F) == 0) { report_error(err_key, pos - 1, DEC_NONCANONICAL); failed = true; break; }
            if (MAXL == 5 && val > 0xFFFFFFFFull) { report_error(err_key, pos - 1, DEC_NONCANONICAL); failed = true; break; }
            const bool ll = (region[bm + (i >> 3)] >> (i & 7)) & 1;
            sink_put<T, kSink, kMode>(out_codes, out_flags, s + i, (U)val, ll, derived);
        }
        if (!failed && pos != endpos) report_error(err_key, pos, DEC_COUNT_MISMATCH);
    }
}

// index checks of decode_stream (container.py:283-291): flags3 = {first != 0,
// non-monotone, last offset beyond the region}
__global__ void k_validate_index(const int64_t *offsets, int64_t nblocks, int64_t region_len, int *flags3) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t o = (uint64_t)offsets[b];
        if (b == 0 && o != 0) flags3[0] = 1;
        if (b + 1 < nblocks && (int64_t)(uint64_t)offsets[b + 1] < (int64_t)o) flags3[1] = 1;
        if (b + 1 == nblocks && o > (uint64_t)region_len) flags3[2] = 1;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int64_t encode_region_capacity(int64_t n, int64_t bs, int width) {
    const int64_t nblocks = n ? (n + bs - 1) / bs : 0;
    const int64_t maxl = width == 32 ? 5 : 10;
    // bitmap bytes are at most 8 per started group of 64 values in each block
    const int64_t words = nblocks * ((bs + 63) / 64);
    const int64_t words_alt = n / 64 + 2 * nblocks;
    return n * maxl + 8 * (words < words_alt ? words : words_alt) + 16;
}

static int64_t blocks_per_tile(int64_t bs) { return bs <= kEncTileMax ? kEncTileMax / bs : 1; }

size_t encode_workspace_bytes(int64_t n, int64_t bs, int width) {
    const int64_t nblocks = n ? (n + bs - 1) / bs : 0;
    if (bs == kEncTileMax) {
        // specialised single-pass path (tile counters); also covers the generic one
        const int64_t V = kEncTileMax;
        const int64_t ntiles = (n + V - 1) / V;
        const size_t gen = (size_t)(ntiles + 2) * 8 + 256;
        const size_t fast = encode4k_workspace_bytes(n, width);
        return fast > gen ? fast : gen;
    }
    if (bs <= kEncTileMax) {
        const int64_t V = blocks_per_tile(bs) * bs;
        const int64_t ntiles = (n + V - 1) / V;
        return (size_t)(ntiles + 2) * 8 + 256;
    }
    // generic path: sizes + offsets + cub scratch
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const int64_t *)nullptr, (int64_t *)nullptr,
                                  (int)(nblocks > 0 ? nblocks : 1));
    return (size_t)nblocks * 16 + cub_bytes + 512;
}

template <typename T, int kSrc, int kMode, bool kUnsafe>
static int encode_dispatch(const EncodeCfg &cfg, EncArgs<T> a, int smem, int grid, cudaStream_t st) {
    auto kern = k_encode<T, kSrc, kMode, kUnsafe>;
    if (int rc = ensure_dyn_smem<k_encode<T, kSrc, kMode, kUnsafe>>(smem, "encode smem attribute")) return rc;
    kern<<<grid, kThreads, smem, st>>>(a);
    return check_launch("encode");
}

template <typename T, int kSrc, int kMode, bool kUnsafe>
static int gen_dispatch(const EncodeCfg &cfg, const typename W<T>::U *x, const uint8_t *fin,
                        const Consts<T> &k, const Consts<T> *kdev, uint8_t *region, uint64_t *index,
                        void *ws, size_t ws_bytes, unsigned long long *trig, long long *region_len,
                        cudaStream_t st) {
    const int64_t nblocks = (cfg.n + cfg.block_size - 1) / cfg.block_size;
    int64_t *sizes = reinterpret_cast<int64_t *>(ws);
    int64_t *offs = sizes + nblocks;
    uintptr_t tp = ((uintptr_t)(offs + nblocks) + 255) & ~(uintptr_t)255;
    void *tmp = (void *)tp;
    size_t tmp_bytes = ws_bytes - (size_t)(tp - (uintptr_t)ws);
    const int grid = (int)((nblocks * 32 + kThreads - 1) / kThreads < resident_grid()
                               ? (nblocks * 32 + kThreads - 1) / kThreads : resident_grid());
    k_gen_sizes<T, kSrc, kMode, kUnsafe><<<grid, kThreads, 0, st>>>(x, fin, k, kdev, cfg.n, cfg.block_size,
                                                                     0, nblocks, sizes);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, offs, (int)nblocks, st);
    if (e != cudaSuccess) return set_error(e, "encode scan");
    k_gen_emit<T, kSrc, kMode, kUnsafe><<<grid, kThreads, 0, st>>>(
        x, fin, k, kdev, cfg.n, cfg.block_size, 0, nblocks, offs, region, index, cfg.base_offset,
        kSrc == 0 ? trig : nullptr);
    k_region_len<<<1, 1, 0, st>>>(offs, sizes, nblocks, region_len);
    note_launch(2);  // sizes + emit (+ this one below)
    return check_launch("encode (generic)");
}

template <typename T>
int launch_encode(const EncodeCfg &cfg, const void *x, const uint8_t *flags_in, const Consts<T> &k,
                  const Consts<T> *kdev, uint8_t *region, uint64_t *index, void *ws,
                  size_t ws_bytes, unsigned long long *trig, long long *region_len,
                  cudaStream_t st) {
    using U = typename W<T>::U;
    const int width = sizeof(T) * 8;
    if (cfg.block_size < 1) return set_error_msg(-1, "block_size must be >= 1");
    if (ws_bytes < encode_workspace_bytes(cfg.n, cfg.block_size, width))
        return set_error_msg(-2, "encode workspace too small");
    if (cfg.n == 0) {
        cudaError_t e = cudaMemsetAsync(region_len, 0, sizeof(long long), st);
        return e == cudaSuccess ? 0 : set_error(e, "encode empty");
    }
    const U *xp = (const U *)x;
    const bool rel = cfg.mode == MODE_REL;
    if (cfg.block_size > kEncTileMax) {
#define GEN(S, M, UN) gen_dispatch<T, S, M, UN>(cfg, xp, flags_in, k, kdev, region, index, ws, ws_bytes, trig, region_len, st)
        if (cfg.src == 1) return GEN(1, MODE_ABS, false);
        if (rel) return cfg.unsafe ? GEN(0, MODE_REL, true) : GEN(0, MODE_REL, false);
        return cfg.unsafe ? GEN(0, MODE_ABS, true) : GEN(0, MODE_ABS, false);
#undef GEN
    }
    // the specialised REL binary32 encoder divides by w through a hoisted refined
    // reciprocal, exact for w in [2^-100, 2^100]; other (degenerate) bounds take
    // the generic kernel with plain IEEE division
    const bool w_ok = !(cfg.mode == MODE_REL && sizeof(T) == 4) ||
                      ((double)k.b >= 0x1p-100 && (double)k.b <= 0x1p100);
    if (cfg.block_size == kEncTileMax && cfg.src == 0 && w_ok && !force_generic_kernels())
        return launch_encode4k<T>(cfg, x, k, kdev, region, index, ws, trig, region_len, st);
    EncArgs<T> a;
    a.x = xp;
    a.fin = flags_in;
    a.k = k;
    a.kdev = kdev;
    a.region = region;
    a.index = index;
    a.n = cfg.n;
    a.bs = cfg.block_size;
    a.K = blocks_per_tile(cfg.block_size);
    a.V = a.K * cfg.block_size;
    a.ntiles = (cfg.n + a.V - 1) / a.V;
    a.base_offset = cfg.base_offset;
    a.bmb = (int)(((cfg.block_size + 63) / 64) * 8);
    const int maxl = W<T>::kMaxVarint;
    a.stage_bytes = (int)(((a.V * maxl + a.K * a.bmb + 32) + 15) / 16 * 16);
    const int vecw = 16 / (int)sizeof(U);
    a.vec_ok = aligned16(x) && (a.V % vecw == 0) && (cfg.src == 0 || (aligned16(flags_in) && a.V % 4 == 0));
    if (sizeof(U) == 8 && cfg.src == 1 && (a.V % 4 != 0)) a.vec_ok = 0;
    a.tiles = reinterpret_cast<unsigned long long *>(ws);
    a.ticket = reinterpret_cast<unsigned int *>(a.tiles + a.ntiles);
    a.trig = trig;
    a.region_len = region_len;
    cudaError_t e = cudaMemsetAsync(ws, 0, (size_t)(a.ntiles + 1) * 8, st);
    if (e != cudaSuccess) return set_error(e, "encode workspace clear");
    const int smem = a.stage_bytes + (int)(a.K * 4);
    int per_sm = (200 * 1024) / (smem + 2048);
    if (per_sm > 2048 / kThreads) per_sm = 2048 / kThreads;
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > a.ntiles) grid = a.ntiles;
    if (cfg.src == 1) return encode_dispatch<T, 1, MODE_ABS, false>(cfg, a, smem, (int)grid, st);
    if (rel) {
        return cfg.unsafe ? encode_dispatch<T, 0, MODE_REL, true>(cfg, a, smem, (int)grid, st)
                          : encode_dispatch<T, 0, MODE_REL, false>(cfg, a, smem, (int)grid, st);
    }
    return cfg.unsafe ? encode_dispatch<T, 0, MODE_ABS, true>(cfg, a, smem, (int)grid, st)
                      : encode_dispatch<T, 0, MODE_ABS, false>(cfg, a, smem, (int)grid, st);
}
template int launch_encode<float>(const EncodeCfg &, const void *, const uint8_t *, const Consts<float> &,
                                  const Consts<float> *, uint8_t *, uint64_t *, void *, size_t,
                                  unsigned long long *, long long *, cudaStream_t);
template int launch_encode<double>(const EncodeCfg &, const void *, const uint8_t *, const Consts<double> &,
                                   const Consts<double> *, uint8_t *, uint64_t *, void *, size_t,
                                   unsigned long long *, long long *, cudaStream_t);

template <typename T, int kSink, int kMode>
static int decode_dispatch(const DecodeCfg &d, const uint8_t *region, const int64_t *offsets, T derived,
                           void *oc, uint8_t *of, unsigned long long *err, cudaStream_t st) {
    const int64_t nblk = d.b1 - d.b0;
    if (nblk <= 0) return 0;
    // the 4096-value kernel stores 128-bit value vectors (and 32-bit flag quads)
    const bool vec_ok = aligned16(oc) && (kSink == 1 || ((uintptr_t)of & 3u) == 0);
    if (d.block_size == kEncTileMax && vec_ok && !force_generic_kernels())
        return launch_decode4k<T>(d, region, offsets, derived, oc, of, err, st);
    if (d.block_size >= 64 && d.block_size <= kEncTileMax) {
        const int maxl = W<T>::kMaxVarint;
        const int bmb = (int)(((d.block_size + 63) / 64) * 8);
        const int buf_bytes = (int)((bmb + d.block_size * maxl + 1 + 16 + 15) / 16 * 16);
        const int smem = buf_bytes + (int)(d.block_size * 2);
        auto kern = k_decode_par<T, kSink, kMode>;
        if (int rc = ensure_dyn_smem<k_decode_par<T, kSink, kMode>>(smem, "decode smem attribute")) return rc;
        int per_sm = (200 * 1024) / (smem + 2048);
        if (per_sm > 2048 / kThreads) per_sm = 2048 / kThreads;
        if (per_sm < 1) per_sm = 1;
        int64_t grid = (int64_t)sm_count() * per_sm;
        if (grid > nblk) grid = nblk;
        kern<<<(int)grid, kThreads, smem, st>>>(d, region, offsets, derived, oc, of, err, buf_bytes);
    } else {
        int64_t grid = (nblk + kThreads - 1) / kThreads;
        if (grid > resident_grid()) grid = resident_grid();
        k_decode_seq<T, kSink, kMode><<<(int)grid, kThreads, 0, st>>>(d, region, offsets, derived, oc, of, err);
    }
    return check_launch("decode");
}

template <typename T>
int launch_decode(const DecodeCfg &d, const uint8_t *region, const int64_t *offsets, T derived,
                  void *out_codes, uint8_t *out_flags, unsigned long long *err_key, cudaStream_t st) {
    if (d.sink == 0) return decode_dispatch<T, 0, MODE_ABS>(d, region, offsets, derived, out_codes, out_flags, err_key, st);
    if (d.mode == MODE_REL) return decode_dispatch<T, 1, MODE_REL>(d, region, offsets, derived, out_codes, out_flags, err_key, st);
    return decode_dispatch<T, 1, MODE_ABS>(d, region, offsets, derived, out_codes, out_flags, err_key, st);
}
template int launch_decode<float>(const DecodeCfg &, const uint8_t *, const int64_t *, float, void *, uint8_t *,
                                  unsigned long long *, cudaStream_t);
template int launch_decode<double>(const DecodeCfg &, const uint8_t *, const int64_t *, double, void *, uint8_t *,
                                   unsigned long long *, cudaStream_t);

int launch_validate_index(const int64_t *offsets, int64_t nblocks, int64_t region_len, int *flags3,
                          cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(flags3, 0, 3 * sizeof(int), st);
    if (e != cudaSuccess) return set_error(e, "validate memset");
    if (nblocks > 0) {
        int64_t grid = (nblocks + kThreads - 1) / kThreads;
        if (grid > resident_grid()) grid = resident_grid();
        k_validate_index<<<(int)grid, kThreads, 0, st>>>(offsets, nblocks, region_len, flags3);
    }
    return check_launch("validate_index");
}

template <typename U>
int launch_block_sizes(const U *codes, int64_t count, int64_t bs, int64_t b0, int64_t b1,
                       int64_t *sizes, cudaStream_t st) {
    using T = typename std::conditional<sizeof(U) == 4, float, double>::type;
    if (b1 <= b0) return 0;
    const int64_t grid = ((b1 - b0) * 32 + kThreads - 1) / kThreads;
    Consts<T> k{};
    k_gen_sizes<T, 1, MODE_ABS, false><<<(int)(grid < resident_grid() ? grid : resident_grid()), kThreads, 0, st>>>(
        codes, nullptr, k, nullptr, count, bs, b0, b1, sizes);
    return check_launch("block_sizes");
}
template int launch_block_sizes<uint32_t>(const uint32_t *, int64_t, int64_t, int64_t, int64_t, int64_t *, cudaStream_t);
template int launch_block_sizes<uint64_t>(const uint64_t *, int64_t, int64_t, int64_t, int64_t, int64_t *, cudaStream_t);

template <typename U>
int launch_emit_blocks(const U *codes, const uint8_t *flags, int64_t count, int64_t bs, int64_t b0,
                       int64_t b1, const int64_t *offsets, uint8_t *out, cudaStream_t st) {
    using T = typename std::conditional<sizeof(U) == 4, float, double>::type;
    if (b1 <= b0) return 0;
    const int64_t grid = ((b1 - b0) * 32 + kThreads - 1) / kThreads;
    Consts<T> k{};
    k_gen_emit<T, 1, MODE_ABS, false><<<(int)(grid < resident_grid() ? grid : resident_grid()), kThreads, 0, st>>>(
        codes, flags, k, nullptr, count, bs, b0, b1, offsets, out, nullptr, 0, nullptr);
    return check_launch("emit_blocks");
}
template int launch_emit_blocks<uint32_t>(const uint32_t *, const uint8_t *, int64_t, int64_t, int64_t, int64_t,
                                          const int64_t *, uint8_t *, cudaStream_t);
template int launch_emit_blocks<uint64_t>(const uint64_t *, const uint8_t *, int64_t, int64_t, int64_t, int64_t,
                                          const int64_t *, uint8_t *, cudaStream_t);

}  // namespace gebq
