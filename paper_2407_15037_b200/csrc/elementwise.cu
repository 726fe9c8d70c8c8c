// elementwise.cu -- CodedArray-level quantize / reconstruct, the NOA range
// pass, exhaustive / sampled sweeps and the device corpus generators, sm_100a.
//
// Memory-bound streaming kernels: every warp moves 512 contiguous values per
// step, each lane four consecutive values per row (one 128-bit LDG for f32,
// two for f64), four rows per lane, so every load / store instruction of a
// warp covers one contiguous 512 B (f32) or 1 KB (f64) span and the lossless
// flags go out as one coalesced 128 B store per row.  Grids are sized to the
// resident-CTA capacity of the 148 SMs and grid-stride over 4096-value tiles.
#include "gebq_common.cuh"
#include "gebq_internal.cuh"

namespace gebq {

// ---------------------------------------------------------------------------
// vector helpers: 4 consecutive values of width U
// ---------------------------------------------------------------------------
template <typename U> struct Vec4;
template <> struct Vec4<uint32_t> {
    __device__ __forceinline__ static void load(const uint32_t *p, uint32_t v[4]) {
        uint4 a = __ldcs(reinterpret_cast<const uint4 *>(p));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
    __device__ __forceinline__ static void store(uint32_t *p, const uint32_t v[4]) {
        __stcs(reinterpret_cast<uint4 *>(p), make_uint4(v[0], v[1], v[2], v[3]));
    }
};
template <> struct Vec4<uint64_t> {
    __device__ __forceinline__ static void load(const uint64_t *p, uint64_t v[4]) {
        ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2 *>(p));
        ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    __device__ __forceinline__ static void store(uint64_t *p, const uint64_t v[4]) {
        __stcs(reinterpret_cast<ulonglong2 *>(p), make_ulonglong2(v[0], v[1]));
        __stcs(reinterpret_cast<ulonglong2 *>(p) + 1, make_ulonglong2(v[2], v[3]));
    }
};

__device__ __forceinline__ void flush_trig(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                           unsigned long long *trig) {
    __shared__ unsigned long long s_trig[4];
    if (threadIdx.x < 4) s_trig[threadIdx.x] = 0;
    __syncthreads();
    t0 = __reduce_add_sync(0xFFFFFFFFu, t0);
    t1 = __reduce_add_sync(0xFFFFFFFFu, t1);
    t2 = __reduce_add_sync(0xFFFFFFFFu, t2);
    t3 = __reduce_add_sync(0xFFFFFFFFu, t3);
    if ((threadIdx.x & 31) == 0) {
        if (t0) atomicAdd(&s_trig[0], (unsigned long long)t0);
        if (t1) atomicAdd(&s_trig[1], (unsigned long long)t1);
        if (t2) atomicAdd(&s_trig[2], (unsigned long long)t2);
        if (t3) atomicAdd(&s_trig[3], (unsigned long long)t3);
    }
    __syncthreads();
    if (threadIdx.x < 4 && s_trig[threadIdx.x]) atomicAdd(&trig[threadIdx.x], s_trig[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// quantize: (bits) -> (codes, lossless flags, 4 trigger counters)
// replaces quantize_{abs,rel}{32,64} (_kernels.py:86-285)
// ---------------------------------------------------------------------------
template <typename T, int kMode, bool kUnsafe>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 5 : 3) k_quantize(const typename W<T>::U *__restrict__ x,
                                                       typename W<T>::U *__restrict__ codes,
                                                       uint8_t *__restrict__ flags, int64_t n,
                                                       Consts<T> k, const Consts<T> *kdev,
                                                       unsigned long long *trig, int vec_ok) {
    using U = typename W<T>::U;
    if (kdev) k = *kdev;  // NOA: constants derived on device from the global range
    RelFast<T> f{};
    RelExact ef{};
    if constexpr (kMode == MODE_REL) {
        f = make_rel_fast<T>(k);
        if constexpr (sizeof(T) == 4) ef = make_rel_exact(k);
    }
    // binary32 REL: the exact-division quantizer of the stream encoder whenever w
    // is in its range (uniform); the filtered one otherwise.  The trigger comes
    // back as a packed 5-bit counter increment (trig_inc; 0 = none).
    auto qv = [&](typename W<T>::U xb, typename W<T>::U &c) -> uint32_t {
        if constexpr (kMode == MODE_REL) {
            if constexpr (sizeof(T) == 4) {
                if (ef.wdiv) return (uint32_t)quantize_rel_exact32<kUnsafe, true>(xb, k, ef, c);
            }
            return trig_inc(quantize_bf<T, kMode, kUnsafe>(xb, k, f, c));
        } else {
            return (uint32_t)quantize_abs_bf<T, kUnsafe, true>(xb, k, c);
        }
    };
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    auto drain = [&](uint32_t tc) {   // at most 16 increments per 5-bit field
        c0 += tc & 31u; c1 += (tc >> 5) & 31u; c2 += (tc >> 10) & 31u; c3 += (tc >> 15) & 31u;
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = vec_ok ? n / kTile : 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * kTile + warp * (kTile / kWarps) + 4 * lane;
        U v[kRows][4];
#pragma unroll
        for (int r = 0; r < kRows; r++) Vec4<U>::load(x + base + 128 * r, v[r]);
        uint32_t tc = 0;
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            uint32_t fl = 0;
#pragma unroll
            for (int s = 0; s < 4; s++) {
                U c;
                const uint32_t inc = qv(v[r][s], c);
                v[r][s] = c;
                fl |= (uint32_t)(inc != 0u) << (8 * s);
                tc += inc;
            }
            Vec4<U>::store(codes + base + 128 * r, v[r]);
            __stcs(reinterpret_cast<uint32_t *>(flags + base + 128 * r), fl);
        }
        drain(tc);
    }
    // scalar tail (or everything when the pointers are not 16 B aligned)
    const int64_t start = ntiles * kTile;
    for (int64_t i = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        U c;
        const uint32_t inc = qv(x[i], c);
        codes[i] = c;
        flags[i] = inc != 0u;
        drain(inc);
    }
    flush_trig(c0, c1, c2, c3, trig);
}

// ---------------------------------------------------------------------------
// reconstruct: (codes, flags) -> value bits; replaces reconstruct_* (_kernels.py:293-354)
// ---------------------------------------------------------------------------
template <typename T, int kMode>
__global__ void __launch_bounds__(kThreads) k_reconstruct(const typename W<T>::U *__restrict__ codes,
                                                          const uint8_t *__restrict__ flags,
                                                          typename W<T>::U *__restrict__ out,
                                                          int64_t n, T derived, int vec_ok) {
    using U = typename W<T>::U;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // binary32: the decode hot loop's reconstruct (exact fast ranges, the plain
    // restatement reconstruct_one outside them)
    const RelDec32 rd = make_rel_dec32(sizeof(T) == 4 && kMode == MODE_REL ? (float)derived : 0.0f);
    auto rec = [&](U c, uint32_t fl) -> U {
        if constexpr (sizeof(T) == 4) return reconstruct32_fast<kMode>(c, fl != 0u, derived, rd);
        else return reconstruct_one<T, kMode>(c, fl != 0u, derived);
    };
    const int64_t ntiles = vec_ok ? n / kTile : 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * kTile + warp * (kTile / kWarps) + 4 * lane;
        U v[kRows][4];
        uint32_t fl[kRows];
#pragma unroll
        for (int r = 0; r < kRows; r++) {
            Vec4<U>::load(codes + base + 128 * r, v[r]);
            fl[r] = __ldcs(reinterpret_cast<const uint32_t *>(flags + base + 128 * r));
        }
#pragma unroll
        for (int r = 0; r < kRows; r++) {
#pragma unroll
            for (int s = 0; s < 4; s++)
                v[r][s] = rec(v[r][s], (fl[r] >> (8 * s)) & 0xFFu);
            Vec4<U>::store(out + base + 128 * r, v[r]);
        }
    }
    const int64_t start = ntiles * kTile;
    for (int64_t i = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rec(codes[i], flags[i]);
}

// ---------------------------------------------------------------------------
// NOA range pass (compute_noa_range, quantizers.py:337-351).
// Finite values map to order-preserving integer keys (total order, -0 < +0);
// keys2[0] = max key, keys2[1] = max of the complemented key (= min), both as
// signed int64 so one MAX allreduce combines shards.  0 / INT64_MIN = none.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t order_key(uint32_t b) { return (b & 0x80000000u) ? ~b : (b | 0x80000000u); }
__device__ __forceinline__ uint64_t order_key(uint64_t b) {
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_noa_minmax(const typename W<T>::U *__restrict__ x,
                                                         int64_t n, long long *keys2, int vec_ok) {
    using X = W<T>;
    using U = typename X::U;
    U kmax = 0, kmin_c = 0;  // 0 = no finite value seen
    auto acc = [&](U b) {
        if (((b >> X::kMantBits) & X::kExpAll) == X::kExpAll) return;  // NaN / Inf skipped
        U key = order_key(b);
        kmax = key > kmax ? key : kmax;
        kmin_c = (U)~key > kmin_c ? (U)~key : kmin_c;
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = vec_ok ? n / kTile : 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * kTile + warp * (kTile / kWarps) + 4 * lane;
        U v[kRows][4];
#pragma unroll
        for (int r = 0; r < kRows; r++) Vec4<U>::load(x + base + 128 * r, v[r]);
#pragma unroll
        for (int r = 0; r < kRows; r++)
#pragma unroll
            for (int s = 0; s < 4; s++) acc(v[r][s]);
    }
    for (int64_t i = ntiles * kTile + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc(x[i]);
    long long a, b;
    if constexpr (sizeof(T) == 4) {
        a = __reduce_max_sync(0xFFFFFFFFu, (unsigned)kmax);
        b = __reduce_max_sync(0xFFFFFFFFu, (unsigned)kmin_c);
    } else {
        for (int off = 16; off; off >>= 1) {
            U o1 = __shfl_xor_sync(0xFFFFFFFFu, kmax, off);
            U o2 = __shfl_xor_sync(0xFFFFFFFFu, kmin_c, off);
            kmax = o1 > kmax ? o1 : kmax;
            kmin_c = o2 > kmin_c ? o2 : kmin_c;
        }
        a = (long long)(kmax ^ 0x8000000000000000ull);
        b = (long long)(kmin_c ^ 0x8000000000000000ull);
    }
    if (lane == 0) {
        atomicMax(&keys2[0], a);
        atomicMax(&keys2[1], b);
    }
}

// R = max - min in the value width (+0 when no finite values), then the NOA
// constants eb_eff = f(eb)*R, eb2 = eb_eff+eb_eff, inv_eb2 = 1/eb2
// (quantizers.py:106-116).  range_out = R widened to f64 (the header's range_bits).
template <typename T>
__global__ void k_noa_derive(const long long *keys2, double eb, Consts<T> *kout, double *range_out) {
    using X = W<T>;
    using U = typename X::U;
    U kmax, kmin_c;
    if constexpr (sizeof(T) == 4) {
        kmax = (U)keys2[0];
        kmin_c = (U)keys2[1];
    } else {
        kmax = (U)keys2[0] ^ 0x8000000000000000ull;
        kmin_c = (U)keys2[1] ^ 0x8000000000000000ull;
    }
    T R = T(0);
    if (kmax != 0) {
        const U top = (U)1 << (X::kBits - 1);
        U kmin = ~kmin_c;
        U bmax = (kmax & top) ? (kmax & ~top) : ~kmax;
        U bmin = (kmin & top) ? (kmin & ~top) : ~kmin;
        R = X::sub(X::from_bits(bmax), X::from_bits(bmin));
    }
    T eps_w;
    if constexpr (sizeof(T) == 4) eps_w = __double2float_rn(eb); else eps_w = eb;
    T eb_eff = X::mul(eps_w, R);
    T eb2 = X::add(eb_eff, eb_eff);
    Consts<T> k;
    k.a = eb_eff;
    k.b = eb2;
    k.c = X::div(T(1), eb2);
    k.thr = (T)(X::kMaxBin - 1);
    *kout = k;
    *range_out = (double)R;
}

// ---------------------------------------------------------------------------
// sweeps: quantize -> reconstruct -> check, tallied per value class
// (sweep_*_on, _kernels.py:717-896).  Patterns come from the index (range),
// an explicit array, or splitmix64 -- no HBM traffic for the first and last.
// Counters: 15 x 16-bit lanes packed in 4 u64 registers (host bounds the
// per-thread pattern count below 2^16).
// ---------------------------------------------------------------------------
template <typename T, int kMode, bool kUnsafe>
__device__ __forceinline__ int sweep_outcome(typename W<T>::U xb, const Consts<T> &k,
                                             const RelFast<T> &f) {
    using X = W<T>;
    using U = typename X::U;
    T xf = X::from_bits(xb);
    if constexpr (kMode == MODE_ABS) {
        if (xf != xf) return 1;
        T t = X::mul(xf, k.c);
        if (!(X::fabs_(t) < k.thr)) return 1;
        T bf;
        int64_t b = round_bin(t, bf);
        if (b >= X::kMaxBin || b <= -X::kMaxBin) return 1;
        T recon = X::mul(bf, k.b);
        T err = X::fabs_(X::sub(xf, recon));
        if (!kUnsafe && !(err <= k.a)) return 1;
        return err <= k.a ? 0 : 2;
    } else {
        // lossless decision from the production (filtered) quantizer; the
        // verdict recomputes the exact IEEE predicate on the reconstruction,
        // so the tallies check the filter against the reference exhaustively
        U code;
        if (quantize_rel_bf<T, kUnsafe>(xb, k, f, code) != TRIG_NONE) return 1;
        U rb = reconstruct_one<T, MODE_REL>(code, false, k.b);
        T q = X::div(X::fabs_(X::from_bits(rb)), X::fabs_(xf));
        return (q <= k.a && X::mul(q, k.a) >= T(1)) ? 0 : 2;
    }
}

struct Tally16 {
    uint64_t r[4] = {0, 0, 0, 0};
    __device__ __forceinline__ void add(int key) {
        uint64_t inc = 1ull << (16 * (key & 3));
        int w = key >> 2;
        r[0] += w == 0 ? inc : 0;
        r[1] += w == 1 ? inc : 0;
        r[2] += w == 2 ? inc : 0;
        r[3] += w == 3 ? inc : 0;
    }
    __device__ __forceinline__ void flush(unsigned long long *tally15) {
#pragma unroll
        for (int key = 0; key < 15; key++) {
            uint32_t v = (uint32_t)((r[key >> 2] >> (16 * (key & 3))) & 0xFFFF);
            v = __reduce_add_sync(0xFFFFFFFFu, v);
            if ((threadIdx.x & 31) == 0 && v) atomicAdd(&tally15[key], (unsigned long long)v);
        }
    }
};

// kSource: 0 = index range (bits = start + i mod 2^32), 1 = explicit array,
// 2 = splitmix64(seed, start + i + 1) (low 32 bits for f32)
template <typename T, int kMode, bool kUnsafe, int kSource>
__global__ void __launch_bounds__(kThreads) k_sweep(uint64_t start, int64_t count,
                                                    const typename W<T>::U *__restrict__ bits,
                                                    uint64_t seed, Consts<T> k,
                                                    unsigned long long *tally15,
                                                    unsigned long long *first_viol,
                                                    int64_t idx_base) {
    using U = typename W<T>::U;
    RelFast<T> f{};
    if constexpr (kMode == MODE_REL) f = make_rel_fast<T>(k);
    Tally16 tl;
    uint64_t first = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        U xb;
        if constexpr (kSource == 0) xb = (U)(start + (uint64_t)i);
        else if constexpr (kSource == 1) xb = bits[i];
        else xb = (U)splitmix64_at(seed, start + (uint64_t)i + 1);
        int o = sweep_outcome<T, kMode, kUnsafe>(xb, k, f);
        tl.add(value_class<T>(xb) * 3 + o);
        if (o == 2 && (uint64_t)i < first) first = (uint64_t)i;
    }
    tl.flush(tally15);
    if (first != ~0ull) atomicMin(first_viol, (unsigned long long)(idx_base + (int64_t)first));
}

// ---------------------------------------------------------------------------
// device corpus generators (splitmix64_fill, _kernels.py:671-685; C2 recipe)
// ---------------------------------------------------------------------------
__global__ void k_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = splitmix64_at(seed, (uint64_t)(start_index + i + 1));
}

// mixed-class f32 patterns from one splitmix64 word each
__global__ void k_gen_mixed_f32(uint32_t *out, int64_t n, uint64_t seed, int64_t start_index) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t w = splitmix64_at(seed, (uint64_t)(start_index + i + 1));
        uint32_t sel = (uint32_t)(w >> 56);
        uint32_t sign = (uint32_t)((w >> 55) & 1) << 31;
        uint32_t lo = (uint32_t)w;
        uint32_t mant = lo & 0x7FFFFFu;
        uint32_t b;
        if (sel < 4) b = sign | 0x7F800000u | (mant | 1u);
        else if (sel < 8) b = sign | 0x7F800000u;
        else if (sel < 12) b = sign | mant;
        else if (sel < 16) b = sign | (0x7F7FFF00u + (lo & 0xFFu));
        else b = sign | ((107u + (uint32_t)((w >> 32) % 41u)) << 23) | mant;
        out[i] = b;
    }
}

// C3 / C5-smooth field (workloads.smooth_field_cb): counter-based, so every
// shard of every world size and the host recipe produce identical bits.
//   g = start + i;  k = g % side, j = (g / side) % side, ii = (g / side^2) % side
//   w = splitmix64(seed, g + 1); s = sum of w's four 16-bit fields (exact)
//   v = ((5 * A[ii]) * B[j]) * C[k] + (s - 131070) * nz   (f64, one rounding each)
// planted (NOA range test): g = 0 NaN, 1 +Inf, 2 -7, total - 1 +7.
template <typename T>
__global__ void k_gen_smooth(T *out, int64_t n, int64_t side, const double *__restrict__ tab,
                             uint64_t seed, int64_t start_index, int plant, int64_t total, double nz) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t g = start_index + i;
        int64_t k = g % side, j = (g / side) % side, ii = (g / side / side) % side;
        uint64_t w = splitmix64_at(seed, (uint64_t)g + 1);
        int64_t s = (int64_t)(w & 0xFFFF) + (int64_t)((w >> 16) & 0xFFFF) + (int64_t)((w >> 32) & 0xFFFF) +
                    (int64_t)(w >> 48);
        double noise = __dmul_rn((double)(s - 131070), nz);
        double v = __dmul_rn(__dmul_rn(__dmul_rn(5.0, tab[ii]), tab[side + j]), tab[2 * side + k]);
        v = __dadd_rn(v, noise);
        if (plant) {
            if (g == 0) v = __longlong_as_double(0x7FF8000000000000ll);
            else if (g == 1) v = __longlong_as_double(0x7FF0000000000000ll);
            else if (g == 2) v = -7.0;
            else if (g == total - 1) v = 7.0;
        }
        if constexpr (sizeof(T) == 4) out[i] = __double2float_rn(v);
        else out[i] = v;
    }
}

// ---------------------------------------------------------------------------
// host launchers (called from capi.cu)
// ---------------------------------------------------------------------------
template <typename T>
int launch_quantize(int mode, const void *x, void *codes, uint8_t *flags, int64_t n,
                    const Consts<T> &k, const Consts<T> *kdev, int unsafe,
                    unsigned long long *trig, cudaStream_t st) {
    using U = typename W<T>::U;
    int vec = aligned16(x) && aligned16(codes) && aligned16(flags);
    auto *xp = (const U *)x;
    auto *cp = (U *)codes;
    if (mode == MODE_REL) {
        if (unsafe) k_quantize<T, MODE_REL, true><<<grid_per_sm(n, 16), kThreads, 0, st>>>(xp, cp, flags, n, k, kdev, trig, vec);
        else k_quantize<T, MODE_REL, false><<<grid_per_sm(n, 16), kThreads, 0, st>>>(xp, cp, flags, n, k, kdev, trig, vec);
    } else {
        if (unsafe) k_quantize<T, MODE_ABS, true><<<grid_per_sm(n, 16), kThreads, 0, st>>>(xp, cp, flags, n, k, kdev, trig, vec);
        else k_quantize<T, MODE_ABS, false><<<grid_per_sm(n, 16), kThreads, 0, st>>>(xp, cp, flags, n, k, kdev, trig, vec);
    }
    return check_launch("quantize");
}
template int launch_quantize<float>(int, const void *, void *, uint8_t *, int64_t, const Consts<float> &,
                                    const Consts<float> *, int, unsigned long long *, cudaStream_t);
template int launch_quantize<double>(int, const void *, void *, uint8_t *, int64_t, const Consts<double> &,
                                     const Consts<double> *, int, unsigned long long *, cudaStream_t);

template <typename T>
int launch_reconstruct(int mode, const void *codes, const uint8_t *flags, void *out, int64_t n,
                       T derived, cudaStream_t st) {
    using U = typename W<T>::U;
    int vec = aligned16(codes) && aligned16(out) && aligned16(flags);
    if (mode == MODE_REL)
        k_reconstruct<T, MODE_REL><<<grid_tiles(n), kThreads, 0, st>>>((const U *)codes, flags, (U *)out, n, derived, vec);
    else
        k_reconstruct<T, MODE_ABS><<<grid_tiles(n), kThreads, 0, st>>>((const U *)codes, flags, (U *)out, n, derived, vec);
    return check_launch("reconstruct");
}
template int launch_reconstruct<float>(int, const void *, const uint8_t *, void *, int64_t, float, cudaStream_t);
template int launch_reconstruct<double>(int, const void *, const uint8_t *, void *, int64_t, double, cudaStream_t);

// key "none" (no finite value seen): 0 for the f32 keys (max taken as unsigned
// 32-bit), INT64_MIN for the signed-int64 view of the f64 keys.  Written by a
// kernel, not a pageable host copy, so the range pass stays graph-capturable.
__global__ void k_noa_init(long long *keys2, long long none) {
    if (threadIdx.x < 2) keys2[threadIdx.x] = none;
}

template <typename T>
int launch_noa_minmax(const void *x, int64_t n, long long *keys2, cudaStream_t st) {
    using U = typename W<T>::U;
    k_noa_init<<<1, 32, 0, st>>>(keys2, sizeof(T) == 8 ? (long long)0x8000000000000000ull : 0ll);
    int rc = check_launch("noa_init");
    if (rc) return rc;
    k_noa_minmax<T><<<grid_per_sm(n, 8), kThreads, 0, st>>>((const U *)x, n, keys2, aligned16(x));
    return check_launch("noa_minmax");
}
template int launch_noa_minmax<float>(const void *, int64_t, long long *, cudaStream_t);
template int launch_noa_minmax<double>(const void *, int64_t, long long *, cudaStream_t);

template <typename T>
int launch_noa_derive(const long long *keys2, double eb, Consts<T> *kout, double *range_out,
                      cudaStream_t st) {
    k_noa_derive<T><<<1, 1, 0, st>>>(keys2, eb, kout, range_out);
    return check_launch("noa_derive");
}
template int launch_noa_derive<float>(const long long *, double, Consts<float> *, double *, cudaStream_t);
template int launch_noa_derive<double>(const long long *, double, Consts<double> *, double *, cudaStream_t);

template <typename T, int kMode, bool kUnsafe>
static void sweep_dispatch(int source, int grid, uint64_t start, int64_t count, const void *bits,
                           uint64_t seed, const Consts<T> &k, unsigned long long *tally15,
                           unsigned long long *first, int64_t idx_base, cudaStream_t st) {
    using U = typename W<T>::U;
    if (source == 0)
        k_sweep<T, kMode, kUnsafe, 0><<<grid, kThreads, 0, st>>>(start, count, (const U *)bits, seed, k, tally15, first, idx_base);
    else if (source == 1)
        k_sweep<T, kMode, kUnsafe, 1><<<grid, kThreads, 0, st>>>(start, count, (const U *)bits, seed, k, tally15, first, idx_base);
    else
        k_sweep<T, kMode, kUnsafe, 2><<<grid, kThreads, 0, st>>>(start, count, (const U *)bits, seed, k, tally15, first, idx_base);
}

// tally15 / first_viol are device buffers (zero / all-ones on entry); the
// first-violation slot receives the sequence index of the first failing pattern.
template <typename T>
int launch_sweep(int mode, int unsafe, int source, uint64_t start, int64_t count, const void *bits,
                 uint64_t seed, const Consts<T> &k, unsigned long long *tally15,
                 unsigned long long *first, cudaStream_t st) {
    // Split so each thread handles < 2^16 patterns per launch (16-bit packed counters).
    const int grid = resident_grid();
    const int64_t per_launch = (int64_t)grid * kThreads * 60000;
    for (int64_t off = 0; off < count; off += per_launch) {
        int64_t c = count - off < per_launch ? count - off : per_launch;
        const void *b = source == 1 ? (const void *)((const char *)bits + off * sizeof(typename W<T>::U)) : bits;
        uint64_t s = start + (uint64_t)off;
        if (mode == MODE_REL) {
            if (unsafe) sweep_dispatch<T, MODE_REL, true>(source, grid, s, c, b, seed, k, tally15, first, off, st);
            else sweep_dispatch<T, MODE_REL, false>(source, grid, s, c, b, seed, k, tally15, first, off, st);
        } else {
            if (unsafe) sweep_dispatch<T, MODE_ABS, true>(source, grid, s, c, b, seed, k, tally15, first, off, st);
            else sweep_dispatch<T, MODE_ABS, false>(source, grid, s, c, b, seed, k, tally15, first, off, st);
        }
        int rc = check_launch("sweep");
        if (rc) return rc;
    }
    return 0;
}
template int launch_sweep<float>(int, int, int, uint64_t, int64_t, const void *, uint64_t, const Consts<float> &,
                                 unsigned long long *, unsigned long long *, cudaStream_t);
template int launch_sweep<double>(int, int, int, uint64_t, int64_t, const void *, uint64_t, const Consts<double> &,
                                  unsigned long long *, unsigned long long *, cudaStream_t);

int64_t sweep_per_launch() { return (int64_t)resident_grid() * kThreads * 60000; }

int launch_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index, cudaStream_t st) {
    k_splitmix64_fill<<<grid_for(n), kThreads, 0, st>>>(out, n, seed, start_index);
    return check_launch("splitmix64_fill");
}
int launch_gen_smooth(int width, void *out, int64_t n, int64_t side, const double *tab, uint64_t seed,
                      int64_t start_index, int plant, int64_t total, double nz, cudaStream_t st) {
    if (n <= 0) return 0;
    if (width == 32)
        k_gen_smooth<float><<<grid_for(n), kThreads, 0, st>>>((float *)out, n, side, tab, seed, start_index, plant,
                                                               total, nz);
    else
        k_gen_smooth<double><<<grid_for(n), kThreads, 0, st>>>((double *)out, n, side, tab, seed, start_index,
                                                                plant, total, nz);
    return check_launch("gen_smooth");
}
int launch_gen_mixed_f32(uint32_t *out, int64_t n, uint64_t seed, int64_t start_index, cudaStream_t st) {
    k_gen_mixed_f32<<<grid_for(n), kThreads, 0, st>>>(out, n, seed, start_index);
    return check_launch("gen_mixed_f32");
}

// ---------------------------------------------------------------------------
// library-log REL variant (quantize_rel32_lib / reconstruct_rel32_lib,
// _kernels.py:356-431): the same guard chain and double-check, but log2 / 2^p
// from the binary64 math library instead of the bit-level approximations.
// Non-conforming by design (the reference says so): CUDA's log2/exp2 are not
// the host libm, so codes may differ from the CPU in rare last-ulp cases; the
// double-check still guarantees the bound.  Benchmark comparisons only.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_quantize_rel32_lib(const uint32_t *__restrict__ x, uint32_t *codes,
                                                                 uint8_t *flags, int64_t n, float op_eps, float w,
                                                                 float thr, int unsafe, unsigned long long *trig) {
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t xb = x[i];
        const float xf = __uint_as_float(xb);
        int tr = TRIG_NONE;
        uint32_t code = xb;
        const uint32_t ab = xb & 0x7FFFFFFFu;
        const uint32_t aexpo = ab >> 23;
        if (xf != xf) tr = TRIG_NAN;
        else if (aexpo == 0xFFu) tr = TRIG_INF;
        else if (aexpo == 0) tr = TRIG_GUARD;
        else {
            const float l = __double2float_rn(log2((double)fabsf(xf)));
            const float t = __fdiv_rn(l, w);
            if (!(fabsf(t) < thr)) tr = TRIG_GUARD;
            else {
                float kf;
                const int32_t kb = round_bin(t, kf);
                if (kb >= (1 << 30) || kb <= -(1 << 30)) tr = TRIG_GUARD;
                else {
                    const float p = __fmul_rn(kf, w);
                    if (!(p > -127.0f && p < 128.0f)) tr = TRIG_GUARD;
                    else {
                        if (!unsafe) {
                            const float recon = __double2float_rn(exp2((double)p));
                            const float q = __fdiv_rn(recon, fabsf(xf));
                            if (!(q <= op_eps && __fmul_rn(q, op_eps) >= 1.0f)) tr = TRIG_DCHECK;
                        }
                        if (tr == TRIG_NONE) code = (zigzag_w(kb) << 1) | (xb >> 31);
                    }
                }
            }
        }
        codes[i] = code;
        flags[i] = tr != TRIG_NONE;
        c0 += tr == TRIG_NAN; c1 += tr == TRIG_INF; c2 += tr == TRIG_GUARD; c3 += tr == TRIG_DCHECK;
    }
    flush_trig(c0, c1, c2, c3, trig);
}

__global__ void __launch_bounds__(kThreads) k_reconstruct_rel32_lib(const uint32_t *__restrict__ codes,
                                                                    const uint8_t *__restrict__ flags, uint32_t *out,
                                                                    int64_t n, float w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = codes[i];
        if (flags[i]) { out[i] = c; continue; }
        const int32_t kb = unzigzag_w(c >> 1);
        const float p = __fmul_rn(__int2float_rn(kb), w);
        const float mag = __double2float_rn(exp2((double)p));
        out[i] = __float_as_uint(mag) | (c << 31);
    }
}

int launch_rel32_lib_quantize(const uint32_t *x, uint32_t *codes, uint8_t *flags, int64_t n, float op_eps, float w,
                              float thr, int unsafe, unsigned long long *trig, cudaStream_t st) {
    if (n <= 0) return 0;
    k_quantize_rel32_lib<<<grid_for(n), kThreads, 0, st>>>(x, codes, flags, n, op_eps, w, thr, unsafe, trig);
    return check_launch("quantize_rel32_lib");
}
int launch_rel32_lib_reconstruct(const uint32_t *codes, const uint8_t *flags, uint32_t *out, int64_t n, float w,
                                 cudaStream_t st) {
    if (n <= 0) return 0;
    k_reconstruct_rel32_lib<<<grid_for(n), kThreads, 0, st>>>(codes, flags, out, n, w);
    return check_launch("reconstruct_rel32_lib");
}

// ---------------------------------------------------------------------------
// verify (verify.py:88-153): the bound predicates of the compressor's
// double-check, evaluated on (original, reconstructed) pairs on the device.
//   out5[0] += violations       (finite original, bits differ, predicate false)
//   out5[1] += special mismatches (NaN/Inf original, bits differ)
//   out5[2]  = min index of a violation (caller sets UINT64_MAX)
//   out5[3]  = max over inexact finite elements of |o - r| (ABS/NOA) or
//              |q - 1| (REL, q = |r| / |o|) as binary64 bits (NaN -> +inf)
//   mask (optional): 1 = violation, 2 = special mismatch, 0 otherwise
// ---------------------------------------------------------------------------
template <typename T, bool kRel>
__global__ void __launch_bounds__(kThreads) k_verify(const typename W<T>::U *__restrict__ o,
                                                     const typename W<T>::U *__restrict__ r, int64_t n,
                                                     T bound, unsigned long long *out5, uint8_t *mask) {
    using X = W<T>;
    using U = typename X::U;
    unsigned long long viol = 0, spec = 0, first = ~0ull, maxe = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const U ob = o[i], rb = r[i];
        const bool eq = ob == rb;
        const bool special = (ob & X::kAbsMask) >= (X::kExpAll << X::kMantBits);
        uint8_t mk = 0;
        if (special) {
            if (!eq) { spec++; mk = 2; }
        } else if (!eq) {
            const T of = X::from_bits(ob), rf = X::from_bits(rb);
            bool ok;
            double dev;
            if constexpr (kRel) {
                const bool same_sign = (ob >> (X::kBits - 1)) == (rb >> (X::kBits - 1));
                const T q = X::div(X::fabs_(rf), X::fabs_(of));
                ok = same_sign && q <= bound && X::mul(q, bound) >= T(1);
                dev = fabs(__dsub_rn((double)q, 1.0));
            } else {
                const T err = X::fabs_(X::sub(of, rf));
                ok = err <= bound;
                dev = (double)err;
            }
            if (dev != dev) dev = __longlong_as_double(0x7FF0000000000000ll);
            const unsigned long long db = (unsigned long long)__double_as_longlong(dev);
            maxe = db > maxe ? db : maxe;
            if (!ok) {
                viol++;
                first = (unsigned long long)i < first ? (unsigned long long)i : first;
                mk = 1;
            }
        }
        if (mask) mask[i] = mk;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        viol += __shfl_xor_sync(0xFFFFFFFFu, viol, off);
        spec += __shfl_xor_sync(0xFFFFFFFFu, spec, off);
        const unsigned long long f2 = __shfl_xor_sync(0xFFFFFFFFu, first, off);
        first = f2 < first ? f2 : first;
        const unsigned long long m2 = __shfl_xor_sync(0xFFFFFFFFu, maxe, off);
        maxe = m2 > maxe ? m2 : maxe;
    }
    if ((threadIdx.x & 31) == 0) {
        if (viol) atomicAdd(&out5[0], viol);
        if (spec) atomicAdd(&out5[1], spec);
        if (first != ~0ull) atomicMin(&out5[2], first);
        if (maxe) atomicMax(&out5[3], maxe);
    }
}

template <typename T>
int launch_verify(int rel, const void *o, const void *r, int64_t n, T bound, unsigned long long *out5,
                  uint8_t *mask, cudaStream_t st) {
    using U = typename W<T>::U;
    if (n <= 0) return 0;
    if (rel) k_verify<T, true><<<grid_per_sm(n, 8), kThreads, 0, st>>>((const U *)o, (const U *)r, n, bound, out5, mask);
    else k_verify<T, false><<<grid_per_sm(n, 8), kThreads, 0, st>>>((const U *)o, (const U *)r, n, bound, out5, mask);
    return check_launch("verify");
}
template int launch_verify<float>(int, const void *, const void *, int64_t, float, unsigned long long *, uint8_t *,
                                  cudaStream_t);
template int launch_verify<double>(int, const void *, const void *, int64_t, double, unsigned long long *,
                                   uint8_t *, cudaStream_t);

}  // namespace gebq
