/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the gebq hot path.
 * See gebq_oracle.h for the usage rule.  Each function cites the reference
 * numba loop it restates (paths relative to /root/reference/pkg/src/gebq/).
 *
 * Compiled with -ffp-contract=off -fno-fast-math -mno-fma: one IEEE op per
 * statement, round-to-nearest-even, no flush-to-zero (x86-64 SSE2 scalar).
 */
#include "gebq_oracle.h"

#include <math.h>
#include <string.h>

#define MAXBIN32 (INT64_C(1) << 30)
#define MAXBIN64 (INT64_C(1) << 62)

enum { TRIG_NAN = 0, TRIG_INF = 1, TRIG_GUARD = 2, TRIG_DCHECK = 3 };
enum { DEC_OK = 0, DEC_TRUNCATED = 1, DEC_NONCANONICAL = 2, DEC_COUNT_MISMATCH = 3 };

typedef union { float f; uint32_t u; } f32u;
typedef union { double f; uint64_t u; } f64u;

static inline float as_f32(uint32_t u) { f32u x; x.u = u; return x.f; }
static inline uint32_t f32_bits(float f) { f32u x; x.f = f; return x.u; }
static inline double as_f64(uint64_t u) { f64u x; x.u = u; return x.f; }
static inline uint64_t f64_bits(double f) { f64u x; x.f = f; return x.u; }

/* 2^(e-127) as binary64, e in [0,255] (_kernels.py:27) */
static inline double pow2_32(int64_t e) { return as_f64((uint64_t)(e - 127 + 1023) << 52); }
/* 2^(e-1023), e in [0,2046]; [2047] = +inf (_kernels.py:28). e = 0 is the
 * denormal 2^-1023. */
static inline double pow2_64(int64_t e) {
    if (e == 2047) return as_f64(UINT64_C(0x7FF0000000000000));
    if (e == 0) return as_f64(UINT64_C(0x0008000000000000));
    return as_f64((uint64_t)e << 52);
}

/* _round_bin (_kernels.py:51-69): ties-to-even via floor + exact remainder */
static inline int64_t round_bin32(float t, float *bf) {
    float f = floorf(t);
    float r = t - f;
    int64_t b = (int64_t)f;
    if (r > 0.5f) { *bf = f + 1.0f; return b + 1; }
    if (r < 0.5f) { *bf = f; return b; }
    if ((b & 1) == 0) { *bf = f; return b; }
    *bf = f + 1.0f;
    return b + 1;
}
static inline int64_t round_bin64(double t, double *bf) {
    double f = floor(t);
    double r = t - f;
    int64_t b = (int64_t)f;
    if (r > 0.5) { *bf = f + 1.0; return b + 1; }
    if (r < 0.5) { *bf = f; return b; }
    if ((b & 1) == 0) { *bf = f; return b; }
    *bf = f + 1.0;
    return b + 1;
}

/* _zigzag / _unzigzag (_kernels.py:72-79) */
static inline uint64_t zigzag(int64_t b) { return (uint64_t)((b << 1) ^ (b >> 63)); }
static inline int64_t unzigzag(uint64_t z) { return (int64_t)(z >> 1) ^ -(int64_t)(z & 1); }

/* ------------------------------------------------------------------ */
/* quantize_abs32 (_kernels.py:86-123)                                  */
void orc_quantize_abs32(const uint32_t *bits, int64_t n, uint32_t *codes, uint8_t *lossless,
                        float eb_eff, float eb2, float inv_eb2, float thr, int unsafe,
                        int64_t *trig) {
    for (int64_t i = 0; i < n; i++) {
        uint32_t xb = bits[i];
        float xf = as_f32(xb);
        if (xf != xf) { lossless[i] = 1; codes[i] = xb; trig[TRIG_NAN]++; continue; }
        float t = xf * inv_eb2;
        if (!(fabsf(t) < thr)) {
            lossless[i] = 1; codes[i] = xb;
            if ((xb & 0x7FFFFFFFu) == 0x7F800000u) trig[TRIG_INF]++; else trig[TRIG_GUARD]++;
            continue;
        }
        float bf;
        int64_t b = round_bin32(t, &bf);
        if (b >= MAXBIN32 || b <= -MAXBIN32) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        if (!unsafe) {
            float recon = bf * eb2;
            float err = fabsf(xf - recon);
            if (!(err <= eb_eff)) { lossless[i] = 1; codes[i] = xb; trig[TRIG_DCHECK]++; continue; }
        }
        lossless[i] = 0;
        codes[i] = (uint32_t)zigzag(b);
    }
}

/* quantize_abs64 (_kernels.py:126-162) */
void orc_quantize_abs64(const uint64_t *bits, int64_t n, uint64_t *codes, uint8_t *lossless,
                        double eb_eff, double eb2, double inv_eb2, double thr, int unsafe,
                        int64_t *trig) {
    for (int64_t i = 0; i < n; i++) {
        uint64_t xb = bits[i];
        double xf = as_f64(xb);
        if (xf != xf) { lossless[i] = 1; codes[i] = xb; trig[TRIG_NAN]++; continue; }
        double t = xf * inv_eb2;
        if (!(fabs(t) < thr)) {
            lossless[i] = 1; codes[i] = xb;
            if ((xb & UINT64_C(0x7FFFFFFFFFFFFFFF)) == UINT64_C(0x7FF0000000000000)) trig[TRIG_INF]++;
            else trig[TRIG_GUARD]++;
            continue;
        }
        double bf;
        int64_t b = round_bin64(t, &bf);
        if (b >= MAXBIN64 || b <= -MAXBIN64) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        if (!unsafe) {
            double recon = bf * eb2;
            double err = fabs(xf - recon);
            if (!(err <= eb_eff)) { lossless[i] = 1; codes[i] = xb; trig[TRIG_DCHECK]++; continue; }
        }
        lossless[i] = 0;
        codes[i] = zigzag(b);
    }
}

/* quantize_rel32 (_kernels.py:165-224) */
void orc_quantize_rel32(const uint32_t *bits, int64_t n, uint32_t *codes, uint8_t *lossless,
                        float op_eps, float w, float thr, int unsafe, int64_t *trig) {
    for (int64_t i = 0; i < n; i++) {
        uint32_t xb = bits[i];
        float xf = as_f32(xb);
        if (xf != xf) { lossless[i] = 1; codes[i] = xb; trig[TRIG_NAN]++; continue; }
        uint32_t ab = xb & 0x7FFFFFFFu;
        int64_t aexpo = (int64_t)(ab >> 23);
        if (aexpo == 0xFF) { lossless[i] = 1; codes[i] = xb; trig[TRIG_INF]++; continue; }
        if (aexpo == 0) { lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue; }
        uint32_t amant = ab & 0x7FFFFFu;
        float frac = 1.0f + (float)amant * 0x1p-23f;
        float l = frac + (float)(aexpo - 128);
        float t = l / w;
        if (!(fabsf(t) < thr)) { lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue; }
        float kf;
        int64_t k = round_bin32(t, &kf);
        if (k >= MAXBIN32 || k <= -MAXBIN32) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        float p = kf * w;
        float biased = p + 127.0f;
        if (!(biased >= 1.0f && biased < 255.0f)) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        if (!unsafe) {
            int64_t expo = (int64_t)biased;
            float rfrac = biased - (float)(expo - 1);
            float recon_mag = (float)((double)rfrac * pow2_32(expo));
            float q = recon_mag / fabsf(xf);
            if (!(q <= op_eps && q * op_eps >= 1.0f)) {
                lossless[i] = 1; codes[i] = xb; trig[TRIG_DCHECK]++; continue;
            }
        }
        uint64_t sign = (uint64_t)(xb >> 31);
        lossless[i] = 0;
        codes[i] = (uint32_t)((zigzag(k) << 1) | sign);
    }
}

/* quantize_rel64 (_kernels.py:227-285) */
void orc_quantize_rel64(const uint64_t *bits, int64_t n, uint64_t *codes, uint8_t *lossless,
                        double op_eps, double w, double thr, int unsafe, int64_t *trig) {
    for (int64_t i = 0; i < n; i++) {
        uint64_t xb = bits[i];
        double xf = as_f64(xb);
        if (xf != xf) { lossless[i] = 1; codes[i] = xb; trig[TRIG_NAN]++; continue; }
        uint64_t ab = xb & UINT64_C(0x7FFFFFFFFFFFFFFF);
        int64_t aexpo = (int64_t)(ab >> 52);
        if (aexpo == 0x7FF) { lossless[i] = 1; codes[i] = xb; trig[TRIG_INF]++; continue; }
        if (aexpo == 0) { lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue; }
        uint64_t amant = ab & UINT64_C(0xFFFFFFFFFFFFF);
        double frac = 1.0 + (double)amant * 0x1p-52;
        double l = frac + (double)(aexpo - 1024);
        double t = l / w;
        if (!(fabs(t) < thr)) { lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue; }
        double kf;
        int64_t k = round_bin64(t, &kf);
        if (k >= MAXBIN64 || k <= -MAXBIN64) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        double p = kf * w;
        double biased = p + 1023.0;
        if (!(biased >= 1.0 && biased < 2047.0)) {
            lossless[i] = 1; codes[i] = xb; trig[TRIG_GUARD]++; continue;
        }
        if (!unsafe) {
            int64_t expo = (int64_t)biased;
            double rfrac = biased - (double)(expo - 1);
            double recon_mag = rfrac * pow2_64(expo);
            double q = recon_mag / fabs(xf);
            if (!(q <= op_eps && q * op_eps >= 1.0)) {
                lossless[i] = 1; codes[i] = xb; trig[TRIG_DCHECK]++; continue;
            }
        }
        uint64_t sign = xb >> 63;
        lossless[i] = 0;
        codes[i] = (zigzag(k) << 1) | sign;
    }
}

/* ------------------------------------------------------------------ */
/* reconstruct_* (_kernels.py:293-354)                                  */
void orc_reconstruct_abs32(const uint32_t *codes, const uint8_t *lossless, int64_t n,
                           uint32_t *out_bits, float eb2) {
    for (int64_t i = 0; i < n; i++) {
        if (lossless[i]) { out_bits[i] = codes[i]; continue; }
        int64_t b = unzigzag((uint64_t)codes[i]);
        out_bits[i] = f32_bits((float)b * eb2);
    }
}

void orc_reconstruct_abs64(const uint64_t *codes, const uint8_t *lossless, int64_t n,
                           uint64_t *out_bits, double eb2) {
    for (int64_t i = 0; i < n; i++) {
        if (lossless[i]) { out_bits[i] = codes[i]; continue; }
        int64_t b = unzigzag(codes[i]);
        out_bits[i] = f64_bits((double)b * eb2);
    }
}

void orc_reconstruct_rel32(const uint32_t *codes, const uint8_t *lossless, int64_t n,
                           uint32_t *out_bits, float w) {
    for (int64_t i = 0; i < n; i++) {
        if (lossless[i]) { out_bits[i] = codes[i]; continue; }
        uint32_t c = codes[i];
        uint32_t sign = c & 1u;
        int64_t k = unzigzag((uint64_t)(c >> 1));
        float p = (float)k * w;
        float biased = p + 127.0f;
        if (biased < 0.0f || !(biased < 256.0f)) biased = 0.0f;
        int64_t expo = (int64_t)biased;
        float rfrac = biased - (float)(expo - 1);
        float mag = (float)((double)rfrac * pow2_32(expo));
        out_bits[i] = f32_bits(sign ? -mag : mag);
    }
}

void orc_reconstruct_rel64(const uint64_t *codes, const uint8_t *lossless, int64_t n,
                           uint64_t *out_bits, double w) {
    for (int64_t i = 0; i < n; i++) {
        if (lossless[i]) { out_bits[i] = codes[i]; continue; }
        uint64_t c = codes[i];
        uint64_t sign = c & 1u;
        int64_t k = unzigzag(c >> 1);
        double p = (double)k * w;
        double biased = p + 1023.0;
        if (biased < 0.0 || !(biased < 2048.0)) biased = 0.0;
        int64_t expo = (int64_t)biased;
        double rfrac = biased - (double)(expo - 1);
        double mag = rfrac * pow2_64(expo);
        out_bits[i] = f64_bits(sign ? -mag : mag);
    }
}

/* ------------------------------------------------------------------ */
/* block payload (_kernels.py:439-664)                                  */
static inline int varint_len(uint64_t c) {
    int nb = 1;
    while (c >= 0x80) { c >>= 7; nb++; }
    return nb;
}

static int64_t block_bytes_u32(const uint32_t *codes, int64_t start, int64_t end) {
    int64_t n = end - start;
    int64_t total = ((n + 63) / 64) * 8;
    for (int64_t i = start; i < end; i++) total += varint_len(codes[i]);
    return total;
}
static int64_t block_bytes_u64(const uint64_t *codes, int64_t start, int64_t end) {
    int64_t n = end - start;
    int64_t total = ((n + 63) / 64) * 8;
    for (int64_t i = start; i < end; i++) total += varint_len(codes[i]);
    return total;
}

void orc_block_sizes_u32(const uint32_t *codes, int64_t count, int64_t block_size, int64_t b0,
                         int64_t b1, int64_t *sizes) {
    for (int64_t b = b0; b < b1; b++) {
        int64_t s = b * block_size, e = s + block_size < count ? s + block_size : count;
        sizes[b] = block_bytes_u32(codes, s, e);
    }
}
void orc_block_sizes_u64(const uint64_t *codes, int64_t count, int64_t block_size, int64_t b0,
                         int64_t b1, int64_t *sizes) {
    for (int64_t b = b0; b < b1; b++) {
        int64_t s = b * block_size, e = s + block_size < count ? s + block_size : count;
        sizes[b] = block_bytes_u64(codes, s, e);
    }
}

static int64_t emit_bitmap(const uint8_t *lossless, int64_t start, int64_t end, uint8_t *out,
                           int64_t pos) {
    int64_t nwords = (end - start + 63) / 64;
    for (int64_t wi = 0; wi < nwords; wi++) {
        uint64_t word = 0;
        int64_t base = start + wi * 64;
        int64_t lim = end - base < 64 ? end - base : 64;
        for (int64_t bi = 0; bi < lim; bi++)
            if (lossless[base + bi]) word |= UINT64_C(1) << bi;
        for (int byi = 0; byi < 8; byi++) out[pos++] = (uint8_t)(word >> (8 * byi));
    }
    return pos;
}

void orc_emit_blocks_u32(const uint32_t *codes, const uint8_t *lossless, int64_t count,
                         int64_t block_size, int64_t b0, int64_t b1, const int64_t *offsets,
                         uint8_t *out) {
    for (int64_t b = b0; b < b1; b++) {
        int64_t s = b * block_size, e = s + block_size < count ? s + block_size : count;
        int64_t pos = emit_bitmap(lossless, s, e, out, offsets[b]);
        for (int64_t i = s; i < e; i++) {
            uint32_t c = codes[i];
            while (c >= 0x80u) { out[pos++] = (uint8_t)((c & 0x7Fu) | 0x80u); c >>= 7; }
            out[pos++] = (uint8_t)c;
        }
    }
}
void orc_emit_blocks_u64(const uint64_t *codes, const uint8_t *lossless, int64_t count,
                         int64_t block_size, int64_t b0, int64_t b1, const int64_t *offsets,
                         uint8_t *out) {
    for (int64_t b = b0; b < b1; b++) {
        int64_t s = b * block_size, e = s + block_size < count ? s + block_size : count;
        int64_t pos = emit_bitmap(lossless, s, e, out, offsets[b]);
        for (int64_t i = s; i < e; i++) {
            uint64_t c = codes[i];
            while (c >= 0x80u) { out[pos++] = (uint8_t)((c & 0x7Fu) | 0x80u); c >>= 7; }
            out[pos++] = (uint8_t)c;
        }
    }
}

/* decode_block_u32 / u64 (_kernels.py:521-603) */
static int decode_block(const uint8_t *buf, int64_t pos, int64_t endpos, int64_t nvals,
                        void *codes_v, int wide, uint8_t *lossless, int64_t out_off,
                        int64_t *errpos) {
    int64_t nwords = (nvals + 63) / 64;
    if (pos + nwords * 8 > endpos) { *errpos = pos; return DEC_TRUNCATED; }
    for (int64_t wi = 0; wi < nwords; wi++) {
        uint64_t word = 0;
        for (int byi = 0; byi < 8; byi++) word |= (uint64_t)buf[pos++] << (8 * byi);
        int64_t base = wi * 64;
        int64_t lim = nvals - base < 64 ? nvals - base : 64;
        for (int64_t bi = 0; bi < lim; bi++) lossless[out_off + base + bi] = (word >> bi) & 1;
    }
    const int maxnb = wide ? 10 : 5;
    for (int64_t i = 0; i < nvals; i++) {
        uint64_t val = 0;
        int shift = 0, nb = 0;
        uint8_t last = 0;
        for (;;) {
            if (pos >= endpos) { *errpos = pos; return DEC_TRUNCATED; }
            uint8_t byte = buf[pos++];
            nb++;
            if (nb > maxnb) { *errpos = pos - 1; return DEC_NONCANONICAL; }
            if (wide && nb == 10 && (byte & 0x7E) != 0) { *errpos = pos - 1; return DEC_NONCANONICAL; }
            val |= (uint64_t)(byte & 0x7F) << shift;
            shift += 7;
            last = byte;
            if ((byte & 0x80) == 0) break;
        }
        if (nb > 1 && (last & 0x7F) == 0) { *errpos = pos - 1; return DEC_NONCANONICAL; }
        if (!wide && val > UINT64_C(0xFFFFFFFF)) { *errpos = pos - 1; return DEC_NONCANONICAL; }
        if (wide) ((uint64_t *)codes_v)[out_off + i] = val;
        else ((uint32_t *)codes_v)[out_off + i] = (uint32_t)val;
    }
    if (pos != endpos) { *errpos = pos; return DEC_COUNT_MISMATCH; }
    *errpos = pos;
    return DEC_OK;
}

static int decode_blocks(const uint8_t *buf, const int64_t *offsets, int64_t noffsets,
                         int64_t region_end, int64_t count, int64_t block_size, int64_t b0,
                         int64_t b1, void *codes, int wide, uint8_t *lossless, int64_t *errpos) {
    for (int64_t b = b0; b < b1; b++) {
        int64_t s = b * block_size, e = s + block_size < count ? s + block_size : count;
        int64_t endpos = b + 1 < noffsets ? offsets[b + 1] : region_end;
        int st = decode_block(buf, offsets[b], endpos, e - s, codes, wide, lossless, s, errpos);
        if (st != DEC_OK) return st;
    }
    *errpos = 0;
    return DEC_OK;
}

int orc_decode_blocks_u32(const uint8_t *buf, const int64_t *offsets, int64_t noffsets,
                          int64_t region_end, int64_t count, int64_t block_size, int64_t b0,
                          int64_t b1, uint32_t *codes, uint8_t *lossless, int64_t *errpos) {
    return decode_blocks(buf, offsets, noffsets, region_end, count, block_size, b0, b1, codes, 0,
                         lossless, errpos);
}
int orc_decode_blocks_u64(const uint8_t *buf, const int64_t *offsets, int64_t noffsets,
                          int64_t region_end, int64_t count, int64_t block_size, int64_t b0,
                          int64_t b1, uint64_t *codes, uint8_t *lossless, int64_t *errpos) {
    return decode_blocks(buf, offsets, noffsets, region_end, count, block_size, b0, b1, codes, 1,
                         lossless, errpos);
}

/* ------------------------------------------------------------------ */
/* sweeps (_kernels.py:695-896)                                         */
static inline int class32(uint32_t xb) {
    uint32_t expo = (xb >> 23) & 0xFFu, mant = xb & 0x7FFFFFu;
    if (expo == 0xFFu) return mant ? 4 : 3;
    if (expo == 0u) return mant ? 1 : 0;
    return 2;
}
static inline int class64(uint64_t xb) {
    uint64_t expo = (xb >> 52) & 0x7FFu, mant = xb & UINT64_C(0xFFFFFFFFFFFFF);
    if (expo == 0x7FFu) return mant ? 4 : 3;
    if (expo == 0u) return mant ? 1 : 0;
    return 2;
}

/* one pattern of sweep_abs32_on; returns outcome 0/1/2 */
static inline int sweep_abs32_one(uint32_t xb, float eb_eff, float eb2, float inv_eb2, float thr,
                                  int unsafe) {
    float xf = as_f32(xb);
    int lossless = 0;
    float bf = 0.0f;
    if (xf != xf) {
        lossless = 1;
    } else {
        float t = xf * inv_eb2;
        if (!(fabsf(t) < thr)) {
            lossless = 1;
        } else {
            int64_t b = round_bin32(t, &bf);
            if (b >= MAXBIN32 || b <= -MAXBIN32) {
                lossless = 1;
            } else if (!unsafe) {
                float recon = bf * eb2;
                float err = fabsf(xf - recon);
                if (!(err <= eb_eff)) lossless = 1;
            }
        }
    }
    if (lossless) return 1;
    float recon = bf * eb2;
    float err = fabsf(xf - recon);
    return err <= eb_eff ? 0 : 2;
}

static inline int sweep_abs64_one(uint64_t xb, double eb_eff, double eb2, double inv_eb2,
                                  double thr, int unsafe) {
    double xf = as_f64(xb);
    int lossless = 0;
    double bf = 0.0;
    if (xf != xf) {
        lossless = 1;
    } else {
        double t = xf * inv_eb2;
        if (!(fabs(t) < thr)) {
            lossless = 1;
        } else {
            int64_t b = round_bin64(t, &bf);
            if (b >= MAXBIN64 || b <= -MAXBIN64) {
                lossless = 1;
            } else if (!unsafe) {
                double recon = bf * eb2;
                double err = fabs(xf - recon);
                if (!(err <= eb_eff)) lossless = 1;
            }
        }
    }
    if (lossless) return 1;
    double recon = bf * eb2;
    double err = fabs(xf - recon);
    return err <= eb_eff ? 0 : 2;
}

static inline int sweep_rel32_one(uint32_t xb, float op_eps, float w, float thr, int unsafe) {
    float xf = as_f32(xb);
    int lossless = 0;
    float recon_mag = 0.0f;
    uint32_t ab = xb & 0x7FFFFFFFu;
    int64_t aexpo = (int64_t)(ab >> 23);
    if (xf != xf || aexpo == 0xFF || aexpo == 0) {
        lossless = 1;
    } else {
        uint32_t amant = ab & 0x7FFFFFu;
        float frac = 1.0f + (float)amant * 0x1p-23f;
        float l = frac + (float)(aexpo - 128);
        float t = l / w;
        if (!(fabsf(t) < thr)) {
            lossless = 1;
        } else {
            float kf;
            int64_t k = round_bin32(t, &kf);
            if (k >= MAXBIN32 || k <= -MAXBIN32) {
                lossless = 1;
            } else {
                float p = kf * w;
                float biased = p + 127.0f;
                if (!(biased >= 1.0f && biased < 255.0f)) {
                    lossless = 1;
                } else {
                    int64_t expo = (int64_t)biased;
                    float rfrac = biased - (float)(expo - 1);
                    recon_mag = (float)((double)rfrac * pow2_32(expo));
                    if (!unsafe) {
                        float q = recon_mag / fabsf(xf);
                        if (!(q <= op_eps && q * op_eps >= 1.0f)) lossless = 1;
                    }
                }
            }
        }
    }
    if (lossless) return 1;
    float q = recon_mag / fabsf(xf);
    return (q <= op_eps && q * op_eps >= 1.0f) ? 0 : 2;
}

static inline int sweep_rel64_one(uint64_t xb, double op_eps, double w, double thr, int unsafe) {
    double xf = as_f64(xb);
    int lossless = 0;
    double recon_mag = 0.0;
    uint64_t ab = xb & UINT64_C(0x7FFFFFFFFFFFFFFF);
    int64_t aexpo = (int64_t)(ab >> 52);
    if (xf != xf || aexpo == 0x7FF || aexpo == 0) {
        lossless = 1;
    } else {
        uint64_t amant = ab & UINT64_C(0xFFFFFFFFFFFFF);
        double frac = 1.0 + (double)amant * 0x1p-52;
        double l = frac + (double)(aexpo - 1024);
        double t = l / w;
        if (!(fabs(t) < thr)) {
            lossless = 1;
        } else {
            double kf;
            int64_t k = round_bin64(t, &kf);
            if (k >= MAXBIN64 || k <= -MAXBIN64) {
                lossless = 1;
            } else {
                double p = kf * w;
                double biased = p + 1023.0;
                if (!(biased >= 1.0 && biased < 2047.0)) {
                    lossless = 1;
                } else {
                    int64_t expo = (int64_t)biased;
                    double rfrac = biased - (double)(expo - 1);
                    recon_mag = rfrac * pow2_64(expo);
                    if (!unsafe) {
                        double q = recon_mag / fabs(xf);
                        if (!(q <= op_eps && q * op_eps >= 1.0)) lossless = 1;
                    }
                }
            }
        }
    }
    if (lossless) return 1;
    double q = recon_mag / fabs(xf);
    return (q <= op_eps && q * op_eps >= 1.0) ? 0 : 2;
}

#define SWEEP_BODY(PAT, CLASS, ONE)                     \
    int64_t first = -1;                                 \
    for (int64_t i = 0; i < n; i++) {                   \
        PAT;                                            \
        int o = ONE;                                    \
        tally[CLASS * 3 + o]++;                         \
        if (o == 2 && first < 0) first = i;             \
    }                                                   \
    return first;

int64_t orc_sweep_abs32_on(const uint32_t *bits, int64_t n, float eb_eff, float eb2,
                           float inv_eb2, float thr, int unsafe, int64_t *tally) {
    SWEEP_BODY(uint32_t xb = bits[i], class32(xb),
               sweep_abs32_one(xb, eb_eff, eb2, inv_eb2, thr, unsafe))
}
int64_t orc_sweep_abs64_on(const uint64_t *bits, int64_t n, double eb_eff, double eb2,
                           double inv_eb2, double thr, int unsafe, int64_t *tally) {
    SWEEP_BODY(uint64_t xb = bits[i], class64(xb),
               sweep_abs64_one(xb, eb_eff, eb2, inv_eb2, thr, unsafe))
}
int64_t orc_sweep_rel32_on(const uint32_t *bits, int64_t n, float op_eps, float w, float thr,
                           int unsafe, int64_t *tally) {
    SWEEP_BODY(uint32_t xb = bits[i], class32(xb), sweep_rel32_one(xb, op_eps, w, thr, unsafe))
}
int64_t orc_sweep_rel64_on(const uint64_t *bits, int64_t n, double op_eps, double w,
                           double thr, int unsafe, int64_t *tally) {
    SWEEP_BODY(uint64_t xb = bits[i], class64(xb), sweep_rel64_one(xb, op_eps, w, thr, unsafe))
}
int64_t orc_sweep_abs32_range(uint64_t start, int64_t count, float eb_eff, float eb2,
                              float inv_eb2, float thr, int unsafe, int64_t *tally) {
    int64_t n = count;
    SWEEP_BODY(uint32_t xb = (uint32_t)(start + (uint64_t)i), class32(xb),
               sweep_abs32_one(xb, eb_eff, eb2, inv_eb2, thr, unsafe))
}
int64_t orc_sweep_rel32_range(uint64_t start, int64_t count, float op_eps, float w, float thr,
                              int unsafe, int64_t *tally) {
    int64_t n = count;
    SWEEP_BODY(uint32_t xb = (uint32_t)(start + (uint64_t)i), class32(xb),
               sweep_rel32_one(xb, op_eps, w, thr, unsafe))
}

/* ------------------------------------------------------------------ */
/* splitmix64 (_kernels.py:671-685)                                     */
void orc_splitmix64_fill(uint64_t *out, int64_t n, uint64_t seed, int64_t start_index) {
    for (int64_t i = 0; i < n; i++) {
        uint64_t z = seed + UINT64_C(0x9E3779B97F4A7C15) * (uint64_t)(start_index + i + 1);
        z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
        z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
        out[i] = z ^ (z >> 31);
    }
}

/* ------------------------------------------------------------------ */
/* compute_noa_range (quantizers.py:337-351): max(finite) - min(finite),  */
/* one subtraction in the value width.                                  */
int orc_noa_range32(const uint32_t *bits, int64_t n, float *r) {
    int any = 0;
    float mx = 0.0f, mn = 0.0f;
    for (int64_t i = 0; i < n; i++) {
        if (((bits[i] >> 23) & 0xFFu) == 0xFFu) continue;
        float v = as_f32(bits[i]);
        if (!any) { mx = mn = v; any = 1; continue; }
        if (v > mx) mx = v;
        if (v < mn) mn = v;
    }
    *r = any ? mx - mn : 0.0f;
    return any;
}
int orc_noa_range64(const uint64_t *bits, int64_t n, double *r) {
    int any = 0;
    double mx = 0.0, mn = 0.0;
    for (int64_t i = 0; i < n; i++) {
        if (((bits[i] >> 52) & 0x7FFu) == 0x7FFu) continue;
        double v = as_f64(bits[i]);
        if (!any) { mx = mn = v; any = 1; continue; }
        if (v > mx) mx = v;
        if (v < mn) mn = v;
    }
    *r = any ? mx - mn : 0.0;
    return any;
}
