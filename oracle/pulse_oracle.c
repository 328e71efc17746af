/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * Plain-C restatement of the PULSE hot path (arxiv 2602.03839 reference,
 * /root/reference/proj/include/pulse).  Each function names the reference
 * lines it restates.  It is the CPU checker for the CUDA kernels: tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg are the only
 * callers.  Pinned by tests/test_oracle.py against the reference's own
 * known-answer vectors (the reference test sources proj/tests/test_<name>.cpp) and against golden
 * fixtures produced by the reference itself (tests/golden/make_golden.py).
 *
 * Status codes follow include/pulse_cuda.h (0 ok, 2 argument, 6 truncation,
 * 7 corrupt stream, 11 index range, 12 dimension).
 */
#include <stdint.h>
#include <string.h>

enum { PO_OK = 0, PO_ARG = 2, PO_TRUNC = 6, PO_CORRUPT = 7, PO_RANGE = 11, PO_DIM = 12 };

/* patch.hpp:296-301 -- every i with cur[i] != prev[i] (bitwise) in ascending
 * order; index is the flat row-major position, value the current bits. */
uint64_t po_diff(const uint16_t *prev, const uint16_t *curr, uint64_t n, int64_t *idx,
                 uint16_t *val) {
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (prev[i] != curr[i]) {
            if (idx) idx[k] = (int64_t)i;
            if (val) val[k] = curr[i];
            ++k;
        }
    }
    return k;
}

/* wire.hpp:17-47 little-endian emitters */
static void put_u16(uint8_t *p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put_u32(uint8_t *p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint32_t get_u32(const uint8_t *p) {
    return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
static uint16_t get_u16(const uint8_t *p) { return (uint16_t)(p[0] | p[1] << 8); }

/* index_coding.hpp:14-29 delta_encode_indices */
int po_delta_encode(const int64_t *in, uint64_t n, int64_t *out) {
    int64_t prev = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (in[i] < 0) return PO_ARG;
        if (i > 0 && in[i] <= prev) return PO_ARG;
        out[i] = i == 0 ? in[i] : in[i] - prev;
        prev = in[i];
    }
    return PO_OK;
}

/* index_coding.hpp:31-50 delta_decode_indices (FormatError -> 3) */
int po_delta_decode(const int64_t *in, uint64_t n, int64_t *out) {
    int64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (i == 0) {
            if (in[0] < 0) return 3;
            acc = in[0];
        } else {
            if (in[i] <= 0) return 3;
            acc += in[i];
        }
        out[i] = acc;
    }
    return PO_OK;
}

/* patch.hpp:120-130 COO_INT32: u32 LE gaps, first absolute; tensor must have
 * fewer than 2^31 elements (patch.hpp:97-103). */
int po_payload_coo_int32(const int64_t *idx, uint64_t n, uint64_t numel, uint8_t *out,
                         uint64_t *nbytes) {
    if (numel >= ((uint64_t)1 << 31)) return PO_DIM;
    for (uint64_t i = 0; i < n; ++i) {
        if (idx[i] < 0 || (i > 0 && idx[i] <= idx[i - 1])) return PO_ARG;
        put_u32(out + 4 * i, (uint32_t)(i == 0 ? idx[i] : idx[i] - idx[i - 1]));
    }
    *nbytes = 4 * n;
    return PO_OK;
}

/* patch.hpp:131-156 FLAT_INT32: one gap stream across the patch's tensors in
 * patch order; `base` advances by numel of every tensor *in the patch*. */
int po_payload_flat(uint32_t n_tensors, const int64_t *const *idx, const uint64_t *counts,
                    const uint64_t *numel, uint8_t *out, uint64_t *sizes) {
    int64_t base = 0, prev_global = 0;
    int any = 0;
    uint64_t off = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) {
        if (numel[t] >= ((uint64_t)1 << 31)) return PO_DIM;
        for (uint64_t i = 0; i < counts[t]; ++i) {
            int64_t global = base + idx[t][i];
            int64_t entry = any ? global - prev_global : global;
            if (entry < 0 || (any && entry == 0)) return PO_ARG;
            if (entry > (int64_t)0xFFFFFFFFll) return PO_DIM;
            put_u32(out + off, (uint32_t)entry);
            off += 4;
            prev_global = global;
            any = 1;
        }
        sizes[t] = 4 * counts[t];
        base += (int64_t)numel[t];
    }
    return PO_OK;
}

/* index_coding.hpp:68-90 write_row_entry / write_col_entry */
static int row_entry(uint8_t *out, uint64_t *pos, int64_t gap) {
    if (gap > (int64_t)0xFFFFFFFFll) return PO_DIM;
    if (gap >= 0xFF) {
        if (out) { out[*pos] = 0xFF; put_u32(out + *pos + 1, (uint32_t)gap); }
        *pos += 5;
    } else {
        if (out) out[*pos] = (uint8_t)gap;
        *pos += 1;
    }
    return PO_OK;
}
static int col_entry(uint8_t *out, uint64_t *pos, int64_t v) {
    if (v > (int64_t)0xFFFFFFFFll) return PO_DIM;
    if (v >= 0xFFFF) {
        if (out) { put_u16(out + *pos, 0xFFFF); put_u32(out + *pos + 2, (uint32_t)v); }
        *pos += 6;
    } else {
        if (out) put_u16(out + *pos, (uint16_t)v);
        *pos += 2;
    }
    return PO_OK;
}

/* index_coding.hpp:108-128 downscale_coo: row stream (u8 gaps, 0xFF escape)
 * followed by the col stream (u16, absolute on a new row, 0xFFFF escape). */
int po_downscale_coo(const int64_t *rows, const int64_t *cols, uint64_t n, uint8_t *out,
                     uint64_t *nbytes) {
    uint64_t pos = 0;
    int rc;
    for (uint64_t i = 0; i < n; ++i) {
        if (rows[i] < 0 || cols[i] < 0) return PO_ARG;
        if (i > 0 && (rows[i] < rows[i - 1] || (rows[i] == rows[i - 1] && cols[i] <= cols[i - 1])))
            return PO_ARG;
        if ((rc = row_entry(out, &pos, i == 0 ? rows[i] : rows[i] - rows[i - 1]))) return rc;
    }
    for (uint64_t i = 0; i < n; ++i) {
        int new_row = i == 0 || rows[i] != rows[i - 1];
        if ((rc = col_entry(out, &pos, new_row ? cols[i] : cols[i] - cols[i - 1]))) return rc;
    }
    *nbytes = pos;
    return PO_OK;
}

/* patch.hpp:157-171 COO_DOWNSCALED view: row = idx / shape.back(),
 * col = idx % shape.back(); rows/cols scratch of n entries each. */
int po_payload_coo_ds(const int64_t *idx, uint64_t n, int64_t cols_extent, int64_t *rows_tmp,
                      int64_t *cols_tmp, uint8_t *out, uint64_t *nbytes) {
    for (uint64_t i = 0; i < n; ++i) {
        rows_tmp[i] = idx[i] / cols_extent;
        cols_tmp[i] = idx[i] % cols_extent;
    }
    return po_downscale_coo(rows_tmp, cols_tmp, n, out, nbytes);
}

/* index_coding.hpp:130-158 upscale_coo (+ read_*_entry :92-100) */
int po_upscale_coo(const uint8_t *p, uint64_t len, uint64_t count, int64_t *rows, int64_t *cols) {
    uint64_t pos = 0;
    int64_t row = 0, col = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (pos + 1 > len) return PO_TRUNC;
        int64_t e = p[pos++];
        if (e == 0xFF) {
            if (pos + 4 > len) return PO_TRUNC;
            e = get_u32(p + pos);
            pos += 4;
        }
        row = i == 0 ? e : row + e;
        rows[i] = row;
    }
    for (uint64_t i = 0; i < count; ++i) {
        int new_row = i == 0 || rows[i] != rows[i - 1];
        if (pos + 2 > len) return PO_TRUNC;
        int64_t e = get_u16(p + pos);
        pos += 2;
        if (e == 0xFFFF) {
            if (pos + 4 > len) return PO_TRUNC;
            e = get_u32(p + pos);
            pos += 4;
        }
        if (new_row) {
            col = e;
        } else {
            if (e <= 0) return PO_CORRUPT;
            col += e;
        }
        cols[i] = col;
    }
    if (pos != len) return PO_CORRUPT;
    return PO_OK;
}

/* patch.hpp:178-262 decode_index_payloads for the whole patch.  On failure
 * *err_tensor names the tensor the reference would have thrown on. */
int po_decode_payloads(uint32_t repr, uint32_t n_tensors, const uint8_t *const *payloads,
                       const uint64_t *lens, const uint64_t *counts, const uint64_t *numel,
                       const int64_t *cols_extent, int64_t *const *idx_out, int64_t *rows_tmp,
                       int64_t *cols_tmp, uint32_t *err_tensor) {
    int64_t flat_base = 0, prev_global = 0;
    int any = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) {
        const uint8_t *p = payloads[t];
        uint64_t len = lens[t], count = counts[t];
        *err_tensor = t;
        if (repr == 1 || repr == 2) {
            if (numel[t] >= ((uint64_t)1 << 31)) return PO_DIM;
            int64_t index = 0;
            for (uint64_t i = 0; i < count; ++i) {
                if (4 * i + 4 > len) return PO_TRUNC;
                int64_t e = get_u32(p + 4 * i);
                if (repr == 1) { /* COO_INT32 :192-215 */
                    if (i == 0) {
                        index = e;
                    } else {
                        if (e == 0) return PO_CORRUPT;
                        index += e;
                    }
                    if (index >= (int64_t)numel[t]) return PO_CORRUPT;
                    idx_out[t][i] = index;
                } else { /* FLAT_INT32 :216-242 */
                    int64_t global;
                    if (!any) {
                        global = e;
                    } else {
                        if (e == 0) return PO_CORRUPT;
                        global = prev_global + e;
                    }
                    int64_t local = global - flat_base;
                    if (local < 0 || local >= (int64_t)numel[t]) return PO_CORRUPT;
                    idx_out[t][i] = local;
                    prev_global = global;
                    any = 1;
                }
            }
            if (4 * count != len) return PO_CORRUPT;
        } else { /* COO_DOWNSCALED :243-258 */
            int rc = po_upscale_coo(p, len, count, rows_tmp, cols_tmp);
            if (rc) return rc;
            for (uint64_t i = 0; i < count; ++i) {
                if (cols_tmp[i] >= cols_extent[t]) return PO_CORRUPT;
                int64_t flat = rows_tmp[i] * cols_extent[t] + cols_tmp[i];
                if (flat >= (int64_t)numel[t]) return PO_CORRUPT;
                idx_out[t][i] = flat;
            }
        }
        flat_base += (int64_t)numel[t];
    }
    return PO_OK;
}

/* patch.hpp:325-339 validate-and-assign (the copy at :311 is the caller's) */
int po_apply(uint16_t *w, uint64_t numel, const int64_t *idx, const uint16_t *val, uint64_t n) {
    int64_t last = -1;
    for (uint64_t i = 0; i < n; ++i) {
        if (idx[i] <= last) return PO_RANGE;
        if (idx[i] >= (int64_t)numel) return PO_RANGE;
        w[idx[i]] = val[i];
        last = idx[i];
    }
    return PO_OK;
}

/* ---- SHA-256 (FIPS 180-4), the digest hash_weights (sha256.hpp:93-116)
 * obtains from OpenSSL EVP.  Restated from the standard, not from OpenSSL. */
typedef struct {
    uint32_t h[8];
    uint64_t bits;
    uint8_t buf[64];
    uint32_t fill;
} po_sha256;

static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

#define ROR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void sha_block(po_sha256 *s, const uint8_t *b) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
        w[i] = (uint32_t)b[4 * i] << 24 | (uint32_t)b[4 * i + 1] << 16 |
               (uint32_t)b[4 * i + 2] << 8 | b[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
        uint32_t s0 = ROR(w[i - 15], 7) ^ ROR(w[i - 15], 18) ^ (w[i - 15] >> 3);
        uint32_t s1 = ROR(w[i - 2], 17) ^ ROR(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = s->h[0], bb = s->h[1], c = s->h[2], d = s->h[3], e = s->h[4], f = s->h[5],
             g = s->h[6], h = s->h[7];
    for (int i = 0; i < 64; ++i) {
        uint32_t t1 = h + (ROR(e, 6) ^ ROR(e, 11) ^ ROR(e, 25)) + ((e & f) ^ (~e & g)) + K256[i] + w[i];
        uint32_t t2 = (ROR(a, 2) ^ ROR(a, 13) ^ ROR(a, 22)) + ((a & bb) ^ (a & c) ^ (bb & c));
        h = g; g = f; f = e; e = d + t1; d = c; c = bb; bb = a; a = t1 + t2;
    }
    s->h[0] += a; s->h[1] += bb; s->h[2] += c; s->h[3] += d;
    s->h[4] += e; s->h[5] += f; s->h[6] += g; s->h[7] += h;
}

uint64_t po_sha256_ctx_size(void) { return sizeof(po_sha256); }

void po_sha256_init(po_sha256 *s) {
    static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    memcpy(s->h, iv, sizeof iv);
    s->bits = 0;
    s->fill = 0;
}

void po_sha256_update(po_sha256 *s, const uint8_t *p, uint64_t n) {
    s->bits += n * 8;
    while (n) {
        if (s->fill == 0 && n >= 64) {
            sha_block(s, p);
            p += 64; n -= 64;
            continue;
        }
        uint32_t take = 64 - s->fill;
        if (take > n) take = (uint32_t)n;
        memcpy(s->buf + s->fill, p, take);
        s->fill += take; p += take; n -= take;
        if (s->fill == 64) { sha_block(s, s->buf); s->fill = 0; }
    }
}

void po_sha256_final(po_sha256 *s, uint8_t *out32) {
    uint64_t bits = s->bits;
    uint8_t pad = 0x80;
    po_sha256_update(s, &pad, 1);
    uint8_t z = 0;
    while (s->fill != 56) po_sha256_update(s, &z, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    po_sha256_update(s, len, 8);
    for (int i = 0; i < 8; ++i) {
        out32[4 * i] = (uint8_t)(s->h[i] >> 24);
        out32[4 * i + 1] = (uint8_t)(s->h[i] >> 16);
        out32[4 * i + 2] = (uint8_t)(s->h[i] >> 8);
        out32[4 * i + 3] = (uint8_t)s->h[i];
    }
}
