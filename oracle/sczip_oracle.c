/*
 * sczip_oracle.c -- CPU restatement of the reference `sczip` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product in paper_2511_11664_b200/; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  It is never
 * linked into, or called by, the product library.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/sczip/) in plain scalar C with the reference's own
 * arithmetic order (float64 where the reference uses float64, Python-int
 * semantics for the rANS state).  Build with -ffp-contract=off so no
 * fused multiply-add changes a rounding the reference performs separately.
 *
 * Status codes mirror the exception classes of errors.py:4-45 (see
 * include/sczip_b200.h for the same numbering used by the product).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
    ORC_OK = 0,
    ORC_INVALID_INPUT = 1,
    ORC_NON_DIVISIBLE = 2,
    ORC_CORRUPT_STREAM = 3,
    ORC_INVALID_CONTAINER = 4,
    ORC_UNSUPPORTED_VERSION = 5,
    ORC_ALPHABET_OVERFLOW = 6,
    ORC_NORMALIZE_ERROR = 7,
    ORC_PRECISION_TOO_SMALL = 8,
    ORC_UNCODABLE_SYMBOL = 9,
    ORC_NO_MEMORY = 50,
};

#define STATE_LOW (1ull << 23) /* rans.py:26 */

/* tensor.py:28-29 _round_half_away_scalar */
static int64_t round_half_away_scalar(double x) {
    double a = floor(fabs(x) + 0.5);
    return (int64_t)copysign(a, x);
}

/* tensor.py:101-122 compute_params.  Python min(x_min, 0.0) returns x_min
 * unless 0.0 < x_min (first argument wins ties), likewise for max. */
int orc_compute_params(double x_min, double x_max, int q_bits, double* scale,
                       int64_t* zero_point) {
    if (!(isfinite(x_min) && isfinite(x_max))) return ORC_INVALID_INPUT;
    if (x_min > x_max) return ORC_INVALID_INPUT;
    if (q_bits < 2 || q_bits > 8) return ORC_INVALID_INPUT;
    int64_t q_max = (1 << q_bits) - 1;
    double lo = (0.0 < x_min) ? 0.0 : x_min;
    double hi = (0.0 > x_max) ? 0.0 : x_max;
    double s;
    int64_t z;
    if (hi == lo) {
        s = 1.0;
        z = 0;
    } else {
        s = (hi - lo) / (double)q_max;
        z = round_half_away_scalar(-lo / s);
    }
    if (z < 0) z = 0;
    if (z > q_max) z = q_max;
    *scale = s;
    *zero_point = z;
    return ORC_OK;
}

/* tensor.py:48 (non-finite check) + tensor.py:127 (t.data.min()/max()). */
int orc_minmax(const float* x, uint64_t n, float* mn, float* mx) {
    float lo = x[0], hi = x[0];
    for (uint64_t i = 0; i < n; ++i) {
        float v = x[i];
        if (!isfinite(v)) return ORC_INVALID_INPUT;
        if (v < lo) lo = v;
        if (v > hi) hi = v;
    }
    *mn = lo;
    *mx = hi;
    return ORC_OK;
}

/* tensor.py:130-140 quantize (+ tensor.py:22-25 _round_half_away).
 * y = float64(x) / scale + z in float64, q = sign(y)*floor(|y|+0.5),
 * clipped to [0, q_max]; mask = (x == 0.0), which includes -0.0. */
void orc_quantize(const float* x, uint64_t n, double scale, int64_t zero_point,
                  int q_bits, uint32_t* q, uint8_t* mask) {
    double q_max = (double)((1 << q_bits) - 1);
    double zf = (double)zero_point;
    for (uint64_t i = 0; i < n; ++i) {
        double y = (double)x[i] / scale;
        y = y + zf;
        double a = floor(fabs(y) + 0.5);
        double r = (y > 0.0) ? a : ((y < 0.0) ? -a : 0.0);
        if (r < 0.0) r = 0.0;
        if (r > q_max) r = q_max;
        q[i] = (uint32_t)r;
        if (mask) mask[i] = (x[i] == 0.0f);
    }
}

/* tensor.py:143-156 dequantize: float32((float64(q) - z) * scale); masked
 * positions come back as +0.0. */
void orc_dequantize(const uint32_t* q, const uint8_t* mask, uint64_t n,
                    double scale, int64_t zero_point, float* out) {
    double zf = (double)zero_point;
    for (uint64_t i = 0; i < n; ++i) {
        double v = ((double)q[i] - zf) * scale;
        out[i] = mask[i] ? 0.0f : (float)v;
    }
}

/* sparse.py:63-69 csr_encode (row-major np.nonzero on ~mask) fused with
 * sparse.py:98-101 concat: D = values ++ col_idx ++ row_counts.
 * d must hold 2*T + n_rows symbols; returns nnz. */
uint64_t orc_csr_concat(const uint32_t* q, const uint8_t* mask,
                        uint64_t n_rows, uint64_t n_cols, uint32_t* d) {
    uint64_t total = n_rows * n_cols, nnz = 0;
    for (uint64_t p = 0; p < total; ++p) nnz += !mask[p];
    uint64_t kv = 0, kc = nnz, kr = 2 * nnz;
    for (uint64_t i = 0; i < n_rows; ++i) {
        uint32_t cnt = 0;
        for (uint64_t j = 0; j < n_cols; ++j) {
            uint64_t p = i * n_cols + j;
            if (!mask[p]) {
                d[kv++] = q[p];
                d[kc++] = (uint32_t)j;
                ++cnt;
            }
        }
        d[kr++] = cnt;
    }
    return nnz;
}

/* Histogram of D for reshape (n_rows x n_cols) without materialising D:
 * the quantity optimizer.py:87-96 (_CostEvaluator.cost) feeds to
 * rans.entropy.  counts must have room for max(2^q, n_cols+1) entries;
 * returns alphabet = max(D)+1 and nnz. */
void orc_stream_counts(const uint32_t* q, const uint8_t* mask, uint64_t n_rows,
                       uint64_t n_cols, int64_t* counts, uint64_t cap,
                       uint64_t* alphabet, uint64_t* nnz_out) {
    memset(counts, 0, cap * sizeof(int64_t));
    uint64_t nnz = 0, amax = 0;
    for (uint64_t i = 0; i < n_rows; ++i) {
        uint64_t cnt = 0;
        for (uint64_t j = 0; j < n_cols; ++j) {
            uint64_t p = i * n_cols + j;
            if (!mask[p]) {
                counts[q[p]]++;
                counts[j]++;
                if (q[p] > amax) amax = q[p];
                if (j > amax) amax = j;
                ++cnt;
            }
        }
        counts[cnt]++;
        if (cnt > amax) amax = cnt;
        nnz += cnt;
    }
    *alphabet = amax + 1;
    *nnz_out = nnz;
}

/* rans.py:76-85 build_counts (np.bincount with AlphabetOverflow guard). */
int orc_build_counts(const uint32_t* d, uint64_t n, uint64_t alphabet,
                     int64_t* counts) {
    if (alphabet < 1) return ORC_INVALID_INPUT;
    memset(counts, 0, alphabet * sizeof(int64_t));
    for (uint64_t i = 0; i < n; ++i) {
        if (d[i] >= alphabet) return ORC_ALPHABET_OVERFLOW;
        counts[d[i]]++;
    }
    return ORC_OK;
}

/* Order used by np.lexsort((arange(A), -remainder)): -remainder ascending
 * (remainder descending), index ascending on ties.  Keys carry their index
 * so the comparator needs no shared state (the CPU baseline is threaded). */
typedef struct {
    double neg_rem;
    uint64_t idx;
} lex_key;
static int cmp_lex(const void* a, const void* b) {
    const lex_key* x = (const lex_key*)a;
    const lex_key* y = (const lex_key*)b;
    if (x->neg_rem < y->neg_rem) return -1;
    if (x->neg_rem > y->neg_rem) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}

/* rans.py:88-131 normalize_frequencies (largest-remainder to 2^precision). */
int orc_normalize(const int64_t* counts, uint64_t alphabet, int precision,
                  int64_t* freqs) {
    int64_t total = 0;
    uint64_t n_present = 0;
    for (uint64_t i = 0; i < alphabet; ++i) {
        total += counts[i];
        n_present += counts[i] > 0;
    }
    if (total <= 0) return ORC_NORMALIZE_ERROR;
    if (precision < 1 || precision > 16) return ORC_INVALID_INPUT;
    int64_t target = (int64_t)1 << precision;
    if ((int64_t)n_present > target) return ORC_PRECISION_TOO_SMALL;
    double ratio = (double)target / (double)total; /* Python int/int */
    lex_key* keys = (lex_key*)malloc(alphabet * sizeof(lex_key));
    if (!keys) return ORC_NO_MEMORY;
    int64_t sum = 0;
    for (uint64_t i = 0; i < alphabet; ++i) {
        double ideal = (double)counts[i] * ratio;
        double fl = floor(ideal);
        freqs[i] = (int64_t)fl;
        keys[i].neg_rem = -(ideal - (double)freqs[i]);
        keys[i].idx = i;
        sum += freqs[i];
    }
    int64_t deficit = target - sum;
    if (deficit > 0) {
        qsort(keys, alphabet, sizeof(lex_key), cmp_lex);
        for (int64_t k = 0; k < deficit && (uint64_t)k < alphabet; ++k)
            freqs[keys[k].idx] += 1;
    }
    free(keys);
    sum = 0;
    for (uint64_t i = 0; i < alphabet; ++i) {
        if (counts[i] > 0 && freqs[i] == 0) freqs[i] = 1;
        sum += freqs[i];
    }
    int64_t surplus = sum - target;
    while (surplus > 0) {
        uint64_t idx = 0;
        for (uint64_t i = 1; i < alphabet; ++i)
            if (freqs[i] > freqs[idx]) idx = i;
        int64_t room = freqs[idx] - 1;
        int64_t cut = room < surplus ? room : surplus;
        if (cut <= 0) return ORC_PRECISION_TOO_SMALL;
        freqs[idx] -= cut;
        surplus -= cut;
    }
    return ORC_OK;
}

/* One lane of rans.py:155-180 encode over symbols d[first + k*stride],
 * k = 0..count-1, pushed in reverse.  Emitted bytes are appended to
 * `emit` (encoder order); returns the final state or 0 on error. */
static int encode_lane(const uint32_t* d, uint64_t first, uint64_t stride,
                       uint64_t count, const int64_t* freqs, const int64_t* cdf,
                       int precision, uint8_t* emit, uint64_t* n_emit,
                       uint64_t* state_out) {
    uint64_t shift = STATE_LOW >> precision;
    uint64_t state = STATE_LOW;
    uint64_t ne = *n_emit;
    for (uint64_t k = count; k-- > 0;) {
        uint32_t x = d[first + k * stride];
        uint64_t f = (uint64_t)freqs[x];
        if (f == 0) return ORC_UNCODABLE_SYMBOL;
        uint64_t bound = (shift << 8) * f;
        while (state >= bound) {
            emit[ne++] = (uint8_t)(state & 0xFF);
            state >>= 8;
        }
        state = ((state / f) << precision) + (uint64_t)cdf[x] + state % f;
    }
    *n_emit = ne;
    *state_out = state;
    return ORC_OK;
}

static int64_t* make_cdf(const int64_t* freqs, uint64_t alphabet) {
    int64_t* cdf = (int64_t*)malloc((alphabet + 1) * sizeof(int64_t));
    if (!cdf) return NULL;
    cdf[0] = 0;
    for (uint64_t i = 0; i < alphabet; ++i) cdf[i + 1] = cdf[i] + freqs[i];
    return cdf;
}

/* rans.py:155-180 encode.  out needs 4 + 2*n bytes (<= 2 bytes per symbol,
 * SURVEY E5).  Layout: 4-byte LE final state + reversed(emitted). */
int orc_rans_encode(const uint32_t* d, uint64_t n, const int64_t* freqs,
                    uint64_t alphabet, int precision, uint8_t* out,
                    uint64_t* out_len) {
    for (uint64_t i = 0; i < n; ++i)
        if (d[i] >= alphabet) return ORC_ALPHABET_OVERFLOW;
    int64_t* cdf = make_cdf(freqs, alphabet);
    uint8_t* emit = (uint8_t*)malloc(2 * n + 8);
    if (!cdf || !emit) {
        free(cdf);
        free(emit);
        return ORC_NO_MEMORY;
    }
    uint64_t ne = 0, state;
    int st = encode_lane(d, 0, 1, n, freqs, cdf, precision, emit, &ne, &state);
    if (st == ORC_OK) {
        for (int b = 0; b < 4; ++b) out[b] = (uint8_t)(state >> (8 * b));
        for (uint64_t i = 0; i < ne; ++i) out[4 + i] = emit[ne - 1 - i];
        *out_len = 4 + ne;
    }
    free(cdf);
    free(emit);
    return st;
}

/* rans.py:183-213 decode with np.searchsorted(cdf, slot, 'right') - 1. */
static uint64_t find_symbol(const int64_t* cdf, uint64_t alphabet, uint64_t slot) {
    /* largest i in [0, alphabet] with cdf[i] <= slot, i.e. searchsorted right - 1 */
    uint64_t lo = 0, hi = alphabet + 1; /* invariant: cdf[lo] <= slot, answer < hi */
    while (hi - lo > 1) {
        uint64_t mid = (lo + hi) / 2;
        if ((uint64_t)cdf[mid] <= slot) lo = mid;
        else hi = mid;
    }
    return lo;
}

int orc_rans_decode(const uint8_t* data, uint64_t len, const int64_t* freqs,
                    uint64_t alphabet, int precision, uint64_t count,
                    uint32_t* out) {
    if (len < 4) return ORC_CORRUPT_STREAM;
    if (precision < 0 || precision > 62) return ORC_CORRUPT_STREAM;
    int64_t* cdf = make_cdf(freqs, alphabet);
    if (!cdf) return ORC_NO_MEMORY;
    uint64_t state = (uint64_t)data[0] | ((uint64_t)data[1] << 8) |
                     ((uint64_t)data[2] << 16) | ((uint64_t)data[3] << 24);
    uint64_t pos = 4, mask = (1ull << precision) - 1;
    int st = ORC_OK;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t slot = state & mask;
        uint64_t sym = find_symbol(cdf, alphabet, slot);
        state = (uint64_t)freqs[sym] * (state >> precision) + slot - (uint64_t)cdf[sym];
        while (state < STATE_LOW) {
            if (pos >= len) {
                st = ORC_CORRUPT_STREAM;
                goto done;
            }
            state = (state << 8) | data[pos++];
        }
        out[i] = (uint32_t)sym;
    }
    if (state != STATE_LOW || pos != len) st = ORC_CORRUPT_STREAM;
done:
    free(cdf);
    return st;
}

/* ---- format v2 (FORMAT.md): interleaved lanes in independent blocks ----
 * D is cut into blocks of `block_syms` symbols (the last may be short).
 * Lane j of a block owns block-local symbols i = j (mod W).  Each lane's
 * state walk is exactly encode_lane (rans.py:134-144 per step).  The
 * encoder walks steps descending and lanes descending, emitting renorm
 * bytes low-first; a block's bytes are W LE u32 final states (lane order)
 * followed by reversed(emitted).  With W=1 and one block this is the v1
 * payload byte for byte. */
int orc_rans_encode_v2(const uint32_t* d, uint64_t n, uint32_t lanes,
                       uint32_t block_syms, const int64_t* freqs,
                       uint64_t alphabet, int precision, uint8_t* out,
                       uint64_t* out_len, uint32_t* block_bytes) {
    if (lanes < 1 || block_syms < lanes || block_syms % lanes) return ORC_INVALID_INPUT;
    for (uint64_t i = 0; i < n; ++i)
        if (d[i] >= alphabet) return ORC_ALPHABET_OVERFLOW;
    int64_t* cdf = make_cdf(freqs, alphabet);
    uint8_t* emit = (uint8_t*)malloc(2 * (uint64_t)block_syms + 8);
    uint64_t* state = (uint64_t*)malloc(lanes * sizeof(uint64_t));
    if (!cdf || !emit || !state) {
        free(cdf);
        free(emit);
        free(state);
        return ORC_NO_MEMORY;
    }
    uint64_t n_blocks = n ? (n + block_syms - 1) / block_syms : 1;
    uint64_t shift = STATE_LOW >> precision;
    uint64_t pos = 0;
    int st = ORC_OK;
    for (uint64_t b = 0; b < n_blocks && st == ORC_OK; ++b) {
        uint64_t base = b * block_syms;
        uint64_t len = n - base < block_syms ? n - base : block_syms;
        if (n == 0) len = 0;
        uint64_t steps = (len + lanes - 1) / lanes;
        uint64_t ne = 0;
        for (uint32_t j = 0; j < lanes; ++j) state[j] = STATE_LOW;
        for (uint64_t s = steps; s-- > 0 && st == ORC_OK;) {
            for (uint32_t j = lanes; j-- > 0;) {
                uint64_t i = s * lanes + j;
                if (i >= len) continue;
                uint32_t x = d[base + i];
                uint64_t f = (uint64_t)freqs[x];
                if (f == 0) {
                    st = ORC_UNCODABLE_SYMBOL;
                    break;
                }
                uint64_t bound = (shift << 8) * f, x0 = state[j];
                while (x0 >= bound) {
                    emit[ne++] = (uint8_t)(x0 & 0xFF);
                    x0 >>= 8;
                }
                state[j] = ((x0 / f) << precision) + (uint64_t)cdf[x] + x0 % f;
            }
        }
        if (st != ORC_OK) break;
        uint64_t start = pos;
        for (uint32_t j = 0; j < lanes; ++j)
            for (int k = 0; k < 4; ++k) out[pos++] = (uint8_t)(state[j] >> (8 * k));
        for (uint64_t i = 0; i < ne; ++i) out[pos++] = emit[ne - 1 - i];
        block_bytes[b] = (uint32_t)(pos - start);
    }
    *out_len = pos;
    free(cdf);
    free(emit);
    free(state);
    return st;
}

int orc_rans_decode_v2(const uint8_t* data, uint64_t len, uint32_t lanes,
                       uint32_t block_syms, uint64_t n_blocks,
                       const uint32_t* block_bytes, const int64_t* freqs,
                       uint64_t alphabet, int precision, uint64_t count,
                       uint32_t* out) {
    if (lanes < 1 || block_syms < lanes || block_syms % lanes) return ORC_CORRUPT_STREAM;
    uint64_t want_blocks = count ? (count + block_syms - 1) / block_syms : 1;
    if (n_blocks != want_blocks) return ORC_CORRUPT_STREAM;
    if (precision < 0 || precision > 62) return ORC_CORRUPT_STREAM;
    uint64_t total = 0;
    for (uint64_t b = 0; b < n_blocks; ++b) total += block_bytes[b];
    if (total != len) return ORC_CORRUPT_STREAM;
    int64_t* cdf = make_cdf(freqs, alphabet);
    uint64_t* state = (uint64_t*)malloc(lanes * sizeof(uint64_t));
    if (!cdf || !state) {
        free(cdf);
        free(state);
        return ORC_NO_MEMORY;
    }
    uint64_t mask = (1ull << precision) - 1, off = 0;
    int st = ORC_OK;
    for (uint64_t b = 0; b < n_blocks && st == ORC_OK; ++b) {
        const uint8_t* p = data + off;
        uint64_t blen = block_bytes[b];
        off += blen;
        uint64_t base = b * block_syms;
        uint64_t nsym = count - base < block_syms ? count - base : block_syms;
        if (count == 0) nsym = 0;
        if (blen < 4ull * lanes) {
            st = ORC_CORRUPT_STREAM;
            break;
        }
        for (uint32_t j = 0; j < lanes; ++j)
            state[j] = (uint64_t)p[4 * j] | ((uint64_t)p[4 * j + 1] << 8) |
                       ((uint64_t)p[4 * j + 2] << 16) | ((uint64_t)p[4 * j + 3] << 24);
        uint64_t pos = 4ull * lanes;
        uint64_t steps = (nsym + lanes - 1) / lanes;
        for (uint64_t s = 0; s < steps && st == ORC_OK; ++s) {
            for (uint32_t j = 0; j < lanes; ++j) {
                uint64_t i = s * lanes + j;
                if (i >= nsym) break;
                uint64_t x = state[j], slot = x & mask;
                uint64_t sym = find_symbol(cdf, alphabet, slot);
                x = (uint64_t)freqs[sym] * (x >> precision) + slot - (uint64_t)cdf[sym];
                while (x < STATE_LOW) {
                    if (pos >= blen) {
                        st = ORC_CORRUPT_STREAM;
                        break;
                    }
                    x = (x << 8) | p[pos++];
                }
                if (st != ORC_OK) break;
                state[j] = x;
                out[base + i] = (uint32_t)sym;
            }
        }
        if (st != ORC_OK) break;
        for (uint32_t j = 0; j < lanes; ++j)
            if (state[j] != STATE_LOW) st = ORC_CORRUPT_STREAM;
        if (pos != blen) st = ORC_CORRUPT_STREAM;
    }
    free(cdf);
    free(state);
    return st;
}

/* sparse.py:104-111 split + sparse.py:72-95 csr_decode: validation order
 * (row count length is structural here), then scatter; all failures are
 * CorruptStream.  q_out/mask_out have n_rows*n_cols entries. */
int orc_csr_decode(const uint32_t* d, uint64_t nnz, uint64_t n_rows,
                   uint64_t n_cols, uint32_t* q_out, uint8_t* mask_out) {
    const uint32_t* v = d;
    const uint32_t* c = d + nnz;
    const uint32_t* r = d + 2 * nnz;
    uint64_t sum = 0;
    for (uint64_t i = 0; i < n_rows; ++i) sum += r[i];
    if (sum != nnz) return ORC_CORRUPT_STREAM;
    for (uint64_t i = 0; i < n_rows; ++i)
        if (r[i] > n_cols) return ORC_CORRUPT_STREAM;
    for (uint64_t k = 0; k < nnz; ++k)
        if (c[k] >= n_cols) return ORC_CORRUPT_STREAM;
    uint64_t k = 0;
    for (uint64_t i = 0; i < n_rows; ++i)
        for (uint64_t t = 0; t < r[i]; ++t, ++k)
            if (t > 0 && c[k] <= c[k - 1]) return ORC_CORRUPT_STREAM;
    uint64_t total = n_rows * n_cols;
    memset(q_out, 0, total * sizeof(uint32_t));
    memset(mask_out, 1, total);
    k = 0;
    for (uint64_t i = 0; i < n_rows; ++i)
        for (uint64_t t = 0; t < r[i]; ++t, ++k) {
            uint64_t p = i * n_cols + c[k];
            q_out[p] = v[k];
            mask_out[p] = 0;
        }
    return ORC_OK;
}

/* ---- whole-tensor round trip (container.py:73-121 with an explicit N) ----
 * Used by the CPU baseline so a timed sample is one C call per tensor.
 * compress: out_payload needs 4*lanes*n_blocks + 2*stream_len bytes. */
typedef struct {
    double scale;
    int64_t zero_point;
    uint64_t nnz;
    uint64_t alphabet;
    uint64_t payload_len;
    uint64_t n_blocks;
} orc_result;

int orc_compress_fixed(const float* x, uint64_t total, int q_bits,
                       uint64_t n_rows, int precision, uint32_t lanes,
                       uint32_t block_syms, int64_t* freqs_out,
                       uint64_t freqs_cap, uint8_t* payload,
                       uint32_t* block_bytes, orc_result* res) {
    if (n_rows < 1 || total % n_rows) return ORC_NON_DIVISIBLE;
    uint64_t n_cols = total / n_rows;
    float mn, mx;
    int st = orc_minmax(x, total, &mn, &mx);
    if (st) return st;
    st = orc_compute_params((double)mn, (double)mx, q_bits, &res->scale, &res->zero_point);
    if (st) return st;
    uint32_t* q = (uint32_t*)malloc(total * sizeof(uint32_t));
    uint8_t* mask = (uint8_t*)malloc(total);
    uint32_t* d = (uint32_t*)malloc((2 * total + n_rows) * sizeof(uint32_t));
    if (!q || !mask || !d) {
        st = ORC_NO_MEMORY;
        goto out;
    }
    orc_quantize(x, total, res->scale, res->zero_point, q_bits, q, mask);
    res->nnz = orc_csr_concat(q, mask, n_rows, n_cols, d);
    uint64_t len = 2 * res->nnz + n_rows, amax = 0;
    for (uint64_t i = 0; i < len; ++i)
        if (d[i] > amax) amax = d[i];
    res->alphabet = amax + 1;
    if (res->alphabet > freqs_cap) {
        st = ORC_INVALID_INPUT;
        goto out;
    }
    int64_t* counts = (int64_t*)malloc(res->alphabet * sizeof(int64_t));
    if (!counts) {
        st = ORC_NO_MEMORY;
        goto out;
    }
    st = orc_build_counts(d, len, res->alphabet, counts);
    if (!st) st = orc_normalize(counts, res->alphabet, precision, freqs_out);
    free(counts);
    if (st) goto out;
    if (lanes == 0) { /* v1 */
        res->n_blocks = 1;
        st = orc_rans_encode(d, len, freqs_out, res->alphabet, precision, payload,
                             &res->payload_len);
    } else {
        res->n_blocks = len ? (len + block_syms - 1) / block_syms : 1;
        st = orc_rans_encode_v2(d, len, lanes, block_syms, freqs_out, res->alphabet,
                                precision, payload, &res->payload_len, block_bytes);
    }
out:
    free(q);
    free(mask);
    free(d);
    return st;
}

int orc_decompress(const uint8_t* payload, uint64_t payload_len, uint32_t lanes,
                   uint32_t block_syms, uint64_t n_blocks,
                   const uint32_t* block_bytes, const int64_t* freqs,
                   uint64_t alphabet, int precision, uint64_t n_rows,
                   uint64_t n_cols, uint64_t nnz, double scale,
                   int64_t zero_point, float* out) {
    uint64_t total = n_rows * n_cols, len = 2 * nnz + n_rows;
    uint32_t* d = (uint32_t*)malloc((len ? len : 1) * sizeof(uint32_t));
    uint32_t* q = (uint32_t*)malloc(total * sizeof(uint32_t));
    uint8_t* mask = (uint8_t*)malloc(total);
    int st;
    if (!d || !q || !mask) {
        st = ORC_NO_MEMORY;
        goto out;
    }
    if (lanes == 0)
        st = orc_rans_decode(payload, payload_len, freqs, alphabet, precision, len, d);
    else
        st = orc_rans_decode_v2(payload, payload_len, lanes, block_syms, n_blocks,
                                block_bytes, freqs, alphabet, precision, len, d);
    if (!st) st = orc_csr_decode(d, nnz, n_rows, n_cols, q, mask);
    if (!st) orc_dequantize(q, mask, total, scale, zero_point, out);
out:
    free(d);
    free(q);
    free(mask);
    return st;
}
