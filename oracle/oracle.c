/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arxiv 1811.10074 ("Parallel sliding window sums", /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1811_10074_b200/) never links, imports or calls it, and
 * shares no code, header, table or constant generator with it.
 *
 * Every function evaluates the paper's DEFINITION directly, with no blocking,
 * fusion or reordering:
 *   orc_slsum   Eq. 2 (Sec. 2.2): y_i = x_i (+) ... (+) x_{i+w-1},
 *               evaluated as the strict left fold of the w addends, the naive
 *               O(wN) algorithm of L42.
 *   orc_prefix  Eq. 1 (L29-31, Sec. 2.1): y_i = x_0 (+) ... (+) x_i.
 *   orc_encode  the sequence R = r_0, r_1, ... of Sec. 2.4 (L67) as 2-bit codes
 *               (A,C,G,T = 0..3, case-insensitive, anything else invalid; R7).
 *   orc_pack    MSB-first packing of those codes, 32 per uint64 (R6).
 *   orc_kmer    the k-mer starting at base i, L67 ("k-mers of R as a sliding sum
 *               over window size k, string concatenation operator"), built from
 *               scratch per position: code = sum_t b_{i+t} 4^{k-1-t}.
 *   orc_hash    the minimap2-style invertible integer hash of BASELINE.json C1,
 *               restricted to b = 2k bits (R5); orc_unhash inverts it.
 *   orc_mz      minimizers, L85 (Sec. 2.4, Fig. 2): for every window of w
 *               consecutive k-mers, the minimum seed s and its position p'
 *               (leftmost on ties, R2); a pair shared by adjacent
 *               windows is stored once -> the SET of (s, p') over valid windows,
 *               listed by ascending p'.
 *   orc_mz_ties the minimap2-compatible variant (R35): every tied
 *               minimum of every window, run-end windows, symmetric k-mers skipped.
 *   orc_seedtable  the seed pointer table + seed position table of Fig. 1
 *               (L63-65), bucketed on the top `bits` bits of the hash (R21).
 *
 * Multi-threading (OpenMP) only splits independent outputs over threads; each
 * output is computed exactly as in the single-threaded loop.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ECAPACITY (-3)
#define ORC_ENOMEM (-5)

/* operator ids -- same numeric values as the public ABI so tests can pass one id */
enum { ORC_MIN_U32 = 0, ORC_MAX_U32 = 1, ORC_ADD_U32 = 2, ORC_ADD_F32 = 3,
       ORC_AFFINE_U32X2 = 4, ORC_MIN_U64 = 5, ORC_CONCAT_U32X2 = 6 };

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------------- */
/* The operators (+) of Eq. 1 / Eq. 2.                                     */
/* ---------------------------------------------------------------------- */
static uint32_t op_min_u32(uint32_t a, uint32_t b) { return a < b ? a : b; }
static uint32_t op_max_u32(uint32_t a, uint32_t b) { return a > b ? a : b; }
static uint32_t op_add_u32(uint32_t a, uint32_t b) { return a + b; } /* mod 2^32 */
static float op_add_f32(float a, float b) { return a + b; }           /* IEEE binary32, RNE */
static uint64_t op_min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }
/* affine maps t -> a t + b over Z/2^32, composed left-after-right:
 * (a,b) (+) (c,d) = (a c, a d + b).  Associative, not commutative. */
static void op_affine(const uint32_t* l, const uint32_t* r, uint32_t* out) {
    uint32_t a = l[0], b = l[1], c = r[0], d = r[1];
    out[0] = a * c;
    out[1] = a * d + b;
}

/* string concatenation of base-s numerals ("k-mers of R as a sliding sum ...
 * string concatenation operator"): an element (v, s) is a string with value v and weight
 * s = sigma^length; (v1,s1) (+) (v2,s2) = (v1 s2 + v2, s1 s2) over Z/2^32.  For symbols
 * (b, sigma) the w-fold is (sum_t b_t sigma^(w-1-t), sigma^w) mod 2^32. */
static void op_concat(const uint32_t* l, const uint32_t* r, uint32_t* out) {
    uint32_t v1 = l[0], s1 = l[1], v2 = r[0], s2 = r[1];
    out[0] = v1 * s2 + v2;
    out[1] = s1 * s2;
}

static void op_pair(int op, const uint32_t* l, const uint32_t* r, uint32_t* out) {
    if (op == ORC_AFFINE_U32X2) op_affine(l, r, out);
    else op_concat(l, r, out);
}

static size_t elem_size(int op) {
    switch (op) {
    case ORC_MIN_U32: case ORC_MAX_U32: case ORC_ADD_U32: case ORC_ADD_F32: return 4;
    case ORC_AFFINE_U32X2: case ORC_MIN_U64: case ORC_CONCAT_U32X2: return 8;
    default: return 0;
    }
}

/* Eq. 2, strict left fold of exactly w addends (L41), for i in [0, n-w]. */
int orc_slsum(int op, uint32_t w, const void* x, void* y, uint64_t n) {
    if (w == 0 || elem_size(op) == 0) return ORC_EINVAL;
    if (n < w) return ORC_OK;
    int64_t nout = (int64_t)(n - w + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nout; i++) {
        switch (op) {
        case ORC_MIN_U32: case ORC_MAX_U32: case ORC_ADD_U32: {
            const uint32_t* xs = (const uint32_t*)x;
            uint32_t acc = xs[i];
            for (uint32_t j = 1; j < w; j++) {
                uint32_t v = xs[i + j];
                acc = op == ORC_MIN_U32 ? op_min_u32(acc, v)
                    : op == ORC_MAX_U32 ? op_max_u32(acc, v) : op_add_u32(acc, v);
            }
            ((uint32_t*)y)[i] = acc;
            break;
        }
        case ORC_ADD_F32: {
            const float* xs = (const float*)x;
            float acc = xs[i];
            for (uint32_t j = 1; j < w; j++) acc = op_add_f32(acc, xs[i + j]);
            ((float*)y)[i] = acc;
            break;
        }
        case ORC_MIN_U64: {
            const uint64_t* xs = (const uint64_t*)x;
            uint64_t acc = xs[i];
            for (uint32_t j = 1; j < w; j++) acc = op_min_u64(acc, xs[i + j]);
            ((uint64_t*)y)[i] = acc;
            break;
        }
        case ORC_AFFINE_U32X2: case ORC_CONCAT_U32X2: {
            const uint32_t* xs = (const uint32_t*)x;
            uint32_t acc[2] = { xs[2 * i], xs[2 * i + 1] }, t[2];
            for (uint32_t j = 1; j < w; j++) {
                op_pair(op, acc, xs + 2 * (i + j), t);
                acc[0] = t[0]; acc[1] = t[1];
            }
            ((uint32_t*)y)[2 * i] = acc[0];
            ((uint32_t*)y)[2 * i + 1] = acc[1];
            break;
        }
        }
    }
    return ORC_OK;
}

/* Eq. 1: prefix sums, strict left fold. */
int orc_prefix(int op, const void* x, void* y, uint64_t n) {
    if (elem_size(op) == 0) return ORC_EINVAL;
    if (n == 0) return ORC_OK;
    switch (op) {
    case ORC_MIN_U32: case ORC_MAX_U32: case ORC_ADD_U32: {
        const uint32_t* xs = (const uint32_t*)x; uint32_t* ys = (uint32_t*)y;
        uint32_t acc = xs[0]; ys[0] = acc;
        for (uint64_t i = 1; i < n; i++) {
            acc = op == ORC_MIN_U32 ? op_min_u32(acc, xs[i])
                : op == ORC_MAX_U32 ? op_max_u32(acc, xs[i]) : op_add_u32(acc, xs[i]);
            ys[i] = acc;
        }
        break;
    }
    case ORC_ADD_F32: {
        const float* xs = (const float*)x; float* ys = (float*)y;
        float acc = xs[0]; ys[0] = acc;
        for (uint64_t i = 1; i < n; i++) { acc = op_add_f32(acc, xs[i]); ys[i] = acc; }
        break;
    }
    case ORC_MIN_U64: {
        const uint64_t* xs = (const uint64_t*)x; uint64_t* ys = (uint64_t*)y;
        uint64_t acc = xs[0]; ys[0] = acc;
        for (uint64_t i = 1; i < n; i++) { acc = op_min_u64(acc, xs[i]); ys[i] = acc; }
        break;
    }
    case ORC_AFFINE_U32X2: case ORC_CONCAT_U32X2: {
        const uint32_t* xs = (const uint32_t*)x; uint32_t* ys = (uint32_t*)y;
        uint32_t acc[2] = { xs[0], xs[1] }, t[2];
        ys[0] = acc[0]; ys[1] = acc[1];
        for (uint64_t i = 1; i < n; i++) {
            op_pair(op, acc, xs + 2 * i, t); acc[0] = t[0]; acc[1] = t[1];
            ys[2 * i] = acc[0]; ys[2 * i + 1] = acc[1];
        }
        break;
    }
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* DNA: encoding, packing, k-mers, hash (Sec. 2.4; Sec. 4).        */
/* ---------------------------------------------------------------------- */
/* One byte -> (code, valid).  Written as a plain switch on purpose. */
static int base_code(uint8_t ch, uint8_t* code) {
    switch (ch) {
    case 'A': case 'a': *code = 0; return 1;
    case 'C': case 'c': *code = 1; return 1;
    case 'G': case 'g': *code = 2; return 1;
    case 'T': case 't': *code = 3; return 1;
    default: *code = 0; return 0;
    }
}

void orc_encode(const uint8_t* s, uint64_t n, uint8_t* code, uint8_t* valid) {
    for (uint64_t i = 0; i < n; i++) valid[i] = (uint8_t)base_code(s[i], &code[i]);
}

/* words[t] holds bases 32t..32t+31, base 32t+j at bits (63-2j, 62-2j);
 * invalid[t] bit j (LSB = j 0) is set iff base 32t+j is invalid.  Tail bits 0. */
void orc_pack(const uint8_t* s, uint64_t n, uint64_t* words, uint32_t* invalid) {
    uint64_t nw = (n + 31) / 32;
    for (uint64_t t = 0; t < nw; t++) { words[t] = 0; invalid[t] = 0; }
    for (uint64_t i = 0; i < n; i++) {
        uint8_t c;
        int ok = base_code(s[i], &c);
        uint64_t t = i / 32, j = i % 32;
        words[t] |= (uint64_t)c << (62 - 2 * j);
        if (!ok) invalid[t] |= (uint32_t)1 << j;
    }
}

/* code of the k-mer starting at base i, from scratch (no rolling). */
uint64_t orc_kmer(const uint8_t* codes, uint64_t i, int k) {
    uint64_t code = 0;
    for (int t = 0; t < k; t++) code = code * 4 + codes[i + (uint64_t)t];
    return code;
}

/* code of the REVERSE COMPLEMENT of the k-mer starting at base i, from scratch: the k-mer
 * read backwards with every base complemented (A<->T, C<->G, i.e. b -> 3 - b), R32. */
uint64_t orc_kmer_rc(const uint8_t* codes, uint64_t i, int k) {
    uint64_t code = 0;
    for (int t = k - 1; t >= 0; t--) code = code * 4 + (uint64_t)(3 - codes[i + (uint64_t)t]);
    return code;
}

/* H_b (R5): all arithmetic mod 2^b, input x in [0, 2^b).
 *   (1) x <- (2^21 - 1) x - 1    (2) x <- x xor (x >> 24)   (3) x <- 265 x
 *   (4) x <- x xor (x >> 14)     (5) x <- 21 x              (6) x <- x xor (x >> 28)
 *   (7) x <- (2^31 + 1) x
 * Each step is a bijection of [0, 2^b) (odd multipliers; xor-shifts). */
uint64_t orc_hash(uint64_t x, int b) {
    const uint64_t m = (b >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << b) - 1);
    x &= m;
    x = (x * (((uint64_t)1 << 21) - 1) - 1) & m;
    x = (x ^ (x >> 24)) & m;
    x = (x * 265u) & m;
    x = (x ^ (x >> 14)) & m;
    x = (x * 21u) & m;
    x = (x ^ (x >> 28)) & m;
    x = (x * (((uint64_t)1 << 31) + 1)) & m;
    return x;
}

static uint64_t inv_mul(uint64_t a, uint64_t m) {
    /* inverse of odd a mod 2^64 by Newton iteration, then masked */
    uint64_t y = a;                       /* correct to 3 bits */
    for (int i = 0; i < 6; i++) y = y * (2 - a * y);
    return y & m;
}

static uint64_t inv_xorshift(uint64_t y, int s, uint64_t m) {
    /* x = y xor (x >> s): iterate; converges after ceil(b/s) rounds */
    uint64_t x = y;
    for (int i = 0; i < 64 / s + 1; i++) x = (y ^ (x >> s)) & m;
    return x;
}

uint64_t orc_unhash(uint64_t y, int b) {
    const uint64_t m = (b >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << b) - 1);
    uint64_t x = y & m;
    x = (x * inv_mul(((uint64_t)1 << 31) + 1, m)) & m;
    x = inv_xorshift(x, 28, m);
    x = (x * inv_mul(21u, m)) & m;
    x = inv_xorshift(x, 14, m);
    x = (x * inv_mul(265u, m)) & m;
    x = inv_xorshift(x, 24, m);
    x = ((x + 1) * inv_mul(((uint64_t)1 << 21) - 1, m)) & m;
    return x;
}

void orc_hash_array(const uint64_t* x, uint64_t* y, uint64_t n, int b) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) y[i] = orc_hash(x[i], b);
}

/* ---------------------------------------------------------------------- */
/* Minimizers (Sec. 2.4, Fig. 2).                                      */
/* ---------------------------------------------------------------------- */
/* key modes: hashed / raw forward code (R4); canonical = the smaller of the forward and the
 * reverse-complement code (strand-symmetric, R32; NEXT f4), hashed or raw */
enum { ORC_KEY_HASH = 0, ORC_KEY_RAW = 1, ORC_KEY_CANON = 2, ORC_KEY_CANON_RAW = 3 };

/*
 * s[0..n)        ASCII bases (local to this call; global position = pos_base + local)
 * read_off       NULL, or nreads+1 ascending local offsets of segment (read) starts;
 *                read_off[0] = 0, read_off[nreads] = n.  Windows never cross a segment.
 * window i       the w k-mers starting at bases i..i+w-1, i.e. bases [i, i+k+w-2]
 *                (R1).  Valid iff all those bases are A/C/G/T and lie in one
 *                segment (R8).
 * p_i            the leftmost position of the minimum key in window i (R2).
 * output         the distinct pairs (key[p], pos_base + p) over valid windows, by
 *                ascending p (L85: "stored only once"), restricted to pairs whose FIRST
 *                valid window lies in [win_lo, win_hi) (so shards partition the output, R25).
 * returns        the number of records (written up to cap), or < 0 on error.
 */
int64_t orc_mz(const uint8_t* s, uint64_t n, int k, int w,
               const uint64_t* read_off, uint64_t nreads, int keymode,
               uint64_t pos_base, uint64_t win_lo, uint64_t win_hi,
               uint64_t* out_key, uint64_t* out_pos, uint64_t cap) {
    if (k < 1 || k > 31 || w < 1 || keymode < ORC_KEY_HASH || keymode > ORC_KEY_CANON_RAW)
        return ORC_EINVAL;
    const uint64_t span = (uint64_t)k + (uint64_t)w - 1;   /* bases per window */
    if (n < span) return 0;
    const uint64_t nk = n - (uint64_t)k + 1;                /* k-mer positions */
    const uint64_t nwin = n - span + 1;                     /* windows */
    uint8_t* code = malloc(n), *valid = malloc(n);
    uint64_t* seg = malloc(n * sizeof(uint64_t));
    uint64_t* key = malloc(nk * sizeof(uint64_t));
    uint64_t* best = malloc(nwin * sizeof(uint64_t));
    uint8_t* wvalid = malloc(nwin);
    uint64_t* first = malloc(nk * sizeof(uint64_t));
    if (!code || !valid || !seg || !key || !best || !wvalid || !first) {
        free(code); free(valid); free(seg); free(key); free(best); free(wvalid); free(first);
        return ORC_ENOMEM;
    }
    orc_encode(s, n, code, valid);
    /* segment id of every base */
    {
        uint64_t r = 0;
        for (uint64_t j = 0; j < n; j++) {
            if (read_off) while (r + 1 < nreads && read_off[r + 1] <= j) r++;
            seg[j] = read_off ? r : 0;
        }
    }
    /* key of every k-mer position, from scratch */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)nk; i++) {
        uint64_t c = orc_kmer(code, (uint64_t)i, k);
        if (keymode == ORC_KEY_CANON || keymode == ORC_KEY_CANON_RAW) {
            uint64_t r = orc_kmer_rc(code, (uint64_t)i, k);
            if (r < c) c = r;
        }
        key[i] = (keymode == ORC_KEY_HASH || keymode == ORC_KEY_CANON) ? orc_hash(c, 2 * k) : c;
    }
    /* every window: validity by scanning its bases; argmin by a strict '<' scan */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)nwin; i++) {
        int ok = 1;
        for (uint64_t j = (uint64_t)i; j < (uint64_t)i + span; j++)
            if (!valid[j] || seg[j] != seg[i]) { ok = 0; break; }
        wvalid[i] = (uint8_t)ok;
        uint64_t b = (uint64_t)i;
        for (uint64_t j = (uint64_t)i + 1; j < (uint64_t)i + (uint64_t)w; j++)
            if (key[j] < key[b]) b = j;
        best[i] = b;
    }
    /* the set of winners, each with the first valid window that selects it */
    for (uint64_t p = 0; p < nk; p++) first[p] = UINT64_MAX;
    for (uint64_t i = 0; i < nwin; i++)
        if (wvalid[i] && first[best[i]] == UINT64_MAX) first[best[i]] = i;
    int64_t cnt = 0;
    for (uint64_t p = 0; p < nk; p++) {
        if (first[p] != UINT64_MAX && first[p] >= win_lo && first[p] < win_hi) {
            if ((uint64_t)cnt < cap) {
                if (out_key) out_key[cnt] = key[p];
                if (out_pos) out_pos[cnt] = pos_base + p;
            }
            cnt++;
        }
    }
    free(code); free(valid); free(seg); free(key); free(best); free(wvalid); free(first);
    return cnt;
}

/*
 * orc_mz_ties -- the minimap2-compatible variant of the minimizers (PAPER.md L87
 * names minimap2 but fixes neither rule; the reading is DESIGN.md R35):
 *   present k-mer  q: bases q..q+k-1 all A/C/G/T and inside one segment (read);
 *   run            a maximal stretch of consecutive present k-mer positions (an N or a read
 *                  start ends it);
 *   symmetric      (canonical key modes only) forward code == reverse-complement code: the
 *                  k-mer keeps its place in the run but is never selected;
 *   windows        in a run of L k-mers: the L-w+1 windows of w consecutive k-mers if L >= w,
 *                  else ONE window, the whole run (the end rule);
 *   selection      in every window, EVERY non-symmetric k-mer whose key equals the window's
 *                  minimum over its non-symmetric k-mers (all tied minima);
 *   output         the selected positions, each once, ascending, with their keys.
 * Same arguments as orc_mz, without the shard range.  Returns the record count.
 */
int64_t orc_mz_ties(const uint8_t* s, uint64_t n, int k, int w,
                    const uint64_t* read_off, uint64_t nreads, int keymode, uint64_t pos_base,
                    uint64_t* out_key, uint64_t* out_pos, uint64_t cap) {
    if (k < 1 || k > 31 || w < 1 || keymode < ORC_KEY_HASH || keymode > ORC_KEY_CANON_RAW)
        return ORC_EINVAL;
    if (n < (uint64_t)k) return 0;
    const uint64_t nk = n - (uint64_t)k + 1;
    const int canon = keymode == ORC_KEY_CANON || keymode == ORC_KEY_CANON_RAW;
    uint8_t* code = malloc(n), *valid = malloc(n);
    uint64_t* seg = malloc(n * sizeof(uint64_t));
    uint64_t* key = malloc(nk * sizeof(uint64_t));
    uint8_t* present = malloc(nk), *sym = malloc(nk), *sel = malloc(nk);
    if (!code || !valid || !seg || !key || !present || !sym || !sel) {
        free(code); free(valid); free(seg); free(key); free(present); free(sym); free(sel);
        return ORC_ENOMEM;
    }
    orc_encode(s, n, code, valid);
    {
        uint64_t r = 0;
        for (uint64_t j = 0; j < n; j++) {
            if (read_off) while (r + 1 < nreads && read_off[r + 1] <= j) r++;
            seg[j] = read_off ? r : 0;
        }
    }
    for (uint64_t q = 0; q < nk; q++) {
        int ok = 1;
        for (uint64_t j = q; j < q + (uint64_t)k; j++)
            if (!valid[j] || seg[j] != seg[q]) { ok = 0; break; }
        present[q] = (uint8_t)ok;
        sym[q] = 0;
        sel[q] = 0;
        key[q] = 0;
        if (!ok) continue;
        uint64_t c = orc_kmer(code, q, k);
        if (canon) {
            uint64_t r = orc_kmer_rc(code, q, k);
            if (r == c) sym[q] = 1;
            if (r < c) c = r;
        }
        key[q] = (keymode == ORC_KEY_HASH || keymode == ORC_KEY_CANON) ? orc_hash(c, 2 * k) : c;
    }
    /* runs [a, b) of present k-mers, then their windows */
    uint64_t a = 0;
    while (a < nk) {
        if (!present[a]) { a++; continue; }
        uint64_t b = a;
        while (b < nk && present[b]) b++;
        const uint64_t L = b - a;
        const uint64_t ww = L >= (uint64_t)w ? (uint64_t)w : L;     /* window length */
        for (uint64_t i = a; i + ww <= b; i++) {                       /* window [i, i+ww) */
            int have = 0;
            uint64_t mn = 0;
            for (uint64_t q = i; q < i + ww; q++)
                if (!sym[q] && (!have || key[q] < mn)) { mn = key[q]; have = 1; }
            if (!have) continue;
            for (uint64_t q = i; q < i + ww; q++)
                if (!sym[q] && key[q] == mn) sel[q] = 1;
        }
        a = b;
    }
    int64_t cnt = 0;
    for (uint64_t q = 0; q < nk; q++) {
        if (!sel[q]) continue;
        if ((uint64_t)cnt < cap) {
            if (out_key) out_key[cnt] = key[q];
            if (out_pos) out_pos[cnt] = pos_base + q;
        }
        cnt++;
    }
    free(code); free(valid); free(seg); free(key); free(present); free(sym); free(sel);
    return cnt;
}

/* ---------------------------------------------------------------------- */
/* Seed table (Fig. 1, L63-65), bucketed on the top bits of the hash.      */
/* ---------------------------------------------------------------------- */
/* fingerprint = the top 32 bits of the 2k-bit key, left-aligned (R21) */
uint32_t orc_fingerprint(uint64_t key, int k) {
    int b = 2 * k;
    return b >= 32 ? (uint32_t)(key >> (b - 32)) : (uint32_t)(key << (32 - b));
}

/*
 * key[m], pos[m]: records (any order).  bucket(e) = fingerprint(key) >> (32 - bits).
 * offsets[2^bits + 1]: offsets[b] = number of records with bucket < b.
 * pos_out[m], fp_out[m] (fp_out may be NULL): records grouped by bucket, and within a
 * bucket in the order they appear in the input (ascending pos for a minimizer list).
 */
int orc_seedtable(const uint64_t* key, const uint64_t* pos, uint64_t m, int k, int bits,
                  uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out) {
    if (k < 1 || k > 31 || bits < 1 || bits > 30 || bits > 2 * k) return ORC_EINVAL;
    const uint64_t nb = (uint64_t)1 << bits;
    uint64_t* cursor = calloc(nb, sizeof(uint64_t));
    if (!cursor) return ORC_ENOMEM;
    for (uint64_t b = 0; b <= nb; b++) offsets[b] = 0;
    for (uint64_t e = 0; e < m; e++) offsets[(orc_fingerprint(key[e], k) >> (32 - bits)) + 1]++;
    for (uint64_t b = 0; b < nb; b++) offsets[b + 1] += offsets[b];
    for (uint64_t b = 0; b < nb; b++) cursor[b] = offsets[b];
    for (uint64_t e = 0; e < m; e++) {
        uint32_t f = orc_fingerprint(key[e], k);
        uint64_t d = cursor[f >> (32 - bits)]++;
        pos_out[d] = pos[e];
        if (fp_out) fp_out[d] = f;
    }
    free(cursor);
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Seed lookup (Sec. 2.4, Fig. 1: "lookups to 'CG' and 'CT'"; NEXT f1) */
/* ---------------------------------------------------------------------- */
/*
 * For every query key q[i]: f = fingerprint(q[i]), b = f >> (32 - bits); the hits of q[i]
 * are the table entries e in b's slice [offsets[b], offsets[b+1]) with fp[e] == f, in table
 * order (ascending position).  When 2k <= 32 the fingerprint is the whole key, so the hits
 * are exactly the stored positions of that seed (R30).
 * hit_off[nq + 1]: hit_off[i] = number of hits of queries < i.  hit_pos[cap]: the hits of
 * query i at hit_off[i] ..; hits beyond cap are counted but not written.
 * Returns the total number of hits, or a negative error.
 */
int64_t orc_lookup(const uint64_t* q, uint64_t nq, int k, int bits, const uint64_t* offsets,
                   const uint32_t* fp, const uint64_t* pos_tab, uint64_t* hit_off,
                   uint64_t* hit_pos, uint64_t cap) {
    if (k < 1 || k > 31 || bits < 1 || bits > 30 || bits > 2 * k) return ORC_EINVAL;
    /* counts, one query at a time */
    hit_off[0] = 0;
    for (uint64_t i = 0; i < nq; i++) {
        uint32_t f = orc_fingerprint(q[i], k);
        uint64_t b = f >> (32 - bits);
        uint64_t c = 0;
        for (uint64_t e = offsets[b]; e < offsets[b + 1]; e++) c += (fp[e] == f);
        hit_off[i + 1] = hit_off[i] + c;
    }
    /* positions (independent per query) */
    #pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < (int64_t)nq; i++) {
        uint32_t f = orc_fingerprint(q[i], k);
        uint64_t b = f >> (32 - bits);
        uint64_t o = hit_off[i];
        for (uint64_t e = offsets[b]; e < offsets[b + 1]; e++)
            if (fp[e] == f) {
                if (o < cap) hit_pos[o] = pos_tab[e];
                o++;
            }
    }
    return (int64_t)hit_off[nq];
}
