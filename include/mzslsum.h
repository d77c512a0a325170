/*
 * mzslsum.h -- C ABI of the B200 (sm_100a) implementation of the hot path of
 * arxiv 1811.10074, "Parallel sliding window sums".
 *
 * The library (paper_1811_10074_b200/libmzslsum.so) computes:
 *   - sliding window sums y_i = x_i (+) ... (+) x_{i+w-1}        (Eq. 2)
 *     by the block suffix/prefix decomposition of Algorithm 2    (L122-152)
 *     or by O(log w) doubling for commutative operators          (abstract L8, L150, L229);
 *   - 2-bit packing of DNA                                        (Sec. 2.4);
 *   - minimizers: rolling k-mer code + invertible hash + sliding window minimum
 *     (the "faster version of the vector input algorithm", L152) + compaction of the
 *     distinct (seed, position) pairs                             (Sec. 2.4, Fig. 2);
 *   - a seed table: pointer table + position table                (Sec. 2.4, Fig. 1),
 *     bucketed on the top bits of the hash, with the phase functions of the
 *     multi-GPU build (count / partition / finalize; NCCL runs between them).
 *
 * CONVENTIONS (all entry points)
 *   - Every array argument is a DEVICE pointer owned by the caller, unless the
 *     parameter name starts with h_ (host).  The library never frees caller memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     *_ex and phase functions are asynchronous and stream-ordered; the plain
 *     convenience calls (slsum_run, mz_extract, seedtable_build with h_m) synchronize.
 *   - Scratch memory comes from the caller's workspace `ws` of `ws_bytes` bytes,
 *     sized by the matching *_workspace_bytes call; passing ws = NULL makes the call
 *     allocate (cudaMallocAsync) and free its own scratch on `stream`.
 *   - Return value 0 = success; negative = error code below (see slsum_strerror).
 *     Degenerate sizes are NOT errors: n < w gives 0 sums, a sequence shorter
 *     than k + w - 1 gives 0 minimizers, m = 0 gives an all-zero pointer table.
 *   - Integer results are bit-identical for any stream, tile size or GPU count.
 *   - Thread safety: stateless; concurrent calls are safe with distinct workspaces.
 */
#ifndef MZSLSUM_H
#define MZSLSUM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ errors */
#define SLSUM_OK            0
#define SLSUM_EINVAL       (-1)  /* NULL pointer, w = 0, k not in [1,31], bad op/kind/bits */
#define SLSUM_EUNSUPPORTED (-2)  /* non-commutative op on the COMMUTATIVE path          */
#define SLSUM_ECAPACITY    (-3)  /* more records than `capacity` (sync calls only)      */
#define SLSUM_ECUDA        (-4)  /* CUDA launch / runtime error                         */
#define SLSUM_ENOMEM       (-5)  /* workspace too small / allocation failed            */

const char* slsum_strerror(int rc);
/* library version, e.g. 0x000100 */
int slsum_version(void);

/* ------------------------------------------------------------------ sliding sums
 * Eq. 2: y_i = x_i (+) x_{i+1} (+) ... (+) x_{i+w-1}, exactly w
 * addends, for i in [0, n-w]; y receives max(0, n-w+1) elements.
 *
 * op (element type of x and y):
 *   SLSUM_MIN_U32       uint32 min
 *   SLSUM_MAX_U32       uint32 max
 *   SLSUM_ADD_U32       uint32 add modulo 2^32
 *   SLSUM_ADD_F32       float32 add (result within 1e-5 |ref| + 1e-6 w of the strict
 *                       left fold; the decomposition regroups the w terms)
 *   SLSUM_AFFINE_U32X2  pairs (a, b) of uint32 (8 bytes per element), the affine map
 *                       t -> a t + b over Z/2^32 composed left-after-right:
 *                       (a,b) (+) (c,d) = (a c, a d + b).  Associative and NOT
 *                       commutative: proves that a path preserves operand order.
 *   SLSUM_MIN_U64       uint64 min (e.g. (key << 32 | pos) argmin keys)
 *   SLSUM_CONCAT_U32X2  pairs (v, s) of uint32: a string with base-sigma value v and weight
 *                       s = sigma^length; (v1,s1) (+) (v2,s2) = (v1 s2 + v2, s1 s2) mod 2^32,
 *                       string concatenation (L67: "k-mers of R as a sliding sum ... string
 *                       concatenation").  With x_i = (symbol_i, sigma) and w = k, y_i is the
 *                       k-mer code of any alphabet (exact while sigma^k <= 2^32) and sigma^k.
 *                       Not commutative (GENERIC, SCALAR; COMMUTATIVE -> EUNSUPPORTED).
 * path:
 *   SLSUM_PATH_GENERIC      Algorithm 2's decomposition with blocks of length w:
 *                           y_i = S[i] (+) P[i+w-1] (S = suffix fold to the end of i's
 *                           block, P = prefix fold from the start of its block), 3 (+)
 *                           per output, any associative op, operand order preserved.
 *   SLSUM_PATH_COMMUTATIVE  ceil(log2 w) doubling rounds (abstract L8: O(P/log w) "for a
 *                           sum with commutative operator"); rejects AFFINE with
 *                           SLSUM_EUNSUPPORTED.
 *   SLSUM_PATH_AUTO         GENERIC (the faster path on B200 for every w).
 *   SLSUM_PATH_RECURRENT    Conclusion (L229): a "recurrent interpretation", speedup
 *                           independent of w.  For an invertible op, y_i = PS[i+w-1] (-)
 *                           PS[i-1] with PS the prefix sums (tile-local; the difference
 *                           cancels the offset).  SLSUM_ADD_U32 only (exact mod 2^32); any
 *                           other op returns SLSUM_EUNSUPPORTED (min/max are not invertible,
 *                           f32 add would lose the tolerance to cancellation).
 *   SLSUM_PATH_SCALAR       Algorithm 1 "ScalarInput" (L95-120): a warp-wide shift register
 *                           of window accumulators; every window is the strict left fold,
 *                           so the result is bit-identical to Eq. 2 evaluated naively for
 *                           EVERY op (f32 add and AFFINE included; "no additional
 *                           requirements on the operator").  O(w) work per output;
 *                           w <= 1024, else SLSUM_EUNSUPPORTED.
 * x, y: device arrays of n and max(0, n-w+1) elements; x and y must not overlap.
 */
enum {
  SLSUM_MIN_U32 = 0,
  SLSUM_MAX_U32 = 1,
  SLSUM_ADD_U32 = 2,
  SLSUM_ADD_F32 = 3,
  SLSUM_AFFINE_U32X2 = 4,
  SLSUM_MIN_U64 = 5,
  SLSUM_CONCAT_U32X2 = 6
};
enum {
  SLSUM_PATH_GENERIC = 0,
  SLSUM_PATH_COMMUTATIVE = 1,
  SLSUM_PATH_AUTO = 2,
  SLSUM_PATH_RECURRENT = 3,
  SLSUM_PATH_SCALAR = 4
};

/* GENERIC path on the default stream; returns after completion. */
int slsum_run(int op, uint32_t w, const void* x, void* y, uint64_t n);
/* asynchronous on `stream`; no workspace needed. */
int slsum_run_ex(int op, uint32_t w, const void* x, void* y, uint64_t n, int path, void* stream);

/* ------------------------------------------------------------------ 2-bit packing
 * Sec. 2.4 (L67) sequence R = r_0 r_1 ...; encoding per DESIGN.md R6/R7:
 * A/a -> 0, C/c -> 1, G/g -> 2, T/t -> 3; every other byte is invalid (code 0).
 * words[t] (uint64, ceil(n/32) of them) holds bases 32t..32t+31, MSB-first: base 32t+j
 * at bits (63-2j, 62-2j).  invalid[t] (uint32, ceil(n/32)) has bit j set iff base
 * 32t+j is invalid.  Bits past n are 0.  seq: n device bytes.
 */
int mz_encode(const uint8_t* seq, uint64_t n, uint64_t* words, uint32_t* invalid, void* stream);

/* ------------------------------------------------------------------ minimizers
 * PAPER.md L85 (Sec. 2.4, Fig. 2) with the readings of DESIGN.md:
 *   k-mer q       code_q = sum_{t<k} b_{q+t} 4^(k-1-t) (2k bits, MSB-first, R6)
 *   key_q         H_2k(code_q) (MZ_KEY_HASH; the masked Wang/minimap2 mix, R5)
 *                 or code_q (MZ_KEY_RAW, Fig. 2's lexicographic order, R4);
 *                 MZ_KEY_CANON / MZ_KEY_CANON_RAW: the same on the canonical code
 *                 min(code_q, revcomp(code_q)) (strand-symmetric minimizers, R32; the
 *                 paper's Fig. 2 is forward-strand only, R10)
 *   window i      the w k-mers q = i .. i+w-1 = bases [i, i+k+w-2] (R1); valid iff all
 *                 those bases are A/C/G/T and no segment (read) starts in (i, i+k+w-2] (R8)
 *   p_i           the leftmost position of the minimum key in window i (R2)
 *   output        every distinct (key[p], pos_base + p) selected by a valid window,
 *                 ascending by position (L85 "stored only once"), each pair emitted by
 *                 the first valid window selecting it (change rule, R3).
 * Input kinds:
 *   MZ_IN_ASCII    seq = n bytes
 *   MZ_IN_PACKED2  seq = ceil(n/32) uint64 words as written by mz_encode; invalid =
 *                  ceil(n/32) uint32 bitmap words, or NULL if every base is valid
 * read_off: NULL, or nreads + 1 ascending LOCAL base offsets, read_off[0] = 0,
 *   read_off[nreads] = n; windows never span two reads (C4 segmented windows).
 * pos_base: added to every emitted position (global offset of seq[0]).
 * [win_lo, win_hi): LOCAL window range whose first-selections are emitted (a shard
 *   owning global windows [a,b) passes bases [a-1, b+k+w-2) with win_lo = 1 when a > 0,
 *   R25); win_hi = UINT64_MAX means "all".
 * out: hash[capacity], pos[capacity] (uint64 each; hash = key), d_count (1 uint64,
 *   device) receives the total number of records even if it exceeds capacity; only the
 *   first min(count, capacity) records are written, in order.
 * Supported: k in [1, 31], w >= 1, 2k >= 1.  Records per window <= 1, so capacity =
 *   number of windows always suffices.
 */
enum { MZ_IN_ASCII = 0, MZ_IN_PACKED2 = 1 };
enum { MZ_KEY_HASH = 0, MZ_KEY_RAW = 1, MZ_KEY_CANON = 2, MZ_KEY_CANON_RAW = 3 };

typedef struct mz_in {
  int kind;                  /* MZ_IN_ASCII or MZ_IN_PACKED2                    */
  const void* seq;           /* device: bytes or packed words                   */
  const uint32_t* invalid;   /* device: invalid bitmap for PACKED2, or NULL     */
  uint64_t n;                /* number of bases                                 */
  const uint64_t* read_off;  /* device: nreads+1 read starts, or NULL           */
  uint64_t nreads;
  uint64_t pos_base;
  uint64_t win_lo;
  uint64_t win_hi;
} mz_in_t;

typedef struct mz_out {
  uint64_t* hash;            /* device, capacity entries */
  uint64_t* pos;             /* device, capacity entries */
  uint64_t capacity;
  uint64_t* d_count;         /* device, 1 entry          */
  uint64_t* items;           /* device, capacity entries, or NULL: packed seed-table items
                                fp(hash) << 32 | (pos mod 2^32), fp = the top 32 bits of the
                                2k-bit key (seedtable_build_items' input)            */
  uint32_t* hist;            /* device, or NULL: the digit counts of the seed table's FIRST
                                radix pass over the written records (the first pass's
                                "upsweep", fused into extraction; seedtable_build_items_ex's
                                `hist`).  seedtable_hist_words(capacity, hist_bucket_bits)
                                uint32 words; zeroed and filled by mz_extract_ex.  Layout:
                                hist[d * nchunks + c] = number of records r < min(count,
                                capacity) with r in chunk c (chunks of the seed table's radix
                                chunk size for m = capacity) and digit d = bits
                                [32 - bucket_bits, 40 - bucket_bits) of fp (the least
                                significant 8 bits of the bucket, as many as it has).  */
  int hist_bucket_bits;      /* bucket_bits of the table the hist is for (1..min(2k,30))  */
} mz_out_t;

/* scratch for mz_extract_ex on n bases (tile descriptors + packed copy for ASCII) */
size_t mz_workspace_bytes(uint64_t n, int k, int w, int kind);
/* asynchronous extraction on `stream`. */
int mz_extract_ex(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out,
                  void* ws, size_t ws_bytes, void* stream);
/* mz_extract_ex with the kernel family forced (a test hook: both families compute the same
 * output, bit for bit).  path 0 = automatic (what mz_extract_ex does: the compile-time-w fast
 * kernel for w <= 16 and 2k <= 50, else the generic one); path 1 = the generic kernel
 * (block-wide segmented S/P scans, any w <= 1024, any k).  Any other value is treated as 1. */
int mz_extract_path(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out,
                    void* ws, size_t ws_bytes, void* stream, int path);
/* BASELINE shape: ASCII input, hashed keys, one segment, pos_base 0, default stream.
 * Synchronous; returns SLSUM_ECAPACITY if the count exceeds out->capacity
 * (*out->d_count then holds the required count). */
int mz_extract(const uint8_t* seq, uint64_t n, int k, int w, mz_out_t* out);

/* minimap2-compatible minimizers (PAPER.md L87 names minimap2 but fixes neither
 * rule; the reading is DESIGN.md R35).  Same inputs, key modes and outputs as mz_extract_ex,
 * with three rules changed:
 *   run      a maximal stretch of consecutive PRESENT k-mers (all k bases A/C/G/T, one read);
 *            windows never leave a run, and a run of L < w k-mers is ONE window (end rule);
 *   ties     EVERY k-mer whose key equals its window's minimum is a record (not only the
 *            leftmost one);
 *   strand   (MZ_KEY_CANON*) a symmetric k-mer (code = its reverse complement; even k only)
 *            keeps its place in the run but is never selected.
 * Output: the distinct selected (key, pos_base + q), ascending q; at most one per k-mer, so
 * capacity = n - k + 1 always suffices.  out->items is written if non-NULL; out->hist must be
 * NULL (SLSUM_EINVAL).  The shard range is not supported: win_lo must be 0 and win_hi
 * UINT64_MAX (else SLSUM_EUNSUPPORTED).  Computed with two sliding window sums (Eq. 2,
 * (+) = min, L38-41) of the keys: the window minima m_j, then M_q = max of the m_j over the
 * windows holding q; q is a record iff key_q = M_q.  Asynchronous on `stream`; workspace
 * mz_ties_workspace_bytes(n, k, w, kind) (about 32 B per base), or NULL to allocate. */
size_t mz_ties_workspace_bytes(uint64_t n, int k, int w, int kind);
int mz_extract_ties(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out,
                    void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ seed table
 * Fig. 1 (L63-65): a pointer table over seeds + a position table.  Seeds are bucketed
 * on the top `bucket_bits` bits of the 2k-bit key (R21):
 *   fp(key)     = key >> (2k-32) if 2k >= 32, else key << (32-2k)   (top-aligned 32 bits)
 *   bucket(key) = fp(key) >> (32 - bucket_bits)
 * offsets[2^bucket_bits + 1] (uint64): offsets[b] = number of records with bucket < b.
 * pos_out[m] (uint64): positions grouped by bucket, ascending position inside a bucket.
 * fp_out[m] (uint32, may be NULL): the fingerprints in the same order.
 * m: number of records; if d_m != NULL the count is read on the device from *d_m and m is
 *   only its upper bound (lets the table follow mz_extract_ex without a host sync).
 * Requires 1 <= bucket_bits <= min(2k, 30).
 */
size_t seedtable_workspace_bytes(uint64_t m, int bucket_bits);
int seedtable_build(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m,
                    int k, int bucket_bits, uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out,
                    void* ws, size_t ws_bytes, void* stream);
/* The same table from the packed items mz_extract_ex wrote (out->items) beside hash/pos: the
 * first radix pass reads the 8-byte items instead of the 16-byte (hash, pos) pairs.  Requires
 * items[i] = fp(hash[i]) << 32 | (pos[i] mod 2^32) and positions ascending (as mz_extract_ex
 * writes them).  hash and pos are still read: pos[0] and pos[m-1] decide the packed path,
 * and the wide path (positions spanning >= 2^32) sorts from hash/pos.  Same workspace and
 * output as seedtable_build.  PRECONDITION: pos ascending.  Unlike seedtable_build, the
 * per-entry range check is not done here (the items already carry pos mod 2^32), so an
 * unsorted pos gives a wrong table, not a fallback. */
int seedtable_build_items(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                          const uint64_t* d_m, int k, int bucket_bits, uint64_t* offsets,
                          uint32_t* fp_out, uint64_t* pos_out, void* ws, size_t ws_bytes, void* stream);

/* seedtable_build_items with a 32-bit position table: pos32_out[m] (uint32) receives every
 * position mod 2^32 -- the positions themselves when they are below 2^32 (one genome of
 * < 4.29 Gbases per table, e.g. C3), half the bytes of pos_out.  Offsets and fp_out as in
 * seedtable_build.  Same workspace (seedtable_workspace_bytes). */
int seedtable_build_items32(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                            const uint64_t* d_m, int k, int bucket_bits, uint64_t* offsets,
                            uint32_t* fp_out, uint32_t* pos32_out, void* ws, size_t ws_bytes, void* stream);

/* Size (uint32 words) of mz_out.hist for a table of `bucket_bits` built from `capacity` records
 * (m = capacity in seedtable_build_items_ex). */
size_t seedtable_hist_words(uint64_t capacity, int bucket_bits);
/* seedtable_build_items / seedtable_build_items32 in one call, optionally starting from the first
 * pass's digit counts that mz_extract_ex accumulated while writing the records (out->hist,
 * out->hist_bucket_bits == bucket_bits, out->capacity == m): the first pass then skips its own
 * count of the items (one read of 8 B per entry).  hist may be NULL (the counts are taken
 * here).  Exactly one of pos_out (uint64) / pos32_out (uint32, positions mod 2^32, R34) is
 * non-NULL.  Same preconditions, workspace and output as seedtable_build_items.  The hist is
 * only used by the packed-item path; the wide path (positions spanning >= 2^32) counts
 * itself. */
int seedtable_build_items_ex(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                             const uint64_t* d_m, int k, int bucket_bits, const uint32_t* hist,
                             uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out, uint32_t* pos32_out,
                             void* ws, size_t ws_bytes, void* stream);

/* Multi-GPU phases (owner(bucket) = bucket >> (bucket_bits - log2 nranks); nranks a
 * power of two; NCCL all_reduce / all_to_all run between these calls):
 *  seedtable_count      counts[2^bits] (uint32) = per-bucket record counts (overwritten).
 *  seedtable_partition  stable partition of the records by owner rank: send_fp/send_pos
 *                       (m entries) grouped by owner, ascending position inside a group;
 *                       send_counts[nranks] (uint64, device) entries per owner.
 *  seedtable_finalize   from the received entries (concatenated in sender-rank order) and
 *                       the all-reduced counts, build this rank's slice of the table:
 *                       offsets_local[2^bits/nranks + 1] starting at 0, pos_out/fp_out
 *                       (m_recv entries).  Concatenating the ranks' slices (offsets
 *                       shifted by the preceding ranks' totals) gives seedtable_build's
 *                       output on the union of the records.
 */
int seedtable_count(const uint64_t* hash, uint64_t m, const uint64_t* d_m, int k, int bucket_bits,
                    uint32_t* counts, void* stream);
size_t seedtable_partition_workspace_bytes(uint64_t m, int nranks);
int seedtable_partition(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m,
                        int k, int bucket_bits, int nranks, uint32_t* send_fp, uint64_t* send_pos,
                        uint64_t* send_counts, void* ws, size_t ws_bytes, void* stream);
/* seedtable_partition_p2p: the partition FUSED with the all-to-all.  The stable
 *   pass on the owner digit writes each entry directly into its owner's receive buffers
 *   (peer_fp[o] uint32 / peer_pos[o] uint64: device pointers, typically peer-mapped symmetric
 *   memory over NVLink), starting at peer_base[o], the number of entries for owner o held by
 *   the senders of lower rank.  peer_fp/peer_pos/peer_base are HOST arrays of nranks values.
 *   Requires nranks >= 2 and pos ascending with pos[m-1] - pos[0] < 2^32 (one shard of < 4.29
 *   Gbases); returns SLSUM_EUNSUPPORTED otherwise (use partition + NCCL all_to_all).  The span
 *   is checked from pos[0] and pos[m-1] before any write; an unsorted pos is detected by the
 *   write pass itself, which then also returns SLSUM_EUNSUPPORTED, but only after it has
 *   written wrong entries into the peers' buffers: the caller must then discard them and
 *   fall back on every rank.  Reads the
 *   device count and two positions (a short synchronization), then runs asynchronously and
 *   synchronizes the stream before returning.  The caller barriers across ranks before the
 *   owners read their buffers. */
size_t seedtable_partition_p2p_workspace_bytes(uint64_t m, int nranks);
int seedtable_partition_p2p(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m,
                            int k, int bucket_bits, int nranks, const uint64_t* peer_fp,
                            const uint64_t* peer_pos, const uint64_t* peer_base, void* ws,
                            size_t ws_bytes, void* stream);
/* seedtable_partition_p2p from the packed items mz_extract_ex wrote (out->items, see
 *   seedtable_build_items): reads 8 B per entry instead of the 16-byte (hash, pos) pair; pos is
 *   read only at pos[0] and pos[m-1] (the narrow precondition and the base of the positions).
 *   PRECONDITION: pos ascending (not re-checked per entry: an unsorted pos gives wrong entries,
 *   not SLSUM_EUNSUPPORTED).  Same workspace (seedtable_partition_p2p_workspace_bytes). */
int seedtable_partition_p2p_items(const uint64_t* items, const uint64_t* pos, uint64_t m, const uint64_t* d_m,
                                  int k, int bucket_bits, int nranks, const uint64_t* peer_fp,
                                  const uint64_t* peer_pos, const uint64_t* peer_base, void* ws,
                                  size_t ws_bytes, void* stream);
size_t seedtable_finalize_workspace_bytes(uint64_t m_recv, int bucket_bits, int nranks);
int seedtable_finalize(const uint32_t* recv_fp, const uint64_t* recv_pos, uint64_t m_recv,
                       const uint32_t* global_counts, int bucket_bits, int rank, int nranks,
                       uint64_t* offsets_local, uint64_t* pos_out, uint32_t* fp_out,
                       void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ seed lookup
 * Fig. 1 (L63-65): "The seed pointer table enables fast lookups to 'CG' and 'CT'" -- the
 * seeding step that consumes the table.  For query key qkey[i] (a 2k-bit
 * hash, or a raw code for a raw table): f = fp(qkey[i]), b = f >> (32 - bucket_bits); its
 * hits are the entries e of bucket b's slice [offsets[b], offsets[b+1]) with fp[e] == f,
 * in table order (ascending position).  When 2k <= 32 the fingerprint is the whole key and
 * the hits are exactly the stored positions of that seed; for 2k > 32 they are the
 * entries that agree on the key's top 32 bits (R30).
 * offsets/fp/pos_tab: a table from seedtable_build (fp_out must have been requested).
 * nq: number of queries, or its upper bound when d_nq (device) holds the count.
 * hit_off[nq + 1] (uint64, device): hit_off[i] = hits of the queries before i;
 *   hit_off[count] = total.  hit_pos[hit_cap]: the hits of query i at hit_off[i]...; hits at
 *   or beyond hit_cap are counted, not written (hit_cap = 0: count only, hit_pos may be NULL).
 * d_total (device, may be NULL): the total number of hits.
 * Asynchronous on `stream`; scratch from ws (seedtable_lookup_workspace_bytes), or an
 * internal cudaMallocAsync when ws == NULL.
 */
size_t seedtable_lookup_workspace_bytes(uint64_t nq);
int seedtable_lookup(const uint64_t* qkey, uint64_t nq, const uint64_t* d_nq, int k, int bucket_bits,
                     const uint64_t* offsets, const uint32_t* fp, const uint64_t* pos_tab,
                     uint64_t* hit_off, uint64_t* hit_pos, uint64_t hit_cap, uint64_t* d_total,
                     void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MZSLSUM_H */
