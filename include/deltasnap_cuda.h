/*
 * deltasnap_cuda.h -- C ABI of the B200 (sm_100a) checkpoint hot path.
 *
 * Drop-in boundary for the reference package `deltasnap` (Check-N-Run,
 * arXiv 2010.08679; /root/reference/pkg/src/deltasnap).  The reference has no
 * FFI: its boundary is the Python API.  Each entry point below replaces the
 * numpy body of one reference function, cited as file:line.  The Python
 * package paper_2010_08679_b200 binds these with ctypes and
 * keeps the reference names, argument meaning and exceptions.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All array pointers are DEVICE pointers
 *    unless the name ends in _host.  `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).  Calls are asynchronous on
 *    `stream` and allocate nothing; scratch comes from a caller workspace
 *    sized by the matching *_workspace_size call.
 *  - Synchronous argument errors are returned as a ds_status.  Data
 *    dependent errors (out-of-range ids, NaN/Inf rows, bad padding) are
 *    OR-ed into a caller-owned device flag word (DS_FLAG_*) that the host
 *    shim reads at its next synchronisation point and raises as the
 *    reference exception.
 *  - Re-entrant: no global mutable state; one stream per caller.
 *
 * Bitmaps are uint32 little-endian words, bit r of a table at word r>>5,
 * bit r&31: byte-identical to the reference's uint8[(rows+7)//8] with bit r
 * at byte r>>3, bit r&7 (tracker.py:25,36).
 *
 * A "table set" is a concatenation of tables inside one word buffer:
 * table t owns words [word_off[t], word_off[t+1]) and rows [0, rows[t]).
 */
#ifndef DELTASNAP_CUDA_H
#define DELTASNAP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DS_API __attribute__((visibility("default")))
#else
#define DS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; 1-6 map 1:1 onto deltasnap/errors.py:4-41. */
typedef enum {
    DS_OK = 0,
    DS_ERR_CONFIG = 1,    /* ConfigError     (errors.py:7-8)   */
    DS_ERR_DATA = 2,      /* DataError       (errors.py:11-12) */
    DS_ERR_SHAPE = 3,     /* ShapeError      (errors.py:15-16) */
    DS_ERR_BOUNDS = 4,    /* BoundsError     (errors.py:19-20) */
    DS_ERR_FORMAT = 5,    /* FormatError     (errors.py:23-24) */
    DS_ERR_INTEGRITY = 6, /* IntegrityError  (errors.py:27-28) */
    DS_ERR_CUDA = 7,      /* CUDA runtime failure (launch/config) */
    DS_ERR_ARG = 8        /* invalid pointer/size argument        */
} ds_status;

/* Device flag bits (data-dependent errors, raised at the next sync). */
#define DS_FLAG_BOUNDS 0x1u    /* mark: id < 0 or >= rows          -> BoundsError    */
#define DS_FLAG_DATA 0x2u      /* NaN/Inf element in a coded row   -> DataError      */
#define DS_FLAG_FORMAT 0x4u    /* nonzero padding bits / bad code  -> FormatError    */
#define DS_FLAG_INTEGRITY 0x8u /* restore row id out of range      -> IntegrityError */
#define DS_FLAG_CAPACITY 0x10u /* output / staging buffer too small -> ValueError    */
#define DS_FLAG_TIMEOUT 0x20u  /* peer count exchange: a rank never published     */

/* Library identity / diagnostics. */
DS_API const char *ds_version(void);
DS_API const char *ds_last_error(void); /* thread-local text of the last non-OK status */
DS_API int ds_device_sm_count(int device);
/* Process-wide HBM fetch size of an L2 miss on the current device (0..128 B;
 * cudaLimitMaxL2FetchGranularity).  64 suits the dim-16 row gather. */
DS_API int ds_set_l2_fetch_granularity(int bytes);
DS_API int ds_get_l2_fetch_granularity(void);

/* ------------------------------------------------------------------ */
/* K1 / tracking (tracker.py:27-36, :91-92, :132-134)                   */
/* ------------------------------------------------------------------ */

/* DirtyBitmap.mark for a table set: idx[i] (int64) belongs to table
 * seg_table[s] for i in [seg_off[s], seg_off[s+1]).  Test-before-set
 * atomicOr into words.  Out-of-range ids set DS_FLAG_BOUNDS and are
 * skipped.  word_off/rows describe the table set (host arrays, at most
 * 64 tables per call); seg_table == NULL maps every segment to table 0. */
DS_API int ds_mark(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
            const int64_t *idx, const int64_t *seg_off_host, const int32_t *seg_table_host,
            int nseg, uint32_t *flags, void *stream);

/* Same with int32 ids (lookup streams of tables below 2^31 rows): halves the
 * index bytes K1 streams. */
DS_API int ds_mark_i32(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
                       const int32_t *idx, const int64_t *seg_off_host,
                       const int32_t *seg_table_host, int nseg, uint32_t *flags, void *stream);

/* Packed mixed-width lookup stream: segment s holds seg_count[s] ids of
 * seg_width[s] BITS starting at byte seg_byte_off[s] of `lookups` (16-byte
 * aligned, as is `lookups`), all marking table seg_table[s].  Widths 4, 8,
 * ..., 28: unsigned ids in an LSB-first bitstream (8 and 16 are plain u8 /
 * u16 arrays); 32 and 64: signed two's-complement int32 / int64.  Each packed
 * segment must be readable up to the next 16-byte boundary.  Sending each
 * table's ids at ceil(log2(rows)) bits (rounded up to a multiple of 4) cuts
 * the lookup bytes the end-to-end path moves over PCIe and K1 streams from
 * HBM.  Same bit semantics and DS_FLAG_BOUNDS behaviour as ds_mark. */
DS_API int ds_mark_packed(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
                          const void *lookups, const int64_t *seg_byte_off_host,
                          const int64_t *seg_count_host, const int32_t *seg_width_host,
                          const int32_t *seg_table_host, int nseg, uint32_t *flags, void *stream);

/* Single-table convenience form (DirtyBitmap.mark). */
DS_API int ds_mark_table(uint32_t *words, int64_t rows, const int64_t *idx, int64_t n, uint32_t *flags,
                  void *stream);

/* ------------------------------------------------------------------ */
/* K0 / bitmap maintenance (tracker.py:38-61, :120-130)                 */
/* ------------------------------------------------------------------ */

/* op 0: dst = a | b (merge_or); op 1: dst |= a (merge_in);
 * op 2: b |= a; a = 0 (reset_interval fold); op 3: a = 0; b = 0 (reset_baseline). */
DS_API int ds_bitmap_op(uint32_t *dst, uint32_t *a, uint32_t *b, int64_t nwords, int op, void *stream);

/* popcount of nwords words into *out (device int64). */
DS_API int ds_popcount(const uint32_t *words, int64_t nwords, int64_t *out, void *stream);

/* ------------------------------------------------------------------ */
/* K2 / compaction (tracker.py:54-58, :100-124)                          */
/* ------------------------------------------------------------------ */

/* Capture both scopes of a tracker in one pass.
 *   interval, baseline: table-set word buffers (same layout);
 *   word_off[ntables+1] and rows[ntables] (device);
 *   ids_int / ids_union: outputs (int64 row ids, per table ascending,
 *     tables concatenated in order), either may be NULL to skip a scope;
 *   counts[2*ntables+2] (device int64): counts[t] interval count of table t,
 *     counts[ntables+1+t] union count; counts[ntables] and counts[2*ntables+1]
 *     the totals;  offsets follow as exclusive prefix sums on the host side.
 *   fold: 0 none, 1 reset_interval (baseline |= interval; interval = 0)
 *     after reading, 2 reset_baseline (both cleared).
 * Workspace: ds_capture_workspace_size(total_words), zero-filled before its
 * first use and not shared by concurrent calls (it holds a completion counter
 * that each call leaves at zero).  Tables whose word offsets are multiples of
 * 4 move with 16-byte loads and stores. */
DS_API size_t ds_capture_workspace_size(int64_t total_words, int ntables);
DS_API int ds_capture(uint32_t *interval, uint32_t *baseline, const int64_t *word_off_host,
               const int64_t *rows_host, int ntables, int64_t *ids_int, int64_t *ids_union,
               int64_t *counts, int fold, void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* K3 / writer (engine.py:118-189, quant.py:93-209,372-382,             */
/*              payload.py:68-104)                                       */
/* ------------------------------------------------------------------ */

/* One table of a shard payload, as seen by the writer. */
typedef struct {
    const float *values;  /* (rows, ld) float32, device */
    const float *aux;     /* (rows, ld) float32 or NULL */
    int64_t ld;           /* row stride in elements (>= dim) */
    int64_t rows;         /* table rows (full checkpoints write all of them) */
    int64_t row_base;     /* global id of local row 0 (row-sharded tables) */
    int64_t ids_off;      /* offset of this table's ids in the id buffer (incremental) */
    uint32_t table_id;
    uint32_t dim;
} ds_table_desc;

/* Shard-level parameters of a checkpoint. */
typedef struct {
    int bitwidth;       /* 2,3,4,8; 0 = fp32 section (mode 0, tag 32) */
    int incremental;    /* 1: records carry u64 row ids, rows from ids */
    int adaptive_bins;  /* 0: naive min/max ranges; else greedy num_bins */
    int adaptive_steps; /* floor(num_bins*ratio + 1e-9) (quant.py:186) */
    int write_headers;  /* 1: write the 24-byte CNR1 section headers */
    int aux;            /* 1: aux_flag set, aux rows appended (payload.py:102-103) */
    int ids_packed;     /* 1: table t's ids start at sum(counts[<t]) (capture's layout);
                           ds_table_desc.ids_off is then ignored */
    int ids_local;      /* 1: ids are table-local rows (capture output); the record
                           carries row_base + id */
    unsigned long long *stats; /* optional device counters (DS_STAT_*), may be NULL */
    const float *staged;       /* optional: rows already gathered by ds_stage_rows (record i
                                  of the packed id order at staged[i * dim]); the tables are
                                  then only used for bounds, row_base and dims */
    const struct ds_peer_exchange *exchange; /* NULL, or the row-sharded count exchange run
                                  inside this launch (below): CTA 0 publishes, the last
                                  CTA waits for every rank and writes exchange->out */
    int64_t staged_rows;       /* capacity of `staged` in rows: a larger dirty total sets
                                  DS_FLAG_CAPACITY and writes no records (like the payload
                                  capacity) instead of reading past the staging buffer */
} ds_ckpt_params;

/* Counters of the certified fast path (diagnostics). */
#define DS_STAT_EXACT_DECISIONS 0 /* greedy comparisons re-decided in exact f64 */
#define DS_STAT_EXACT_CODES 1     /* element codes recomputed in exact f64      */
#define DS_STAT_ROWS 2            /* rows coded                                 */
#define DS_STAT_COUNT 4

/* Payload layout for ntables tables: given per-table row counts (device,
 * counts[t]; full checkpoints pass NULL and use rows), computes on device
 *   sec_off[t]   byte offset of table t's section (header) in the payload,
 *   sec_off[ntables] total payload bytes,
 * and the tile schedule the writer uses.  Everything stays on device; the
 * whole call is ONE kernel launch (layout, records, exact fixups, error sum).
 * The workspace must be zero-filled before its first use and not be shared
 * by calls in flight at the same time (it holds a completion counter that
 * each call leaves at zero). */
DS_API size_t ds_writer_workspace_size(int ntables, int64_t max_rows, int64_t dim);
DS_API int ds_write_payload(const ds_table_desc *tables_host, int ntables, const ds_ckpt_params *p,
                     const int64_t *ids, const int64_t *counts, uint8_t *payload,
                     int64_t payload_capacity, int64_t *sec_off, double *err_sum,
                     uint32_t *flags, void *workspace, size_t workspace_bytes, void *stream);

/* Stall-window staging: gather the dirty rows named by
 * ids (table-local, packed per table in table order, counts[ntables] =
 * total, capture_into's layout) into staged[k * dim] so the writer can run
 * from the copy (ds_ckpt_params.staged) while training updates the tables.
 * max_rows is the staging capacity in rows; a larger total sets
 * DS_FLAG_CAPACITY (the total stays on the device). */
DS_API int ds_stage_rows(const ds_table_desc *tables_host, int ntables, const int64_t *ids,
                         const int64_t *counts, int64_t max_rows, float *staged, uint32_t *flags,
                         void *stream);

/* Upper bound of the payload bytes for the given row counts (host math). */
DS_API int64_t ds_record_size(int64_t dim, int bitwidth, int aux, int incremental);

/* ------------------------------------------------------------------ */
/* K4 / restore (engine.py:459-485, payload.py:60-65, quant.py:385-395) */
/* ------------------------------------------------------------------ */

/* Apply one section body (records only, header parsed on the host) to a
 * (local) table holding global rows [row_lo, row_hi):
 *   incremental: record row ids; ids outside [0, table_rows) set
 *     DS_FLAG_INTEGRITY; ids outside [row_lo, row_hi) are skipped (other
 *     rank's rows); applied rows also set their since-baseline bit
 *     (engine.py:476) in baseline_words (may be NULL);
 *   full: record i is global row i; only [row_lo, row_hi) is applied.
 * Nonzero padding bits set DS_FLAG_FORMAT. */
DS_API int ds_restore_section(const uint8_t *body, int64_t nrec, int64_t dim, int bitwidth, int aux,
                       int incremental, int64_t table_rows, int64_t row_lo, int64_t row_hi,
                       float *values, int64_t ld, float *aux_values, uint32_t *baseline_words,
                       uint32_t *flags, void *stream);

/* One section of a payload for ds_restore_payload. */
typedef struct {
    int64_t body_off;      /* byte offset of the section's first record in `payload` */
    int64_t nrec;          /* records in the section (row_count) */
    float *values;         /* the (local) table: rows [row_lo, row_hi) of table_rows */
    float *aux_values;     /* may be NULL */
    uint32_t *baseline;    /* since-baseline words of the table (may be NULL) */
    int64_t ld;            /* row stride of values / aux_values (floats) */
    int64_t table_rows;    /* global rows of the table */
    int64_t row_lo, row_hi;
} ds_restore_sec;

/* Every section of one payload in ONE launch (same semantics as
 * ds_restore_section per section).  Sections share dim, bitwidth, aux and
 * kind; flags[k] receives section k's DS_FLAG_* bits (so the host raises the
 * first failing section's error, engine.py:459-472).  At most 64 sections. */
DS_API int ds_restore_payload(const uint8_t *payload, const ds_restore_sec *secs_host, int nsec,
                              int64_t dim, int bitwidth, int aux, int incremental, uint32_t *flags,
                              void *stream);

/* ------------------------------------------------------------------ */
/* Training step with tracking folded in (sim.py:140-155)  */
/* ------------------------------------------------------------------ */

typedef struct {
    float *values;     /* [rows, ld] fp32 */
    float *aux;        /* may be NULL: no aux update */
    uint32_t *words;   /* the table's interval bitmap words (may be NULL: no tracking) */
    int64_t ld;
    int64_t rows;
} ds_train_table;

/* apply_batch for nbatches batches in order: for every table t and batch b,
 * values[idx] += delta and aux[idx] += delta * delta with np.add.at's
 * semantics (every index in array order: bit-identical float sums) and the
 * rows' dirty bits set.  ids/deltas are table-major, then batch order:
 * segment t * nbatches + b = [seg_off[.], seg_off[. + 1]) of idx (device
 * int64) and of delta (device float [*, dim]); at most 4096 ids per
 * segment.  Out-of-range ids set DS_FLAG_BOUNDS and are skipped. */
DS_API int ds_train_apply(const ds_train_table *tables_host, int ntables, int nbatches, int64_t dim,
                          const int64_t *idx, const float *delta, const int64_t *seg_off,
                          uint32_t *flags, void *stream);

/* The same update for a whole interval at once: rows (device int64) holds
 * every table's ids stably sorted by row (table t at sorted positions
 * [table_off[t], table_off[t+1]), host array), order[i] the position of the
 * i-th sorted id in delta ([n, dim] device floats, batch order).  Each row's
 * updates are then one run in np.add.at order; a warp applies a run with
 * lanes over elements.  Same results as ds_train_apply over the batches. */
DS_API int ds_train_apply_sorted(const ds_train_table *tables_host, int ntables,
                                 const int64_t *table_off_host, int64_t dim, const int64_t *rows,
                                 const int64_t *order, const float *delta, uint32_t *flags,
                                 void *stream);

/* The same update for a whole interval with the in-tree stable radix sort
 * (ds_sort_pairs_u32): idx (device int64, table t's lookups at positions
 * [table_off[t], table_off[t+1]) of a host offset array, batch order inside
 * a table) and delta ([n, dim]); the (table, row) pairs are stably sorted,
 * each row's run is applied in np.add.at order by one warp and its dirty
 * bit set.  Out-of-range ids set DS_FLAG_BOUNDS and are skipped.  Needs
 * ceil(log2(ntables)) + ceil(log2(max_rows + 1)) <= 32 and a workspace of
 * ds_train_interval_workspace_size(n) + ds_train_interval_delta_bytes(n, dim)
 * bytes (the sort, then the deltas gathered into sorted order). */
DS_API size_t ds_train_interval_workspace_size(int64_t n);
DS_API size_t ds_train_interval_delta_bytes(int64_t n, int64_t dim);
DS_API int ds_train_apply_interval(const ds_train_table *tables_host, int ntables,
                                   const int64_t *table_off_host, int64_t dim, const int64_t *idx,
                                   const float *delta, void *workspace, size_t workspace_bytes,
                                   uint32_t *flags, void *stream);

/* Stable LSD radix sort (8-bit digits) of n (u32 key, u32 value) pairs by the
 * low key_bits bits of the key; inputs intact, outputs must not alias them;
 * workspace of ds_sort_workspace_size(n) bytes. */
DS_API size_t ds_sort_workspace_size(int64_t n);
DS_API int ds_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                             uint32_t *vals_out, int64_t n, int key_bits, void *workspace,
                             size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* Payload checksum (store.py:46-47 checksum())      */
/* ------------------------------------------------------------------ */

/* CRC-32 (IEEE, = zlib.crc32) of n device bytes into *out (device uint32),
 * asynchronously, one launch: 32 KB chunks per CTA; each chunk shifts its CRC
 * by the bytes after it with precomputed GF(2) operators and xors it into
 * *out.  The workspace argument is reserved (may be NULL;
 * ds_crc32_workspace_size returns a small constant). */
DS_API size_t ds_crc32_workspace_size(int64_t n);
DS_API int ds_crc32(const uint8_t *data, int64_t n, uint32_t *out, void *workspace,
                    size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* Row-sharded count exchange over NVLink peer memory     */
/* ------------------------------------------------------------------ */

/* The one exchange of the row-sharded checkpoint: every rank's int64
 * dirty counts (per table, then their total) to every rank, so each knows
 * where its records land in the shard payload.  A collective beside the
 * writer costs more than its bytes (its kernel holds SMs that the writer's
 * resident CTAs need), so the exchange runs inside the writer's launch
 * (ds_ckpt_params.exchange): CTA 0 stores this rank's counts into every
 * peer's exchange buffer over NVLink (CUDA IPC mappings) and releases the
 * slot's epoch flag at system scope; the last CTA to finish waits (acquire)
 * until every rank's flag shows the epoch -- normally already true, the
 * peers published when their writers started -- and copies the slots out.
 *
 * Exchange buffer (ds_peer_buffer_size(world, ntables + 1) bytes, own
 * cudaMalloc, zero-filled): flags uint32[2][world], then int64
 * slots[2][world][ntables + 1]; epoch e uses parity e & 1.  The epoch must
 * grow by one per exchange starting at 1, and every rank runs the same
 * sequence of exchanges; a rank publishes e + 1 only after its own wait for
 * e (stream order gives that), so no slot is overwritten before every rank
 * has read it.  A rank missing after timeout_ns sets DS_FLAG_TIMEOUT in
 * *flags and the wait gives up.
 *   ds_peer_alloc   cudaMalloc + zero + cudaIpcGetMemHandle (64-byte handle out)
 *   ds_peer_open    cudaIpcOpenMemHandle of a peer's handle (lazy peer access)
 *   ds_peer_close / ds_peer_free */
#define DS_PEER_MAX 64
typedef struct ds_peer_exchange {
    void *peers[DS_PEER_MAX]; /* every rank's exchange buffer, this rank's included */
    int64_t *out;             /* device int64[world * (ntables + 1)], rank-major */
    uint32_t *flags;          /* device flag word for DS_FLAG_TIMEOUT */
    int64_t timeout_ns;
    int world, rank;
    uint32_t epoch;
} ds_peer_exchange;
DS_API size_t ds_peer_buffer_size(int world, int n);
DS_API int ds_peer_alloc(size_t bytes, void **ptr, uint8_t *handle64);
DS_API int ds_peer_open(const uint8_t *handle64, void **ptr);
DS_API int ds_peer_close(void *ptr);
DS_API int ds_peer_free(void *ptr);

/* ------------------------------------------------------------------ */
/* Row-matrix codec entry points (quant.py API mirror)                  */
/* ------------------------------------------------------------------ */

/* quantize_rows (quant.py:93-106): codes[n,d] from x[n,d] and f32 ranges. */
DS_API int ds_quantize_rows(const float *x, int64_t n, int64_t d, const float *mins, const float *maxs,
                     int bitwidth, uint8_t *codes, void *stream);
/* dequantize_rows (quant.py:109-115); codes >= 2^N set DS_FLAG_FORMAT. */
DS_API int ds_dequantize_rows(const uint8_t *codes, int64_t n, int64_t d, const float *mins,
                       const float *maxs, int bitwidth, float *out, uint32_t *flags,
                       void *stream);
/* reconstruction_errors (quant.py:134-138), exact numpy order, f64 out. */
DS_API int ds_reconstruction_errors(const float *x, int64_t n, int64_t d, const float *mins,
                             const float *maxs, int bitwidth, double *out, void *stream);
/* adaptive_params_rows (quant.py:160-209): greedy ranges (NaN/Inf flag). */
DS_API int ds_adaptive_params_rows(const float *x, int64_t n, int64_t d, int bitwidth, int num_bins,
                            int steps, float *mins, float *maxs, uint32_t *flags,
                            unsigned long long *stats, void *stream);
/* naive x.min(axis=1) / x.max(axis=1). */
DS_API int ds_row_minmax(const float *x, int64_t n, int64_t d, float *mins, float *maxs, void *stream);
/* pack_code_rows / unpack_code_rows (quant.py:376-395). */
DS_API int ds_pack_code_rows(const uint8_t *codes, int64_t n, int64_t d, int bitwidth, uint8_t *out,
                      uint32_t *flags, void *stream);
DS_API int ds_unpack_code_rows(const uint8_t *packed, int64_t n, int64_t d, int bitwidth, uint8_t *out,
                        uint32_t *flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DELTASNAP_CUDA_H */
