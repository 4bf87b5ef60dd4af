/*
 * alto_b200.h — C ABI of the B200-native ALTO hot path (libalto_b200.so).
 *
 * The reference (arXiv 2102.10245, package `altotensor`, /root/reference/pkg)
 * is pure Python: its boundary is the Python API in
 * pkg/src/altotensor/__init__.py:9-92, not an FFI.  Every entry point below
 * replaces the arithmetic of one reference function (cited per function); the
 * Python package paper_2102_10245_b200 binds them with ctypes and keeps the
 * reference signatures on top.
 *
 * Conventions
 *   - extern "C"; plain pointers, element counts, and a cudaStream_t passed as
 *     `void*` (NULL = legacy default stream).  No torch types.
 *   - All data pointers are DEVICE pointers unless the name says `host`.
 *   - The caller owns every buffer.  Scratch memory is passed in as a
 *     caller-allocated workspace whose size comes from a *_workspace_bytes()
 *     query.  The library never allocates or frees caller memory.
 *   - Calls are stream-ordered and asynchronous unless documented otherwise.
 *   - Return status: ALTO_OK, or an ALTO_E* code; alto_last_error() returns a
 *     thread-local message for the last failing call.
 *   - Keys ("indices" in the reference) are stored as n_words little-endian
 *     uint64 per element, least-significant word first, array-of-structs
 *     ((nnz, n_words) row-major), exactly like pkg/src/altotensor/layout.py:151.
 */
#ifndef ALTO_B200_H
#define ALTO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALTO_MAX_ORDER 8
#define ALTO_MAX_BITS 128

enum alto_status {
  ALTO_OK = 0,
  ALTO_EINVAL = 1,     /* invalid argument -> Python ValueError            */
  ALTO_ECUDA = 2,      /* CUDA runtime error                               */
  ALTO_EUNSUPPORTED = 3,
  ALTO_ENCCL = 4,
  ALTO_ESINGULAR = 5   /* normal equations singular -> np.linalg.LinAlgError */
};

enum alto_dtype { ALTO_F32 = 0, ALTO_F64 = 1, ALTO_I64 = 2 /* fixed-point MTTKRP output */ };

/* Bit layout of the linearized index (pkg/src/altotensor/layout.py:38-71).
 * Filled on the host from AltoLayout.positions; pos[n][g] is the key bit
 * holding bit g of mode n. */
typedef struct alto_layout {
  int32_t order;                     /* N                                   */
  int32_t n_words;                   /* 1 (width 64) or 2 (width 128)       */
  int32_t total_bits;                /* sum of bits[]                       */
  int32_t width;                     /* 64 or 128                           */
  int64_t dims[ALTO_MAX_ORDER];
  int32_t bits[ALTO_MAX_ORDER];
  uint8_t pos[ALTO_MAX_ORDER][64];
} alto_layout;

const char* alto_last_error(void);
int alto_version(void);

/* Size in bytes of the device-resident encode/decode tables for a layout
 * (byte-indexed deposit tables per mode, byte-indexed extract tables per key
 * byte).  alto_build_tables fills a caller-allocated device buffer of that
 * size (synchronous host->device copy of host-computed tables). */
size_t alto_tables_bytes(const alto_layout* lay);
int alto_build_tables(const alto_layout* lay, void* d_tables, void* stream);

/* K1 — linearize_array (layout.py:148-160, range check layout.py:135-145).
 * coords: (M, order) int64 row-major.  keys: (M, n_words) uint64.
 * *d_bad (device int64, caller-zeroed to -1 beforehand is NOT required: the
 * call resets it) receives the lowest row index holding an out-of-range
 * coordinate, or -1. */
int alto_linearize(const alto_layout* lay, const void* d_tables,
                   const int64_t* coords, int64_t m, uint64_t* keys,
                   int64_t* d_bad, void* stream);

/* K4 — extract_mode_array / delinearize_array (layout.py:163-182).
 * mode >= 0: out is (M,) int64 for that mode; mode == -1: out is (M, order).
 * Bits above total_bits (flags) are ignored (layout.py:125). */
int alto_delinearize(const alto_layout* lay, const void* d_tables,
                     const uint64_t* keys, int64_t m, int32_t mode,
                     int64_t* out, void* stream);

/* K2 — stable LSD radix sort of (keys, payload) over key bits
 * [0, total_bits): replaces np.lexsort + co-permutation (format.py:79-82,
 * :94-97).  payload_bytes in {0, 4, 8}.  Result lands in keys/payload. */
size_t alto_sort_workspace_bytes(int64_t m, int32_t n_words, int32_t payload_bytes);
int alto_sort_pairs(uint64_t* keys, void* payload, int64_t m, int32_t n_words,
                    int32_t payload_bytes, int32_t total_bits, void* workspace,
                    size_t workspace_bytes, void* stream);

/* K3 — duplicate check (format.py:98-99): *d_first = lowest i>0 with
 * key[i] == key[i-1] over all words, or -1. */
int alto_find_duplicate(const uint64_t* keys, int64_t m, int32_t n_words,
                        int64_t* d_first, void* stream);

/* K5 — partition (format.py:127-154).  Equal-nnz ranges, larger first
 * (format.py:136-140).  intervals: (count, order, 2) int64, per-partition
 * min/max of every mode, (0,-1) for empty partitions (format.py:146-149).
 * spans: (count, 2, n_words) uint64 first/last key of each partition (empty
 * partitions left untouched). */
int alto_partition(const alto_layout* lay, const void* d_tables,
                   const uint64_t* keys, int64_t m, int64_t count,
                   int64_t* intervals, uint64_t* spans, void* stream);

/* K6 — apply_boundary_flags (format.py:257-285): out_keys = keys with bit
 * flag_bit set on every element whose `mode` coordinate lies in one of its
 * partition's overlap ranges.  Overlaps in CSR form: partition l owns ranges
 * [ov_ptr[l], ov_ptr[l+1]) of (ov_lo[], ov_hi[]), ascending and disjoint.
 * d_offsets: the plan's partition offsets (count+1, device), any
 * non-decreasing split of [0, m) as the reference accepts; NULL = the
 * equal-size partition of `partition` (format.py:136-140). */
int alto_apply_flags(const alto_layout* lay, const void* d_tables,
                     const uint64_t* keys, int64_t m, int64_t count,
                     int32_t mode, int32_t flag_bit, const int64_t* ov_ptr,
                     const int64_t* ov_lo, const int64_t* ov_hi, const int64_t* d_offsets,
                     uint64_t* out_keys, void* stream);
/* read_flags / clear_flags (format.py:288-299). */
int alto_read_flags(const uint64_t* keys, int64_t m, int32_t n_words,
                    int32_t flag_bit, uint8_t* out, void* stream);
int alto_clear_flags(const uint64_t* keys, int64_t m, int32_t n_words,
                     int32_t flag_bit, uint64_t* out_keys, void* stream);

/* ---- MTTKRP (mttkrp.py) ------------------------------------------------ */

/* Per-mode device plan for the streaming kernel: the sorted stream is cut
 * into tiles of `tile` elements; for each tile the mode-`mode` interval is
 * recorded (tile_lo/tile_hi, int32 each, (ntiles,)). */
int64_t alto_mttkrp_ntiles(int64_t m, int32_t tile);
int alto_tile_intervals(const alto_layout* lay, const void* d_tables,
                        const uint64_t* keys, int64_t m, int32_t tile,
                        int32_t* tile_lo /* (ntiles, order) */,
                        int32_t* tile_hi /* (ntiles, order) */, void* stream);

typedef struct alto_mttkrp_args {
  const alto_layout* lay;
  const void* d_tables;
  const uint64_t* keys;          /* (M, n_words) */
  const void* values;            /* (M,) value_dtype */
  int64_t m;
  int32_t mode;
  int32_t rank;
  int32_t value_dtype;           /* ALTO_F32 / ALTO_F64 */
  int32_t factor_dtype;          /* ALTO_F32 / ALTO_F64 */
  const void* factors[ALTO_MAX_ORDER]; /* (I_n, rank) row-major, factor_dtype */
  void* out;                     /* (I_mode, rank) row-major, out_dtype     */
  int32_t out_dtype;             /* ALTO_F64 (reference dtype), ALTO_F32, or
                                    ALTO_I64: deterministic fixed point,
                                    out = round(value * *fixed_scale)
                                    (streaming kernel only)                 */
  int32_t tile;                  /* elements per tile (multiple of 256, <= 1024) */
  int32_t zero_out;              /* 1: out is zeroed first (stream-ordered) */
  /* Hot-row plan (optional, from alto_hot_plan): rows with many elements
   * are touched by nearly every tile, and same-address float64 REDs from all
   * tiles serialise in one L2 slice.  Their per-tile partials go instead to
   * `hot_copies` replicated buffers (tile % hot_copies), reduced into `out`
   * by a second kernel in a fixed order.  hot_slot: (I_mode,) int32, slot or
   * -1; hot_rows: (n_hot,) int32; hot_buf: hot_copies * n_hot * rank
   * elements of out_dtype, zero on entry and left zero on exit (copies are
   * summed in float64). */
  const int32_t* hot_slot;
  const int32_t* hot_rows;
  int32_t n_hot;
  int32_t hot_copies;
  void* hot_buf;
  int32_t flags;                 /* ALTO_STREAM_* tuning switches (0 = default) */
  /* Optional per-tensor / per-mode plan (BLCO-style): `packed` holds every
   * key bit-permuted so each mode's bits are contiguous (same bits, same
   * element order; alto_pack_keys) and `pos` each element's row-sorted slot
   * in its 128-element sub-tile for this mode (alto_subtile_order).  With
   * both set, the specialised kernels skip the byte-table decode and the
   * in-tile sort. */
  const uint64_t* packed;
  const uint8_t* pos;
  const double* fixed_scale;     /* device scalar for ALTO_I64 output (alto_fixed_scale) */
  /* Per-mode stream (built by alto_mode_stream for this mode): keys, values
   * and its tile length.  When set, the mode-stream kernel runs (orders 3-5,
   * ranks 16/32, max_n I_n*rank*sizeof(factor) < 2^32; else ALTO_EUNSUPPORTED)
   * and, for ALTO_F32 output, hot_buf holds float64 copies. */
  const uint64_t* mkeys;
  const void* mvals;
  int32_t mtile;
  /* Per-row copy counts (alto_hot_copies): with hot_base set, hot_slot holds
   * hot_code (dim int32: (first copy << 5) | log2(copies), or -1), hot_base
   * the per-slot first copy (n_hot+1), and hot_buf hot_base[n_hot] * rank
   * elements of out_dtype (zero on entry, left zero); hot_copies is ignored.
   * Required with a mode stream (mkeys); optional for the ALTO-order kernels
   * (plan built with tile 128 and flags 0). */
  const int32_t* hot_base;
  int32_t mrr;                   /* mode stream built with ALTO_MS_ROUND_ROBIN (1) or ALTO_MS_BLOCKED (2) */
  /* Paired input modes (mode stream, or packed + pos; float32 values and factors, rank
   * 16, orders 4-5): input modes pair_a[i], pair_b[i] (i < n_pairs, disjoint,
   * not `mode`) are gathered together as one row of pair_tab[i], the
   * row-wise product table of their factors (alto_krp_pair: row
   * ia * I_b + ib), so one gather replaces two.  I_a * I_b * rank * 4 must
   * stay below 2^32 bytes; ALTO_EUNSUPPORTED otherwise. */
  int32_t n_pairs;
  int32_t pair_a[2];
  int32_t pair_b[2];
  const void* pair_tab[2];
  /* Delta mode stream (alto_mode_stream with ALTO_MS_DELTA): the row of each
   * lane group's first element (ntiles * 8 int32); NULL for plain streams. */
  const int32_t* mbase;
  /* L2 residency of gathered factor rows (mode-stream kernel, float32
   * factors): the first l2_hot_bytes[n] bytes of mode n's factor — its most
   * referenced rows when rows are numbered by popularity — are gathered with
   * an L2 evict_last policy and the rest of it with evict_first, so the
   * re-used head stays cached while the stream, the tail rows and the output
   * rows pass through (0 = default policy). */
  uint32_t l2_hot_bytes[ALTO_MAX_ORDER];
} alto_mttkrp_args;

/* Row-wise (Khatri-Rao) product table of two factors for paired input modes:
 * out[ia * rows_b + ib][r] = fa[ia][r] * fb[ib][r], (rows_a * rows_b, rank)
 * row-major, dtype ALTO_F32 or ALTO_F64. */
int alto_krp_pair(const void* fa, int64_t rows_a, const void* fb, int64_t rows_b, int32_t rank, int32_t dtype,
                  void* out, void* stream);

/* Deterministic MTTKRP support (ALTO_I64 output).  alto_sumabs / alto_absmax:
 * float64 sum of |x| / max |x| (fixed-order two-stage reductions, `ws` from
 * alto_cpd_workspace_bytes).  alto_fixed_scale: scale = 2^(61 - ceil(log2 B))
 * for B = product of the nterms device scalars (a bound on every partial
 * sum: sum|v| * prod max|F|), so int64 partial sums cannot overflow.
 * alto_fixed_to_float: out = in / scale as float32 or float64. */
int alto_sumabs(const void* x, int32_t dtype, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream);
int alto_absmax(const void* x, int32_t dtype, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream);
int alto_fixed_scale(const double* terms, int32_t nterms, double* scale, void* stream);
int alto_fixed_to_float(const int64_t* in, const double* scale, void* out, int32_t out_dtype, int64_t n,
                        void* stream);

/* Workspace of alto_hot_rows (a sort of the mode's dim row counts). */
size_t alto_topk_rows_workspace_bytes(int64_t dim);
/* Hot-row plan by rank: the (up to) k rows with the most elements, keeping
 * only rows with more than min_count; slots 0..*d_count-1 in descending
 * count order (rows -1 padded; slot_map dim int32: slot or -1); workspace
 * of alto_topk_rows_workspace_bytes(dim) bytes. */
int alto_hot_rows(const int64_t* row_ptr, int64_t dim, int32_t k, int64_t min_count, int32_t* rows,
                  int32_t* slot_map, int32_t* d_count, void* ws, size_t ws_bytes, void* stream);

/* Mode-contiguous re-encoding of sorted ALTO keys: packed[i] holds mode n's
 * coordinate in bits [sum_{m<n} b_m, +b_n) (same n_words as the keys). */
int alto_pack_keys(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m,
                   uint64_t* packed, void* stream);
/* Per-mode sub-tile order: pos[i] = slot of element i inside its 128-element
 * sub-tile after a stable counting sort by its `mode` coordinate (identity
 * for sub-tiles whose rows span more than 512). */
int alto_subtile_order(const alto_layout* lay, const uint64_t* packed, int64_t m, int32_t mode, uint8_t* pos,
                       void* stream);

/* Per-mode stream of the MTTKRP (alto_mstream.cuh), built once per tensor
 * and mode like the reference's per-mode plans / flagged key copies
 * (_make_backend, cpd.py:149-181): the sorted ALTO stream cut into tiles of
 * `tile` consecutive elements (contiguous key ranges), each tile stably
 * sorted by its `mode` coordinate and split into 8 slices of tile/8 elements
 * stored interleaved (sorted position p of tile t at t*tile + (p % (tile/8))*8
 * + p / (tile/8)).  Keys hold the element's coordinates re-packed for the
 * mode — input modes ascending, then `mode`, from bit 0, no field straddling
 * a 64-bit word — and, when hot_slot (dim int32, slot or -1) is given, bit
 * 64*n_words-1 set on elements of hot rows.  Returns ALTO_EUNSUPPORTED when
 * that layout does not fit below bit 64*n_words-1.  skeys / svals
 * hold ceil(m/tile)*tile elements (the tail is zero padding).  value_dtype
 * ALTO_F32 or ALTO_F64; tile a multiple of 128 with m / tile < 2^31. */
size_t alto_mode_stream_workspace_bytes(int64_t m);
#define ALTO_MS_ROW_MAJOR 1 /* flags: sort the whole stream by the mode's coordinate (stable: ALTO order
                               within a row), not tile by tile */
#define ALTO_MS_ROUND_ROBIN 4 /* flags: lane group s of a tile takes sorted positions s, s+8, ... (stream
                                 stored in sorted order) instead of a contiguous slice */
#define ALTO_MS_DELTA 8 /* flags (row-major only): one 64-bit key word per element — the input
                           coordinates plus the row increment from the previous element of the same
                           lane group (base_rows[tile * 8 + group] holds each group's first row);
                           ALTO_EUNSUPPORTED if fewer than 8 increment bits are left, and
                           *d_overflow (device int32, zeroed by the call) is set when an increment
                           does not fit (the caller then builds a plain stream) */
#define ALTO_MS_BLOCKED 16 /* flags (row-major only): a warp step covers groups*u consecutive sorted
                              elements; lane group s takes elements s, s+groups, ... of the step and
                              its u elements are stored contiguously (sorted element k*groups+s of a
                              step at s*u+k); delta increments refer to the element `groups`
                              positions earlier and base_rows holds ntiles * groups rows.  u and
                              groups come from alto_mstream_block, passed as ALTO_MS_BLOCK(u, groups) */
#define ALTO_MS_BLOCK(u, groups) (ALTO_MS_BLOCKED | ((u) << 8) | ((groups) << 12))
/* Step shape of the blocked mode-stream kernel for a tensor order, rank,
 * value dtype and number of paired input modes: *u elements per lane group
 * and *groups lane groups per warp (ALTO_EUNSUPPORTED when no kernel covers
 * the shape: float32 values, orders 3-5, ranks 16/32). */
int alto_mstream_block(int32_t order, int32_t rank, int32_t value_dtype, int32_t n_pairs, int32_t* u,
                       int32_t* groups);
int alto_mode_stream(const alto_layout* lay, const uint64_t* packed, const void* values, int32_t value_dtype,
                     int64_t m, int32_t mode, int32_t tile, int32_t flags, const int32_t* hot_slot,
                     uint64_t* skeys, void* svals, int32_t* base_rows, int32_t* d_overflow,
                     void* ws, size_t ws_bytes, void* stream);

/* Hot-row copy plan of the mode-stream kernel: hot row s (hot_rows[s],
 * from alto_hot_rows) gets copies = 2^lg replicated partial rows, lg the
 * smallest with 2^lg * bound >= estimated merges (count/(tile/8) + 2 for a
 * row-major stream, flags & ALTO_MS_ROW_MAJOR; else min(count, tiles) +
 * count/(tile/8)), lg <= max_lg; copies are laid out slot by slot:
 * hot_base[s] = first copy (n_hot+1 entries), hot_code[row] = (hot_base << 5)
 * | lg.  hot_code must be pre-filled with -1 for the other rows. */
int alto_hot_copies(const int64_t* row_ptr, const int32_t* hot_rows, int32_t n_hot, int64_t m, int32_t tile,
                    int32_t flags, int32_t bound, int32_t max_lg, int32_t* hot_code, int32_t* hot_base,
                    void* stream);

/* COO coalesce on the device (coo.py:97-114): rows sorted lexicographically
 * with mode 0 as the primary key (stable), duplicates summed in float64 in
 * that order from 0.0 (bitwise equal to the reference's np.bincount).
 * coords (m, order) int64 row-major, values (m,) float64; bits[n] =
 * bits_for(I_n) (host array, sum <= 128); out_coords / out_values hold up to
 * m rows; *d_count (device int64) receives the number of distinct rows. */
size_t alto_coalesce_workspace_bytes(int64_t m, int32_t n_words);
int alto_coalesce(const int64_t* coords, const double* values, int64_t m, int32_t order, const int32_t* bits,
                  int64_t* out_coords, double* out_values, int64_t* d_count, void* ws, size_t ws_bytes,
                  void* stream);

/* Streaming-kernel switches (alto_mttkrp_args.flags). */
#define ALTO_STREAM_GENERIC 128  /* bypass the specialised (order 3-5, rank 16/32) kernels */
#define ALTO_STREAM_MS_L2_NORMAL 2048 /* tuning: mode-stream loads without the L2 evict_first policy */

/* Build the hot-row plan of one mode from its row pointer (alto_row_index):
 * rows with more than `tau` elements get slots (at most hmax);
 * *d_nhot (device int32) receives the slot count. */
int alto_hot_plan(const int64_t* row_ptr, int64_t dim, int64_t tau, int32_t hmax,
                  int32_t* hot_slot, int32_t* hot_rows, int32_t* d_nhot, void* stream);

/* K7/K8 — streaming ALTO MTTKRP (mttkrp.py:80-105 contributions,
 * :132-224 conflict resolution).  Each CTA streams tiles of the sorted
 * stream; a tile whose output-mode interval is short is counting-sorted by
 * output row on chip (its interval buffer), its contributions reduced in
 * registers per row segment and merged with one atomic update per (tile,
 * row) — the Buffered scheme at CTA granularity; a wide tile merges per
 * element run (the Atomic scheme).  Hot rows use the replicated buffers of
 * the hot plan.  Not bitwise reproducible (atomics), like the reference's
 * atomic path with several workers. */
int alto_mttkrp(const alto_mttkrp_args* a, void* stream);

/* Largest decoded coordinate of every mode (flag bits ignored), out_max
 * (order,) device uint64.  Used to validate container files before a
 * corrupt key can reach a kernel as an out-of-range row. */
int alto_coord_max(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m,
                   uint64_t* out_max, void* stream);

/* ---- K8/K9: slice interval buffers + deterministic pull ------------------
 * The Buffered scheme of the reference (_par_buffered, mttkrp.py:132-175:
 * per-partition interval buffers, then a pull in ascending partition order)
 * and its Atomic scheme (_par_atomic, mttkrp.py:178-224: flagged elements
 * merge with atomics, unflagged ones store directly) over the mode's
 * row-major stream (alto_mode_stream with ALTO_MS_ROW_MAJOR, contiguous
 * slices).  A slice (T/8 consecutive stream positions) is a partition whose
 * output interval is contiguous: rows inside it are owned (plain stores),
 * only its first/last row can be shared with a neighbouring slice (the
 * boundary-flag rows of apply_boundary_flags, format.py:257-285).
 *   atomic = 0 (Buffered): shared-row partials go to the slice's record
 *     slots (slice_rec: per slice (first-run slot, last-run slot), -1 =
 *     owned), then the pull sums each shared row's records in float64 in
 *     slot order with a fixed two-level shape (chunks of 64 records:
 *     chunk_off/chunk_seg/seg_chunk_off; multi-chunk segments `mseg` sum their
 *     float64 chunk partials `part`): bitwise reproducible.
 *   atomic = 1: shared rows (seg_row) are zeroed, then merged with RED.
 * Empty rows are zero-filled by the stage (no memset).  Orders 3-5, ranks
 * 16/32 (8/64: float32, Buffered), value/factor/out dtypes f32/f32/f32,
 * f32/f32/f64, f64/f64/f64, f32/f64/f64 (float32 values, float64 factors:
 * computed in float64).  Returns ALTO_EUNSUPPORTED for other shapes. */
typedef struct alto_pull_args {
  const alto_layout* lay;
  const uint64_t* mkeys;        /* mode stream keys (alto_mode_stream)       */
  const void* mvals;            /* mode stream values                        */
  int32_t value_dtype;
  int32_t tile;                 /* stream tile T (slices of T/8)             */
  int64_t m;
  int32_t mode;
  int32_t rank;
  int32_t factor_dtype;
  int32_t out_dtype;
  int32_t atomic;
  int32_t pad_;
  const void* factors[ALTO_MAX_ORDER];
  void* out;                    /* (I_mode, rank), fully written             */
  const int32_t* slice_rec;     /* (nslices, 2)                              */
  void* rec;                    /* (n_rec, rank) in the factor dtype         */
  int64_t n_seg;                /* shared rows                               */
  const int32_t* seg_row;       /* (n_seg,)                                  */
  int64_t n_chunks;
  const int64_t* chunk_off;     /* (n_chunks+1,) record offsets              */
  const int32_t* chunk_seg;     /* (n_chunks,)                               */
  const int64_t* seg_chunk_off; /* (n_seg+1,)                                */
  int64_t n_mseg;
  const int32_t* mseg;          /* (n_mseg,) segments with > 1 chunk         */
  double* part;                 /* (n_chunks, rank) float64 chunk partials   */
  const int32_t* slice_rows;    /* (nslices, 2) first / last row per slice (alto_pull_slice_rows) */
  const int32_t* mbase;         /* delta stream (ALTO_MS_DELTA): each slice's first row, else NULL */
  /* Paired input modes, as in alto_mttkrp_args (float32 values and factors,
   * rank 16, orders 4-5): pair_tab[i] = alto_krp_pair table of modes
   * pair_a[i], pair_b[i]; one gather replaces two. */
  int32_t n_pairs;
  int32_t pair_a[2];
  int32_t pair_b[2];
  const void* pair_tab[2];
} alto_pull_args;
int alto_mttkrp_pull(const alto_pull_args* a, void* stream);
/* Plan helper: first and last output row of every slice of a mode stream,
 * first_last (nslices, 2) int32; base = the delta stream's base rows (NULL
 * for a plain stream). */
int alto_pull_slice_rows(const alto_layout* lay, const uint64_t* mkeys, int64_t m, int32_t mode, int32_t tile,
                         const int32_t* base, int32_t* first_last, void* stream);

/* Exact-order engine (deterministic; bitwise equal to the reference for
 * float64 data): for mode `mode`, `row_perm` lists element indices sorted by
 * (mode coordinate, element index) and `row_ptr` (I_mode+1) delimits rows.
 * Partition boundaries `part_off` (count+1) split each row's sum, and the
 * per-partition partials are combined in ascending partition order — the
 * Buffered stage + pull of mttkrp.py:148-172 (count = 1 gives mttkrp_seq,
 * mttkrp.py:108-117). */
/* Elements per row of mode `mode` (a histogram of the mode's coordinates):
 * counts (I_mode,) uint32, zeroed by the caller.  The hot-row plans need only
 * these (their prefix sum is alto_row_index's row_ptr). */
int alto_row_counts(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int32_t mode,
                    uint32_t* counts, void* stream);
size_t alto_row_index_workspace_bytes(int64_t m, int64_t dim);
int alto_row_index(const alto_layout* lay, const void* d_tables,
                   const uint64_t* keys, int64_t m, int32_t mode,
                   int32_t* row_perm /* (M,), or NULL: row_ptr only */, int64_t* row_ptr /* (dim+1,) */,
                   void* workspace, size_t workspace_bytes, void* stream);
int alto_mttkrp_exact(const alto_mttkrp_args* a, const int32_t* row_perm,
                      const int64_t* row_ptr, const int64_t* part_off,
                      int64_t count, void* stream);

/* COO MTTKRP over a coordinate list (mttkrp_oracle, mttkrp.py:64-77),
 * coords (M, order) int64, float64 atomics (not reproducible bit for bit). */
int alto_mttkrp_coo(const int64_t* coords, const double* values, int64_t m,
                    int32_t order, int32_t mode, int32_t rank,
                    const double* const* factors_host_array /* host array of N device ptrs */,
                    double* out, int64_t out_rows, void* stream);
/* The same in the reference's arithmetic order: elements stably sorted by
 * output row, each row summed in input order (np.add.at, mttkrp.py:75) with
 * contributions ((v * F_a) * F_b) ... in ascending mode order, float64, no
 * contraction — bitwise equal to mttkrp_oracle.  Caller workspace of
 * alto_mttkrp_coo_workspace_bytes(m, out_rows) bytes. */
size_t alto_mttkrp_coo_workspace_bytes(int64_t m, int64_t out_rows);
int alto_mttkrp_coo_ordered(const int64_t* coords, const double* values, int64_t m,
                            int32_t order, int32_t mode, int32_t rank,
                            const double* const* factors_host_array,
                            double* out, int64_t out_rows, void* ws, size_t ws_bytes, void* stream);

/* ---- CP-ALS (cpd.py) --------------------------------------------------- */
/* All reductions below are two-stage with a fixed block count, so results
 * are bitwise reproducible run to run (cpd_als determinism,
 * pkg/tests/test_cpd.py:125-130).  `ws` is a caller workspace of at least
 * alto_cpd_workspace_bytes(rank) bytes. */
size_t alto_cpd_workspace_bytes(int32_t rank);

/* K10 gram (cpd.py:66-68): G = F^T F accumulated in float64. F (rows, rank). */
int alto_gram(const void* f, int32_t f_dtype, int64_t rows, int32_t rank, double* g,
              void* ws, size_t ws_bytes, void* stream);
/* K10 _hadamard_grams (cpd.py:71-77): V = 1 * prod over n != skip of G_n, in
 * mode order (skip = -1: all).  grams_host_array: host array of `order`
 * device pointers. */
int alto_hadamard_grams(const double* const* grams_host_array, int32_t order, int32_t skip,
                        int32_t rank, double* v, void* stream);
/* K11 + K12 (cpd.py:80-95, :116-120): solve X V = M by Cholesky (retry once
 * with ridge 1e-12 tr(V)/R), lambda = column 2-norms of X, X /= lambda
 * (zero-safe).  Writes X (float64) to x64 and, when x32 != NULL, a float32
 * copy.  *d_status (device int32): 0 ok, 1 ridge used, 2 singular. */
int alto_solve_normalize(const double* v, const double* mttkrp, int64_t rows, int32_t rank,
                         double* x64, float* x32, double* lambda, int32_t* d_status,
                         void* ws, size_t ws_bytes, void* stream);
/* K13 fit terms (cpd.py:124-146): out2[0] = sum_{i,r} M[i,r] F[i,r] lambda_r,
 * out2[1] = lambda^T V_all lambda. */
/* Fused factor update for ranks 16 / 32 (K11+K12+K10): Cholesky of V (ridge
 * retry as alto_solve_normalize), X = M V^-1 in two streaming passes (column
 * norms, then normalised X written as float64 and optional float32 copy),
 * lambda = column 2-norms, and gram = X^T X of the normalised X.  mttkrp is
 * (rows, rank) float32 or float64 (m_dtype).  Rank 16 runs X = M W
 * (W = V^-1) and the Gram on the float64 tensor cores (mma.sync m8n8k4);
 * flags & ALTO_CPD_SCALAR selects the scalar substitution kernels (rank 32
 * always uses them).  ALTO_EUNSUPPORTED for other ranks. */
#define ALTO_CPD_SCALAR 1
int alto_cpd_update(const double* v, const void* mttkrp, int32_t m_dtype, int64_t rows, int32_t rank, double* x64,
                    float* x32, double* lambda, double* gram, int32_t* d_status, int32_t flags, void* ws,
                    size_t ws_bytes, void* stream);
int alto_fit_terms(const double* mttkrp, const double* f, const double* lambda,
                   const double* v_all, int64_t rows, int32_t rank, double* out2,
                   void* ws, size_t ws_bytes, void* stream);
/* sum of squares of values in float64 (cpd.py:211). */
int alto_sumsq(const void* values, int32_t dtype, int64_t m, double* out,
               void* ws, size_t ws_bytes, void* stream);
/* Key-range-sharded CP-ALS pieces (multi-GPU).  row_mask
 * (I_n bytes, NULL = all rows) selects the rows this shard owns so each row
 * is counted once before the cross-shard all-reduce. */
int alto_gram_masked(const void* f, int32_t f_dtype, int64_t rows, int32_t rank, const uint8_t* row_mask,
                     double* g_partial, void* ws, size_t ws_bytes, void* stream);
/* X V = M (Cholesky + ridge retry), no normalisation. */
int alto_solve_rows(const double* v, const double* mttkrp, int64_t rows, int32_t rank, double* x64,
                    int32_t* d_status, void* ws, size_t ws_bytes, void* stream);
/* out[r] = sum over masked rows of X[i, r]^2. */
int alto_colsumsq(const double* x, int64_t rows, int32_t rank, const uint8_t* row_mask, double* out,
                  void* ws, size_t ws_bytes, void* stream);
/* lambda = sqrt(colsumsq); X /= lambda (zero-safe); optional float32 copy. */
int alto_normalize(double* x64, float* x32, int64_t rows, int32_t rank, const double* colsumsq, double* lambda,
                   const int32_t* d_status, void* stream);
/* out[0] = sum over masked rows of M[i,r] F[i,r] lambda_r. */
int alto_fit_inner_masked(const double* mttkrp, const double* f, const double* lambda, int64_t rows, int32_t rank,
                          const uint8_t* row_mask, double* out, void* ws, size_t ws_bytes, void* stream);
/* K14 shared-row exchange: buf[i, :] = src[rows[i], :] (pack) and
 * dst[rows[i], :] = buf[i, :] (unpack); rows (n,) int64 device array. */
int alto_pack_rows(const void* src, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, void* buf,
                   void* stream);
int alto_unpack_rows(void* dst, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, const void* buf,
                     void* stream);
/* dst[rows[k]] += buf[k] (rows unique within a call): the owner-side reduce of
 * the owner-directed shared-row exchange (dist.py). */
int alto_add_rows(void* dst, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, const void* buf,
                  void* stream);
/* Cast helpers for factor uploads: out32[i] = (float)in64[i]. */
int alto_cast_f64_f32(const double* in, float* out, int64_t n, void* stream);
int alto_cast_f32_f64(const float* in, double* out, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ALTO_B200_H */
