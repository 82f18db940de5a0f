/*
 * picasso.h — C ABI of the B200-native PICASSO packed sparse-embedding hot path.
 *
 * The operation (§III, arXiv 2204.04903): the embedding layer of a wide-and-deep
 * model looks up multi-hot categorical IDs of many feature fields (L131-140) through the
 * operator chain Unique -> Partition -> Gather -> Shuffle -> Stitch -> SegmentReduction
 * (L209-215); its backward pass is the mirror image (L219).  D-Packing (L319-362) merges the
 * fields whose tables share an embedding dimension into one packed ID stream served by one
 * fused pass; K-Packing (L364-382) fuses Unique&Partition and Shuffle&Stitch.  HybridHash
 * (L459-522, Alg. 1) keeps the top-k frequent rows in hot storage.  The backward ends in a
 * sparse optimizer update of the touched rows (north star; not specified by the paper).
 *
 * Conventions (every entry point):
 *  - All functions return picasso_status; no C++ type or exception crosses the ABI.
 *  - "device" pointers are CUDA global-memory pointers on the ctx's device; "host" pointers
 *    are ordinary host memory.  The caller owns every buffer (ids, offsets, out, dY,
 *    weights, optimizer state, workspace).  The library never allocates device memory in
 *    the step path; the ctx owns host objects, its NCCL communicator, one internal stream
 *    (the forward's overlapped transpose, joined before the forward returns) and, with the
 *    peer-memory exchange (section 7), its IPC window and owner table (allocated once).
 *  - Work is enqueued on the caller's stream and is asynchronous.  fwd and bwd_update never
 *    synchronise the host when world == 1 or with the peer-memory exchange at world > 1
 *    (the step is CUDA-graph capturable).
 *  - Argument / plan errors are synchronous return codes.  Device-detected errors (ID out
 *    of range in ROWS mode, capacity overflow, offsets that are not a CSR over the IDs, a peer
 *    timeout) are latched in a device word and reported by picasso_last_error (which
 *    synchronises the stream it last used).
 *  - One ctx per rank; a ctx is not thread-safe.
 */
#ifndef PICASSO_H_
#define PICASSO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PICASSO_OK = 0,
    PICASSO_ERR_INVALID_ARG = -1,   /* bad pointer / size / enum value */
    PICASSO_ERR_PLAN_MISMATCH = -2, /* plan or field layout inconsistent with the call */
    PICASSO_ERR_ID_RANGE = -3,      /* ROWS mode: a raw ID outside [0, V_t) (latched) */
    PICASSO_ERR_CAPACITY = -4,      /* batch / ids / workspace larger than the ctx was built for */
    PICASSO_ERR_CUDA = -5,          /* a CUDA runtime call failed */
    PICASSO_ERR_NCCL = -6,          /* an NCCL call failed */
    PICASSO_ERR_STATE = -7          /* call order violated (bwd_update without a preceding fwd) */
} picasso_status;

typedef enum { PICASSO_POOL_SUM = 0, PICASSO_POOL_MEAN = 1 } picasso_pool;
typedef enum { PICASSO_OPT_ADAGRAD = 0, PICASSO_OPT_ADAM_LAZY = 1 } picasso_opt;
/* Row of a raw ID in its table (reading O4): ROWS: row = raw (0 <= raw < V_t);
 * HASH: row = floor(mix64(raw XOR salt_t) * V_t / 2^64), mix64 = SplitMix64's output mix. */
typedef enum { PICASSO_IDS_ROWS = 0, PICASSO_IDS_HASH = 1 } picasso_id_mode;

typedef struct picasso_ctx picasso_ctx;

/* ------------------------------------------------------------------------------------ */
/* 1. Planning — D-Packing with Eq. 1.  Host only, pure, deterministic.
 *   Groups tables by embedding dim (ascending dim).  vparam(group) = sum_t dim_t * count_t
 *   (Eq. 1 with ID_freq = count/N, reading O15); count_t = table_warmup_count[t] (ID
 *   occurrences seen in warm-up iterations, L353-354) or, when NULL, the number of fields
 *   that reference t.  split == 1: a group with vparam above the mean is split into
 *   min(#tables, ceil(vparam / min_vparam)) shards (reading O14; reproduces the paper's
 *   four-shard example L358-362), members dealt round-robin by descending dim_t*count_t.
 *   split = k >= 2: every group is dealt the same way into min(#tables, k) packs — the
 *   K-Interleaving groups of L424-443 (at world > 1 with the peer-memory exchange, pack p's
 *   exchange then overlaps pack p-1's pool and owner update).
 *   Within a pack tables are ordered by ascending index; table_base[t] = rows of the pack's
 *   earlier tables, so pack key = table_base[t] + row.
 * In : n_fields F >= 1, field_to_table [F] (host), n_tables T >= 1, table_rows [T] (> 0),
 *      table_dim [T] (> 0), table_warmup_count [T] or NULL, split.
 * Out (caller-allocated host arrays): field_to_pack [F], table_to_pack [T], table_base [T],
 *      pack_dim [T], pack_rows [T] (first *n_packs entries valid), *n_packs.
 * Errors: PICASSO_ERR_INVALID_ARG on NULL pointers, F/T <= 0, out-of-range table index,
 *      non-positive rows/dims. */
picasso_status picasso_pack_plan(int32_t n_fields, const int32_t *field_to_table, int32_t n_tables,
                                 const int64_t *table_rows, const int32_t *table_dim,
                                 const uint64_t *table_warmup_count, int32_t split,
                                 int32_t *field_to_pack, int32_t *table_to_pack, int64_t *table_base,
                                 int32_t *pack_dim, int64_t *pack_rows, int32_t *n_packs);

/* The plan, as returned by picasso_pack_plan, plus the model's per-field output columns.
 * All pointers are host pointers; the ctx copies them. */
typedef struct {
    int32_t n_fields, n_tables, n_packs;
    const int32_t *field_to_table; /* [F] */
    const int32_t *table_to_pack;  /* [T] */
    const int64_t *table_base;     /* [T] */
    const int64_t *table_rows;     /* [T] */
    const int32_t *table_dim;      /* [T]; 1 <= dim <= 512.  Stored at the kernel dim (picasso_kernel_dim:
                                      the next of 4, 8, 16, 32, 64, 128, 256, 384, 512): weights, state,
                                      and the field's out / dY column block are kernel-dim wide, the
                                      padding columns are 0 in out and must be 0 in dY and the tables */
    const uint64_t *table_salt;    /* [T] HASH-mode salts (NULL = all 0) */
    const int64_t *field_col;      /* [F] first column of field f in the [B, out_width] output
                                      (a multiple of 4) */
    int64_t out_width;             /* row stride of out / dY in floats (multiple of 4) */
    const int32_t *pack_group;     /* [P] K-Interleaving group of each pack (picasso_pack_plan_kinterleave;
                                      -1 = preset excluded, ahead of the groups), or NULL: one group per
                                      pack.  Groups must be contiguous and ascending in pack order. */
} picasso_plan_view;

typedef struct {
    int32_t max_batch;     /* B per rank per step, upper bound */
    int64_t max_ids;       /* ID occurrences per rank per step, upper bound (< 2^31) */
    int32_t pool;          /* picasso_pool */
    int32_t id_mode;       /* picasso_id_mode */
    int32_t opt;           /* picasso_opt */
    float eps;             /* Adagrad 1e-10 / Adam 1e-8 */
    float beta1, beta2;    /* Adam (0.9, 0.999) */
    int64_t max_recv;      /* world > 1: keys this rank may receive per step as an owner
                              (0 = 2 * max_ids); exceeding it fails the step with CAPACITY */
    int64_t cache_max_bytes; /* world > 1: largest hot-storage capacity picasso_hot_cache_refresh
                              will be asked for (0 = no HybridHash: no FCounter, no hot rows) */
    int32_t exchange;        /* world > 1: 0 = NVLink peer memory (section 7; the rows / G buffers
                              live in the IPC window, not the workspace), 1 = NCCL AllToAllv
                              (section 5; loopback: device copies) */
    int64_t max_step_unique; /* world == 1: D-Interleaving (section 8) — distinct keys one step's
                              micro-batches may touch together (sizes the step accumulator's
                              index: 2 x 16 B per key); 0 = off */
    int64_t max_step_floats; /* D-Interleaving: fp64 accumulator values (sum of D over the step's
                              distinct keys); 0 = max_step_unique x the largest pack dim */
    int32_t cold_tier;       /* world == 1: 1 = HybridHash with a host-DRAM cold tier (section 9):
                              the packs' weights / state passed to picasso_bind live in pinned,
                              device-mapped host memory and up to cache_max_bytes of their
                              hottest rows are cached in HBM; 0 = tables in device memory */
} picasso_ctx_opts;

/* 1b. K-Interleaving plan (Eq. 3).
 *   picasso_interleave_capacity : Eq. 3, Capacity_g = min over ops of rbound[i] / rparam[i] in
 *     parameters per step ("we simply treat the parameter volume as the cost in embedding lookup
 *     and exchange", L437-438): e.g. rbound = bytes an op's dominant resource (HBM, NVLink) moves
 *     in one interleaving slot at its measured rate, rparam = its bytes per parameter.  Ops with
 *     rparam 0 never bind; none binding gives +inf.
 *   picasso_pack_plan_kinterleave : D-Packing (as picasso_pack_plan, split 0) where (1) the tables
 *     flagged in `excluded` ([T] or NULL) — the paper's "preset excluded embedding", L444-447 —
 *     form one pack per dim placed first, outside the chain (pack_group -1); (2) every other dim
 *     group of volume V = sum_t dim_t * count_t (Eq. 1) is cut into min(#tables, ceil(V /
 *     capacity_g)) packs, tables dealt round-robin by descending dim_t * count_t; (3) those packs
 *     are joined, in order, into interleaving groups of at most capacity_g parameters (a pack above
 *     it stays alone).  capacity_g <= 0 or +inf: one pack per dim, one group.  With the peer-memory
 *     exchange at world > 1 each group has its own barrier: group g's pool (forward) and owner
 *     update (backward) run beside group g+1's exchange; excluded packs run first and wait on
 *     no group.  Out: as picasso_pack_plan, plus pack_group [<=T], *n_groups (excluded packs
 *     not counted). */
picasso_status picasso_interleave_capacity(int32_t n_ops, const double *rbound, const double *rparam,
                                           double *capacity);
picasso_status picasso_pack_plan_kinterleave(int32_t n_fields, const int32_t *field_to_table, int32_t n_tables,
                                             const int64_t *table_rows, const int32_t *table_dim,
                                             const uint64_t *table_warmup_count, double capacity_g,
                                             const uint8_t *excluded, int32_t *field_to_pack, int32_t *table_to_pack,
                                             int64_t *table_base, int32_t *pack_dim, int64_t *pack_rows,
                                             int32_t *pack_group, int32_t *n_packs, int32_t *n_groups);

/* Row width the kernels store a table of embedding dim `dim` at (1 <= dim <= 512): the next of 4, 8,
 * 16, 32, 64, 128, 256, 384, 512.  INVALID_ARG outside that range. */
picasso_status picasso_kernel_dim(int32_t dim, int32_t *kdim);

/* NCCL unique id (128 bytes, host) for picasso_ctx_create; rank 0 calls it and broadcasts
 * the bytes to the other ranks (e.g. over torch.distributed). */
picasso_status picasso_nccl_unique_id(uint8_t *out);

/* 2. Context.  rank/world (1 <= world <= 8): this rank's place in the row-sharded group —
 * owner of pack key k is rank k mod world, at local row k div world (reading O3; PAPER.md
 * L192-195 model parallelism).  nccl_uid: world > 1 with one process per GPU — the 128-byte
 * NCCL id; the communicator is created in picasso_bind (a collective over the world).
 * nccl_uid == NULL with world > 1: "loopback" — all ranks live in this process on one device
 * and are driven together through picasso_group_* (tests of W up to 8 without 8 GPUs).
 * Errors: INVALID_ARG / PLAN_MISMATCH on inconsistent plans or options. */
picasso_status picasso_ctx_create(const picasso_plan_view *plan, int32_t rank, int32_t world,
                                  const uint8_t *nccl_uid, const picasso_ctx_opts *opts, picasso_ctx **out);
/* Bytes of device workspace the ctx needs (depends on max_batch, max_ids, plan). */
picasso_status picasso_workspace_size(const picasso_ctx *ctx, size_t *bytes);
/* Rows of pack p held by this rank: ceil((pack_rows[p] - rank) / world). */
picasso_status picasso_pack_local_rows(const picasso_ctx *ctx, int32_t pack, int64_t *rows);
/* Attach caller-owned device memory: workspace (>= picasso_workspace_size bytes, 256-B
 * aligned); pack_weight[p] = fp32 [local_rows_p, pack_dim_p] row-major; pack_state1[p] =
 * Adagrad accumulator or Adam m (same shape); pack_state2[p] = Adam v (NULL for Adagrad).
 * Synchronous (uploads the plan tables into the workspace). */
picasso_status picasso_bind(picasso_ctx *ctx, void *workspace, size_t bytes, float *const *pack_weight,
                            float *const *pack_state1, float *const *pack_state2);
picasso_status picasso_ctx_destroy(picasso_ctx *ctx);

/* 3. Forward — packed lookup.  For every pack: ID hashing
 * into pack keys, fused Unique&Partition (first-occurrence unique + inverse; reading O1),
 * row gather fused with SegmentReduction (stitch fused away):
 *     out[b, col(f) + d] = sum_{j in seg(f,b)} W_t[row_j][d]   (ascending j; mean: / len;
 *                                                              empty segment: 0)
 * ids     : device int64 [n_ids], field-major: field f, then sample b, then j.
 * offsets : device int32 [F*batch + 1]; seg(f,b) = [offsets[f*B+b], offsets[f*B+b+1]),
 *           offsets[0] == 0, non-decreasing, offsets[F*B] == n_ids.
 * out     : device fp32 [batch, out_width], fully overwritten.
 * Keeps the per-step state (unique keys, inverse, segment map) in the workspace for the
 * next picasso_packed_lookup_bwd_update, and reads `offsets` again there (mean combiner: bag
 * lengths): offsets must stay valid and unchanged until that backward has been enqueued.
 * Index path: at world == 1 the Unique of every pack comes from one stable LSD sort of the
 * step's (pack key, position) items, which also yields the backward's rows in ascending-key
 * order; the row-sharded step does the same from 2^20 IDs per rank on (its exchange then reads
 * the sort's first-occurrence views) and below that uses the hash-table Unique + uid transpose
 * (PICASSO_INDEX=hash everywhere); all give the same forward and the same updates.
 * offsets that are not such a CSR latch INVALID_ARG (picasso_last_error); the step then runs
 * on a substitute layout that keeps every access in bounds, and its results are meaningless.
 * Errors: CAPACITY if batch > max_batch or n_ids > max_ids; STATE if not bound. */
picasso_status picasso_packed_lookup_fwd(picasso_ctx *ctx, const int64_t *ids, const int32_t *offsets,
                                         int32_t batch, int64_t n_ids, float *out, void *stream);

/* 4. Backward + sparse update — the mirror of the forward: for every
 * unique row u of the last forward,
 *     G_u = sum_{j : inverse[j] = u} dY[b(j), col(f(j)) + .]   (mean: dY / len)
 * then, for touched rows only (reading O9), Adagrad: acc += G^2; w -= lr*G/(sqrt(acc)+eps),
 * or lazy Adam (torch SparseAdam form, bias correction with the 1-based `step`).
 * grad_out: device fp32 [batch, out_width] (dY, same layout as out); may be NULL when the
 * forward's batch was 0 (at world > 1 such a rank still takes part in the step).
 * Summation: each contribution formed in fp32, accumulated in fp64, rounded once (reading O6);
 * the order is fixed (ascending occurrence within equal-cost tiles, tile pieces combined in
 * tile order), so results are bitwise deterministic run to run.
 * Errors: STATE without a preceding fwd; INVALID_ARG for a NULL grad_out with batch > 0. */
picasso_status picasso_packed_lookup_bwd_update(picasso_ctx *ctx, const float *grad_out, float lr,
                                                int64_t step, void *stream);

/* Last latched error (synchronises the ctx's last stream).  msg may be NULL. */
picasso_status picasso_last_error(picasso_ctx *ctx, char *msg, size_t len);

/* ------------------------------------------------------------------------------------ */
/* Introspection of the last forward's intermediates (tests; synchronise the stream).
 * Copies into caller device buffers; *n receives the element count (copy truncated at cap).
 *   picasso_get_unique : pack keys of pack p in first-occurrence order (int64 [U_p])
 *   picasso_get_inverse: per occurrence of pack p's key stream (pack fields in ascending
 *                        field order, then b, then j) its index into unique (int32 [N_p])
 * After a sort-indexed forward (world == 1, or world > 1 with the peer-memory exchange) the
 * step itself numbers rows by key; these two
 * first-occurrence views (reading O1) are built from the sorted items on the first call after
 * the forward (a few extra kernels on the ctx's last stream), valid until the next forward. */
picasso_status picasso_get_unique(picasso_ctx *ctx, int32_t pack, int64_t *dst, int64_t cap, int64_t *n);
picasso_status picasso_get_inverse(picasso_ctx *ctx, int32_t pack, int32_t *dst, int64_t cap, int64_t *n);

/* Number of CUDA kernel launches the last fwd / bwd_update enqueued (host counters). */
picasso_status picasso_launch_count(const picasso_ctx *ctx, int64_t *fwd, int64_t *bwd);

/* Phase timing with CUDA events recorded on the caller's stream around each phase of the
 * step: 0 = ID hash + Unique (+ Partition at world > 1), 1 = gather/pool (k_pool),
 * 2 = occurrence transpose (radix sort + k_csr_bounds), 3 = segment-sum (+ optimizer at
 * world == 1), 4 = owner dedup + gather (world > 1), 5 = owner reduce + optimizer (world > 1).
 * The exchanges themselves are outside every phase.  picasso_profile_read synchronises,
 * writes the summed milliseconds of each phase since the last read into ms[6] (host), the
 * number of steps into *calls, and resets.  Off by default. */
/* on: 0 off, 1 on, 2 on for a step about to be captured into a CUDA graph (world == 1): the
 * recorded events become graph nodes, so picasso_profile_read after each replay returns that
 * replay's phase times without resetting the event list. */
picasso_status picasso_profile_enable(picasso_ctx *ctx, int32_t on);
picasso_status picasso_profile_read(picasso_ctx *ctx, float *ms, int64_t *calls);

/* Per-pack unique counts of the last forward as an int32 [n_packs + 1] prefix (uid range of
 * pack p = [u[p], u[p+1])), copied asynchronously on `stream` into dst (device memory or
 * pinned host memory).  Enqueue-only; the caller synchronises. */
picasso_status picasso_unique_offsets(picasso_ctx *ctx, int32_t *dst, void *stream);
/* Per pack (the first 64): ms of its pool (Gather + Stitch + SegmentReduction) and of its backward kernels
 * (segment-sum and update) in the profiled steps since the last picasso_profile_read (host arrays
 * [cap]; call before picasso_profile_read, which resets them; world == 1 backward only). */
picasso_status picasso_profile_read_packs(picasso_ctx *ctx, float *pool_ms, float *bwd_ms, int32_t cap);

/* ------------------------------------------------------------------------------------ */
/* 5. Row-sharded step at world > 1 (PAPER.md L192-195 MP strategy, L209-215 operators).
 * With NCCL (one process per GPU) the ordinary picasso_packed_lookup_fwd / _bwd_update run
 * the sharded step: Unique & Partition -> counts exchange (one host synchronisation: NCCL
 * needs host-side sizes) -> IDs AllToAllv -> owner dedup + Gather -> rows AllToAllv ->
 * pooling from the received rows (Stitch fused) ; backward: segment-sum into the send
 * layout -> gradients AllToAllv -> owner reduce over <= world contributions (source rank
 * ascending, fp64) + optimizer.  Per-requester gradient partials travel as fp32 (reading O6).
 * The loopback group runs the same phases for all ranks of one process, with device copies
 * for the exchanges; its arguments are per-rank arrays of what fwd/bwd_update take. */
typedef struct picasso_group picasso_group;

/* 6. HybridHash hot storage (Alg. 1), world > 1 and cache_max_bytes > 0.
 * FCounter counts every key once per rank-step in which it is in that rank's unique set
 * (reading O11; owners count received keys, ranks count their hot hits).  The caller applies
 * Alg. 1's schedule: after picasso_packed_lookup_bwd_update of iteration itr, call
 * picasso_hot_cache_refresh when itr >= warmup_iters and itr % flush_iters == 0 (reading O13;
 * the paper warms up 100 steps, L795).  The refresh writes the replicas back to the owners,
 * selects the longest prefix of all keys sorted by (count desc, pack asc, key asc) whose rows
 * (weights + optimizer state, 4*D*(1+n_state) bytes each) fit capacity_bytes (<= the ctx's
 * cache_max_bytes), and replicates those rows on every rank, slots in ascending key (grouped by
 * pack).  The selection runs on the devices: the ranks AllReduce per-pack count histograms and
 * a key-bin histogram of the rows at the cut count, so each finds the same cut without moving
 * candidate lists (exact while FCounter values stay below 65535; larger counts share the top
 * histogram bin and are then ordered by key).  From then on hot keys are served
 * by the local replica, skip the AllToAllv, and their gradients are summed over the ranks
 * (AllReduce) so every replica applies the same update.  Results equal the uncached step
 * (tier transparency) up to the fp32 cross-rank sum of hot gradients.  capacity_bytes = 0:
 * write back and drop (e.g. before a checkpoint).  world == 1: no-op (the table itself is the
 * hot storage; reading O18).  Collective: every rank calls it (NCCL mode).  stats (host, may
 * be NULL) describe the new hot set and the last forward's hit ratio over unique keys
 * (P:L796). */
typedef struct {
    int64_t k;                /* hot rows */
    int64_t bytes;            /* bytes of hot storage in use (weights + optimizer state) */
    int64_t hot_uniques;      /* last forward: unique keys served by the replica ... */
    int64_t uniques;          /* ... out of this many unique keys of the rank */
    double hit_ratio_unique;  /* hot_uniques / uniques */
    double refresh_ms;        /* host wall time of this refresh (from the drained stream to its end) */
    double propose_ms, select_ms;  /* of which: histograms + threshold + tie cut; bitmap + staging */
} picasso_cache_stats;
picasso_status picasso_hot_cache_refresh(picasso_ctx *ctx, size_t capacity_bytes, void *stream,
                                         picasso_cache_stats *stats);
picasso_status picasso_group_hot_cache_refresh(picasso_group *group, size_t capacity_bytes, void *stream,
                                               picasso_cache_stats *stats /* [world] or NULL */);
/* Current hot keys (tests): pack and pack key of each hot slot, slot order = ascending global key
 * (host arrays). */
picasso_status picasso_get_hot_keys(picasso_ctx *ctx, int32_t *pack, int64_t *key, int64_t cap, int64_t *n);
picasso_status picasso_group_create(picasso_ctx *const *ctxs, int32_t world, picasso_group **out);
picasso_status picasso_group_destroy(picasso_group *group);
picasso_status picasso_group_fwd(picasso_group *group, const int64_t *const *ids, const int32_t *const *offsets,
                                 const int32_t *batch, const int64_t *n_ids, float *const *out, void *stream);
picasso_status picasso_group_bwd_update(picasso_group *group, const float *const *grad_out, float lr, int64_t step,
                                        void *stream);
/* Owner-side intermediate of the last forward (world > 1; tests, synchronises): the owner's
 * unique local rows of pack p in first-occurrence order of the received lists concatenated by
 * source rank (int64, copied to dst), and the per-peer key counts this rank sent (int64 [world],
 * host). */
picasso_status picasso_get_owner_unique(picasso_ctx *ctx, int32_t pack, int64_t *dst, int64_t cap, int64_t *n);
picasso_status picasso_get_send_counts(picasso_ctx *ctx, int64_t *host_counts);
/* Partition of the last forward (world > 1; tests, synchronises): the local rows (key div W,
 * reading O3) this rank requested from `owner` for pack `pack`, in send order — the pack's
 * unique keys with key mod W == owner in first-occurrence order (PAPER.md L211 Partition,
 * SPEC.md L113-118; = oracle_partition's list; after a sort-indexed step with the peer-memory
 * exchange the same rows in ascending order).  Hot keys (HybridHash) are not sent.  dst: host
 * int64 [cap]; n: the list length. */
picasso_status picasso_get_send_list(picasso_ctx *ctx, int32_t owner, int32_t pack, int64_t *dst, int64_t cap,
                                     int64_t *n);

/* 8. D-Interleaving (Eq. 2), world == 1, opts.max_step_unique > 0.
 * A step's batch is sliced into micro-batches (per field, samples [b0, b1): the caller slices
 * ids / offsets) that flow through the layer one after another, so every batch-proportional
 * buffer — out, dY, and the ctx's per-ID / per-unique scratch (max_batch, max_ids) — is sized
 * for one micro-batch; the update is applied once, with the whole batch's gradient:
 *   picasso_micro_batch_size : Eq. 2, BS_micro = min over ops of rbound[i] / rinstance[i]
 *                              (host arrays [n_ops]; e.g. bytes of device memory an op may use /
 *                              its bytes per sample measured in warm-up, L416-421), clamped to
 *                              batch, then the batch evenly divided: n_micro = ceil(batch /
 *                              BS_micro), bs_micro = ceil(batch / n_micro).  CAPACITY if a bound
 *                              admits no sample at all.
 *   picasso_dinterleave_begin : starts a step (clears the step accumulator).
 *   then per micro-batch: picasso_packed_lookup_fwd (unchanged: its output rows are the whole
 *      batch's rows of those samples, bit-exact — the tables are not updated until apply), and
 *   picasso_packed_lookup_bwd_accumulate(grad_out = that micro-batch's dY, out's layout): its
 *      per-unique G rows (rounded once from fp64) added in fp64 to the step accumulator;
 *   picasso_dinterleave_apply : G = fp32(accumulated sum) of every row any micro-batch touched,
 *      and the optimizer step (as picasso_packed_lookup_bwd_update; step is 1-based).
 * Results equal the whole batch's step (bit-exact under dyadic dY; otherwise within 1 ulp of G:
 * reading O6').  More distinct keys than max_step_unique latch CAPACITY (the step's
 * update is then incomplete).  picasso_packed_lookup_bwd_update is refused (STATE) between begin
 * and apply. */
picasso_status picasso_micro_batch_size(int32_t n_ops, const double *rbound, const double *rinstance, int32_t batch,
                                        int32_t *bs_micro, int32_t *n_micro);
picasso_status picasso_dinterleave_begin(picasso_ctx *ctx, void *stream);
picasso_status picasso_packed_lookup_bwd_accumulate(picasso_ctx *ctx, const float *grad_out, void *stream);
picasso_status picasso_dinterleave_apply(picasso_ctx *ctx, float lr, int64_t step, void *stream);
/* The last D-Interleaving step's accumulator use (synchronises): distinct keys and fp64 values
 * (host int64) — the warm-up measurement that sizes max_step_unique / max_step_floats. */
picasso_status picasso_dinterleave_stats(picasso_ctx *ctx, int64_t *rows, int64_t *floats);

/* 7. Exchange over NVLink peer memory (kernel-initiated Shuffle&Stitch).
 * Replaces the NCCL AllToAllv of section 5 with one shared window per rank (barrier flags,
 * bucket counts, send list, rows / G buffer; cudaMalloc'ed by the library, freed at destroy):
 * owners read the requested keys from the requesters' send lists, store the gathered rows
 * straight into the requesters' rows buffers (Gather + Shuffle + Stitch in one kernel), and in
 * the backward pull the requesters' G rows into the reduce + optimizer kernel.  Sizes stay on
 * the device (no host synchronisation inside a step: a step can be captured in a CUDA graph);
 * ranks meet at three device-side barriers per step (system-scope release/acquire flags; a
 * peer missing for 20 s latches a sticky "peer timeout" instead of hanging: from then on the owner
 * update kernels leave the tables and optimizer state untouched, and picasso_last_error — which
 * every caller must check after a step in this mode — returns PICASSO_ERR_STATE until the
 * context is destroyed).  Results are
 * bit-identical to section 5 (same layouts, same source-ordered sums).  HybridHash hot rows
 * keep their NCCL AllReduce.  Requirements: every rank built with the same plan and max_ids,
 * one GPU per rank, peer access between the GPUs (NVLink / NVSwitch).
 *   picasso_p2p_handle : after picasso_bind: allocates this rank's window and writes its CUDA
 *                        IPC handle (64 bytes) into handle_out (host).
 *   picasso_p2p_open   : handles = the world ranks' 64-byte handles, rank order (host; own
 *                        entry ignored); maps the peers' windows.  Collective in effect: every
 *                        rank must open before any rank steps.
 *   picasso_group_p2p  : loopback group: the same path with the ranks' windows as plain
 *                        pointers on one device (no barriers: the host orders the phases). */
/* 7b. NVLS multicast for the HybridHash hot-row gradients (world > 1, peer-memory exchange, cache on).
 * Instead of an NCCL AllReduce, each rank's hot-row gradient rows and occurrence counts sit in a
 * multicast-bound buffer; after the backward barrier every rank reduces 1/W of it inside the
 * NVSwitch (multimem.ld_reduce) and broadcasts the sums to all ranks (multimem.st), then a second
 * barrier.  Collective setup, in this order on every rank (after picasso_p2p_open):
 *   picasso_nvls_create : rank 0 creates the multicast object and exports it as a POSIX file
 *                         descriptor (*fd_out; other ranks: -1); every rank sizes the buffer.
 *   (the caller passes rank 0's descriptor to the other processes, e.g. SCM_RIGHTS)
 *   picasso_nvls_open   : fd = that descriptor in this process (ignored on rank 0); imports the
 *                         object and adds this rank's device.
 *   (a host barrier: every rank has opened)
 *   picasso_nvls_bind   : binds this rank's device memory, maps the unicast and multicast views,
 *                         and routes the hot-row gradients there.
 * PICASSO_ERR_CUDA when the GPUs / driver lack multicast or fabric handles: the step then keeps
 * the NCCL AllReduce. */
picasso_status picasso_nvls_create(picasso_ctx *ctx, int32_t *fd_out);
picasso_status picasso_nvls_open(picasso_ctx *ctx, int32_t fd);
picasso_status picasso_nvls_bind(picasso_ctx *ctx);
picasso_status picasso_p2p_handle(picasso_ctx *ctx, void *handle_out);
picasso_status picasso_p2p_open(picasso_ctx *ctx, const void *handles);
picasso_status picasso_group_p2p(picasso_group *group);

#ifdef __cplusplus
}
#endif
#endif /* PICASSO_H_ */
