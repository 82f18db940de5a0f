/*
 * picasso_oracle.cpp — CPU ORACLE for the PICASSO packed sparse-embedding hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2204_04903_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * What it computes, written as the plain definitions (no packing, no hashing tables,
 * no cache, no blocking, no reordering):
 *   - row mapping of a raw categorical ID into its table     (reading O4)
 *   - Eq. 1 CalcVParam and the D-Packing plan
 *   - forward: per field, per sample SegmentReduction
 *   - Unique / Partition intermediates, per rank and pack
 *   - backward ("mirror image of the forward pass", L219):
 *       G_t[row] = sum over the global batch of dY (or dY/len)
 *   - sparse Adagrad / lazy Adam on the touched rows (north star; readings O9, O10)
 *   - Alg. 1 FCounter top-k hot-set selection
 *
 * Precision: the paper trains in full precision ("full-precision training", fp32,
 * PAPER.md L577; accuracy loss "intolerable", L164).  The oracle therefore computes in
 * fp32; the forward SegmentReduction sums sequentially left to right from +0.0f (SPEC.md
 * L157, L165: "fixed left-to-right order, no reassociation"); the backward's per-row
 * gradient sum, whose precision the paper does not fix, accumulates in fp64 and rounds
 * once (reading O6).  Built with -ffp-contract=off -fno-fast-math (no FMA contraction).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC worked examples, brute force on
 * tiny inputs, float64 dense incidence-matrix closed forms (Y = A·W, dW = A^T·dY),
 * torch.nn.functional.embedding_bag, torch.optim.Adagrad / SparseAdam sparse paths,
 * SplitMix64 published known-answer vectors, the paper's four-shard example.
 */
#ifdef _OPENMP
#include <omp.h>
#endif
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <unordered_set>
#include <vector>

extern "C" {

/* ---- status codes (same numeric meaning as the product ABI, defined independently) ---- */
enum { OR_OK = 0, OR_INVALID = -1, OR_MISMATCH = -2, OR_ID_RANGE = -3, OR_CAPACITY = -4 };

enum { OR_IDS_ROWS = 0, OR_IDS_HASH = 1 };
enum { OR_POOL_SUM = 0, OR_POOL_MEAN = 1 };
enum { OR_OPT_ADAGRAD = 0, OR_OPT_ADAM = 1 };

/* Model description: F fields, T tables.  field_col[f] = first output column of f. */
typedef struct {
    int32_t n_fields;
    int32_t n_tables;
    const int32_t *field_to_table; /* [F] */
    const int64_t *table_rows;     /* [T] */
    const int32_t *table_dim;      /* [T] */
    const uint64_t *table_salt;    /* [T] (HASH mode) */
    int32_t id_mode;               /* OR_IDS_ROWS | OR_IDS_HASH */
    int32_t pool;                  /* OR_POOL_SUM | OR_POOL_MEAN */
    const int64_t *field_col;      /* [F] */
} oracle_model;

/* One rank's batch, field-major: segment (f,b) = ids[offsets[f*B+b] .. offsets[f*B+b+1]). */
typedef struct {
    int32_t batch;           /* B */
    const int64_t *ids;      /* [N] */
    const int32_t *offsets;  /* [F*B+1] */
    const float *dy;         /* [B, dy_stride] (backward only; may be NULL) */
    int64_t dy_stride;
} oracle_batch;

typedef struct {
    int32_t kind;          /* OR_OPT_ADAGRAD | OR_OPT_ADAM */
    float lr;
    float eps;             /* Adagrad 1e-10, Adam 1e-8 */
    float beta1, beta2;    /* Adam */
} oracle_opt;

/* ------------------------------------------------------------------------------------ */
/* Row mapping.  Reading O4: PAPER.md L115 only says IDs go through "various
 * hashing"; we fix
 *   ROWS mode: row = raw, error unless 0 <= raw < V
 *   HASH mode: row = floor(mix64(raw XOR salt) * V / 2^64)   ("multiply-high" range map)
 * mix64 = the SplitMix64 output function (Steele, Lea, Flood 2014), constants as published. */
uint64_t oracle_mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int32_t oracle_row_of(int32_t mode, int64_t raw, uint64_t salt, int64_t V, int64_t *row) {
    if (V <= 0) return OR_INVALID;
    if (mode == OR_IDS_ROWS) {
        if (raw < 0 || raw >= V) return OR_ID_RANGE;
        *row = raw;
        return OR_OK;
    }
    if (mode == OR_IDS_HASH) {
        unsigned __int128 p = (unsigned __int128)oracle_mix64((uint64_t)raw ^ salt) * (uint64_t)V;
        *row = (int64_t)(uint64_t)(p >> 64);
        return OR_OK;
    }
    return OR_INVALID;
}

/* ------------------------------------------------------------------------------------ */
/* Eq. 1: CalcVParam(T) = N * sum_{t in T} ( t_dim * sum_{ID in t} ID_freq ).
 * With ID_freq = count(ID)/N (frequencies from warm-up statistics, L353-354) this is
 * sum_t t_dim * count_t, count_t = number of ID occurrences that hit table t (reading O15). */
double oracle_calc_vparam(int32_t n, const int32_t *dims, const double *id_freq_sums, double N) {
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i) s += (double)dims[i] * id_freq_sums[i];
    return N * s;
}

/* D-Packing plan.
 *  1. one group per distinct embedding dim ("we pack up categorical feature IDs when their
 *     embedding tables share the same feature dimension", L334-336), groups in ascending dim;
 *  2. vparam per group by Eq. 1, count_t from warm-up counts (NULL: every field referencing
 *     t contributes 1 — uniform traffic per field);
 *  3. a group whose vparam is above the mean over groups is "evenly split into multiple
 *     shards" (L357-358).  Reading O14: shards = min(#tables, ceil(vparam / min vparam)),
 *     which reproduces the paper's example (dim 8 and dim 32, uniform: four shards,
 *     L358-362).  Tables are never split; members go round-robin in descending per-table
 *     vparam (ties: ascending table index);
 *  4. packs are numbered group by group (ascending dim), shards in order; within a pack,
 *     tables are ordered by ascending table index and table_base[t] is the running row sum.
 * split == 0 skips step 3. */
int32_t oracle_pack_plan(int32_t n_fields, const int32_t *field_to_table, int32_t n_tables,
                         const int64_t *table_rows, const int32_t *table_dim,
                         const uint64_t *table_warmup_count, int32_t split,
                         int32_t *field_to_pack, int32_t *table_to_pack, int64_t *table_base,
                         int32_t *pack_dim, int64_t *pack_rows, int32_t *n_packs) {
    if (n_fields <= 0 || n_tables <= 0) return OR_INVALID;
    std::vector<double> cnt(n_tables, 0.0);
    for (int32_t f = 0; f < n_fields; ++f) {
        int32_t t = field_to_table[f];
        if (t < 0 || t >= n_tables) return OR_INVALID;
    }
    for (int32_t t = 0; t < n_tables; ++t)
        if (table_rows[t] <= 0 || table_dim[t] <= 0) return OR_INVALID;
    if (table_warmup_count) {
        for (int32_t t = 0; t < n_tables; ++t) cnt[t] = (double)table_warmup_count[t];
    } else {
        for (int32_t f = 0; f < n_fields; ++f) cnt[field_to_table[f]] += 1.0;
    }
    /* groups by distinct dim, ascending */
    std::vector<int32_t> dims;
    for (int32_t t = 0; t < n_tables; ++t) dims.push_back(table_dim[t]);
    std::sort(dims.begin(), dims.end());
    dims.erase(std::unique(dims.begin(), dims.end()), dims.end());
    int32_t G = (int32_t)dims.size();
    std::vector<std::vector<int32_t>> members(G);
    for (int32_t t = 0; t < n_tables; ++t) {
        int32_t g = (int32_t)(std::lower_bound(dims.begin(), dims.end(), table_dim[t]) - dims.begin());
        members[g].push_back(t);
    }
    std::vector<double> vp(G, 0.0);
    double N = 0.0; /* total ID occurrences in the warm-up statistics (reading O15: global N) */
    for (int32_t t = 0; t < n_tables; ++t) N += cnt[t];
    for (int32_t g = 0; g < G; ++g) {
        /* Eq. 1 with ID_freq sums = count_t / N, times N */
        std::vector<int32_t> d;
        std::vector<double> fs;
        for (int32_t t : members[g]) {
            d.push_back(table_dim[t]);
            fs.push_back(N > 0 ? cnt[t] / N : 0.0);
        }
        vp[g] = N > 0 ? oracle_calc_vparam((int32_t)d.size(), d.data(), fs.data(), N) : 0.0;
    }
    double mean = 0.0, mn = 0.0;
    for (int32_t g = 0; g < G; ++g) mean += vp[g];
    mean /= (double)G;
    mn = vp[0];
    for (int32_t g = 1; g < G; ++g) mn = std::min(mn, vp[g]);
    int32_t P = 0;
    for (int32_t g = 0; g < G; ++g) {
        int32_t shards = 1;
        if (split && vp[g] > mean && mn > 0.0) {
            double q = std::ceil(vp[g] / mn);
            shards = (int32_t)std::min<double>((double)members[g].size(), q);
            if (shards < 1) shards = 1;
        }
        /* round-robin by descending per-table vparam, ties ascending table index */
        std::vector<int32_t> ord = members[g];
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
            double va = (double)table_dim[a] * cnt[a], vb = (double)table_dim[b] * cnt[b];
            if (va != vb) return va > vb;
            return a < b;
        });
        for (size_t i = 0; i < ord.size(); ++i) table_to_pack[ord[i]] = P + (int32_t)(i % shards);
        for (int32_t s = 0; s < shards; ++s) {
            pack_dim[P + s] = dims[g];
            pack_rows[P + s] = 0;
        }
        P += shards;
    }
    for (int32_t t = 0; t < n_tables; ++t) { /* ascending table index within each pack */
        int32_t p = table_to_pack[t];
        table_base[t] = pack_rows[p];
        pack_rows[p] += table_rows[t];
    }
    for (int32_t f = 0; f < n_fields; ++f) field_to_pack[f] = table_to_pack[field_to_table[f]];
    *n_packs = P;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Forward (PAPER.md L213-215 SegmentReduction):
 *   out[b][col(f)+d] = sum_{j in seg(f,b)} W_t[row_j][d]   (ascending j, from +0.0f)
 *   mean: that sum / (float)len; an empty segment gives 0 (reading O5).
 * Tables are given unpacked: tables[t] is [V_t, D_t] row-major. */
int32_t oracle_forward(const oracle_model *m, const oracle_batch *bt, float *const *tables,
                       float *out, int64_t out_stride) {
    const int32_t F = m->n_fields, B = bt->batch;
    for (int32_t f = 0; f < F; ++f) {
        const int32_t t = m->field_to_table[f];
        const int32_t D = m->table_dim[t];
        for (int32_t b = 0; b < B; ++b) {
            const int32_t s0 = bt->offsets[(int64_t)f * B + b], s1 = bt->offsets[(int64_t)f * B + b + 1];
            float *o = out + (int64_t)b * out_stride + m->field_col[f];
            for (int32_t d = 0; d < D; ++d) {
                float acc = 0.0f;
                for (int32_t j = s0; j < s1; ++j) {
                    int64_t row;
                    int32_t st = oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0,
                                               m->table_rows[t], &row);
                    if (st) return st;
                    acc = acc + tables[t][row * D + d];
                }
                const int32_t len = s1 - s0;
                if (m->pool == OR_POOL_MEAN && len > 0) acc = acc / (float)len;
                o[d] = acc;
            }
        }
    }
    return OR_OK;
}

/* Rows a set of query segments needs (for row-sampled parity at full scale). */
int64_t oracle_segment_rows(const oracle_model *m, const oracle_batch *bt, int64_t n_q,
                            const int32_t *q_field, const int32_t *q_sample, int64_t cap,
                            int32_t *out_table, int64_t *out_row) {
    int64_t n = 0;
    const int32_t B = bt->batch;
    for (int64_t q = 0; q < n_q; ++q) {
        const int32_t f = q_field[q], b = q_sample[q], t = m->field_to_table[f];
        for (int32_t j = bt->offsets[(int64_t)f * B + b]; j < bt->offsets[(int64_t)f * B + b + 1]; ++j) {
            int64_t row;
            if (oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0, m->table_rows[t], &row))
                return OR_ID_RANGE;
            if (n < cap) { out_table[n] = t; out_row[n] = row; }
            ++n;
        }
    }
    return n;
}

/* Forward for selected segments only; rows come from a sparse (table,row)->values list
 * (values [n_rows, ld]).  Same arithmetic as oracle_forward. */
int32_t oracle_forward_sampled(const oracle_model *m, const oracle_batch *bt, int64_t n_rows,
                               const int32_t *r_table, const int64_t *r_row, const float *r_val,
                               int64_t ld, int64_t n_q, const int32_t *q_field,
                               const int32_t *q_sample, float *out_q /*[n_q, ld]*/) {
    std::unordered_map<uint64_t, int64_t> where;
    where.reserve((size_t)n_rows * 2 + 1);
    for (int64_t i = 0; i < n_rows; ++i) where[((uint64_t)r_table[i] << 48) ^ (uint64_t)r_row[i]] = i;
    const int32_t B = bt->batch;
    int32_t status = OR_OK;
    /* the segments are independent: the all-cores baseline build (-fopenmp, bench.py) splits them
     * over threads; every segment's sum is the same sequential loop either way */
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t q = 0; q < n_q; ++q) {
        const int32_t f = q_field[q], b = q_sample[q], t = m->field_to_table[f];
        const int32_t D = m->table_dim[t];
        const int32_t s0 = bt->offsets[(int64_t)f * B + b], s1 = bt->offsets[(int64_t)f * B + b + 1];
        for (int32_t d = 0; d < D; ++d) {
            float acc = 0.0f;
            for (int32_t j = s0; j < s1; ++j) {
                int64_t row;
                if (oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0, m->table_rows[t], &row)) {
                    status = OR_ID_RANGE;
                    break;
                }
                auto it = where.find(((uint64_t)t << 48) ^ (uint64_t)row);
                if (it == where.end()) {
                    status = OR_MISMATCH;
                    break;
                }
                acc = acc + r_val[it->second * ld + d];
            }
            const int32_t len = s1 - s0;
            if (m->pool == OR_POOL_MEAN && len > 0) acc = acc / (float)len;
            out_q[q * ld + d] = acc;
        }
    }
    return status;
}

/* ------------------------------------------------------------------------------------ */
/* K-Interleaving.
 * Eq. 3 (L433-436): Capacity_g = min_{op in layer} RBound_op / RParam_op, "the parameter volume
 * as the cost in embedding lookup and exchange" (L437-438): ops with RParam 0 do not bind.  */
double oracle_interleave_capacity(int32_t n_ops, const double *rbound, const double *rparam) {
    double c = INFINITY;
    for (int32_t i = 0; i < n_ops; ++i)
        if (rparam[i] > 0.0 && rbound[i] / rparam[i] < c) c = rbound[i] / rparam[i];
    return c;
}

/* The interleaving plan (reading O22), written out step by step:
 *  1. the "preset excluded embedding" tables (L444-447) form one pack per dim (ascending dim),
 *     numbered first, group -1 (no control dependencies on the other groups);
 *  2. every other dim group (ascending dim) has parameter volume V = sum_t dim_t * count_t (Eq. 1,
 *     count_t as in oracle_pack_plan); it becomes min(#tables, ceil(V / Capacity_g)) packs (1 if
 *     Capacity_g is not a positive finite number), tables dealt round-robin in descending
 *     dim_t * count_t (ties: ascending index) — each pack a packed operation within the capacity;
 *  3. groups of packed operations (L427-432): the packs, in order, are joined into a group while
 *     its volume stays <= Capacity_g; a pack that does not fit starts the next group;
 *  4. table_base: running row sum in ascending table index within each pack.
 * Returns the number of packs; *n_groups receives the number of groups (excluded packs not
 * counted). */
int32_t oracle_kinterleave_plan(int32_t n_fields, const int32_t *field_to_table, int32_t n_tables,
                                const int64_t *table_rows, const int32_t *table_dim,
                                const uint64_t *warmup_count, double capacity, const uint8_t *excluded,
                                int32_t *table_to_pack, int64_t *table_base, int32_t *pack_dim,
                                int64_t *pack_rows, int32_t *pack_group, int32_t *n_groups) {
    std::vector<double> cnt(n_tables, 0.0);
    for (int32_t f = 0; f < n_fields; ++f) cnt[field_to_table[f]] += 1.0;
    if (warmup_count)
        for (int32_t t = 0; t < n_tables; ++t) cnt[t] = (double)warmup_count[t];
    std::vector<int32_t> dims;
    for (int32_t t = 0; t < n_tables; ++t) dims.push_back(table_dim[t]);
    std::sort(dims.begin(), dims.end());
    dims.erase(std::unique(dims.begin(), dims.end()), dims.end());
    std::vector<double> pvol;
    int32_t P = 0;
    /* step 1 */
    for (int32_t d : dims) {
        bool any = false;
        double v = 0.0;
        for (int32_t t = 0; t < n_tables; ++t)
            if (excluded && excluded[t] && table_dim[t] == d) {
                table_to_pack[t] = P;
                v += (double)table_dim[t] * cnt[t];
                any = true;
            }
        if (any) {
            pack_dim[P] = d;
            pack_group[P] = -1;
            pvol.push_back(v);
            ++P;
        }
    }
    const int32_t n_ex = P;
    /* step 2 */
    for (int32_t d : dims) {
        std::vector<int32_t> ord;
        double V = 0.0;
        for (int32_t t = 0; t < n_tables; ++t)
            if (!(excluded && excluded[t]) && table_dim[t] == d) {
                ord.push_back(t);
                V += (double)table_dim[t] * cnt[t];
            }
        if (ord.empty()) continue;
        int32_t shards = 1;
        if (capacity > 0.0 && std::isfinite(capacity)) {
            double q = std::ceil(V / capacity);
            shards = (int32_t)std::min<double>((double)ord.size(), q);
            if (shards < 1) shards = 1;
        }
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
            double va = (double)table_dim[a] * cnt[a], vb = (double)table_dim[b] * cnt[b];
            if (va != vb) return va > vb;
            return a < b;
        });
        for (int32_t s = 0; s < shards; ++s) {
            pack_dim[P + s] = d;
            pvol.push_back(0.0);
        }
        for (size_t i = 0; i < ord.size(); ++i) {
            table_to_pack[ord[i]] = P + (int32_t)(i % shards);
            pvol[P + (int32_t)(i % shards)] += (double)table_dim[ord[i]] * cnt[ord[i]];
        }
        P += shards;
    }
    /* step 3 */
    int32_t g = -1;
    double in_group = 0.0;
    for (int32_t p = n_ex; p < P; ++p) {
        if (g == -1 || (in_group > 0.0 && in_group + pvol[p] > capacity)) {
            g += 1;
            in_group = 0.0;
        }
        pack_group[p] = g;
        in_group += pvol[p];
    }
    *n_groups = g + 1;
    /* step 4 */
    for (int32_t p = 0; p < P; ++p) pack_rows[p] = 0;
    for (int32_t t = 0; t < n_tables; ++t) {
        table_base[t] = pack_rows[table_to_pack[t]];
        pack_rows[table_to_pack[t]] += table_rows[t];
    }
    return P;
}

/* ------------------------------------------------------------------------------------ */
/* Intermediates of the packed operation (bit-exact targets).
 * Key stream of pack p on one rank (reading O2): the pack's fields in ascending field
 * index, then sample b, then j; key = table_base[t] + row. */
int64_t oracle_pack_key_stream(const oracle_model *m, const int32_t *field_to_pack,
                               const int64_t *table_base, const oracle_batch *bt, int32_t pack,
                               int64_t cap, int64_t *keys_out) {
    int64_t n = 0;
    const int32_t B = bt->batch;
    for (int32_t f = 0; f < m->n_fields; ++f) {
        if (field_to_pack[f] != pack) continue;
        const int32_t t = m->field_to_table[f];
        for (int32_t b = 0; b < B; ++b)
            for (int32_t j = bt->offsets[(int64_t)f * B + b]; j < bt->offsets[(int64_t)f * B + b + 1]; ++j) {
                int64_t row;
                if (oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0, m->table_rows[t], &row))
                    return OR_ID_RANGE;
                if (n < cap) keys_out[n] = table_base[t] + row;
                ++n;
            }
    }
    return n;
}

/* Unique (reading O1 = first-occurrence order):
 * uniq = distinct keys in order of first occurrence; inverse[i] = index of keys[i] in uniq. */
int64_t oracle_unique(int64_t n, const int64_t *keys, int64_t *uniq, int32_t *inverse) {
    std::unordered_map<int64_t, int32_t> seen;
    seen.reserve((size_t)n * 2 + 1);
    int64_t U = 0;
    for (int64_t i = 0; i < n; ++i) {
        auto it = seen.find(keys[i]);
        if (it == seen.end()) {
            seen.emplace(keys[i], (int32_t)U);
            uniq[U] = keys[i];
            inverse[i] = (int32_t)U;
            ++U;
        } else {
            inverse[i] = it->second;
        }
    }
    return U;
}

/* Partition (reading O3 = key mod W): per-owner lists in
 * unique order, concatenated by owner; counts[w] = list length; local_row = key div W. */
int32_t oracle_partition(int64_t U, const int64_t *uniq, int32_t W, int64_t *out_keys,
                         int64_t *out_local_row, int64_t *counts) {
    if (W < 1) return OR_INVALID;
    int64_t n = 0;
    for (int32_t w = 0; w < W; ++w) {
        counts[w] = 0;
        for (int64_t i = 0; i < U; ++i)
            if (uniq[i] % W == w) {
                out_keys[n] = uniq[i];
                out_local_row[n] = uniq[i] / W;
                ++n;
                ++counts[w];
            }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Backward + sparse update over the GLOBAL batch = the rank batches concatenated in rank
 * order (reading O6/O9).  For each table t and row:
 *   G_t[row] = sum over occurrences (r, f with table t in ascending f, b, j) of
 *              dY_r[b][col(f)+.]   (mean: dY_r[b][col(f)+.] / (float)len)
 * ("mirror image").  Each contribution is formed in fp32 (the paper's
 * precision: dY is fp32, mean divides in fp32), the sum is accumulated in fp64 in that order
 * and rounded once to fp32 (reading O6: the paper fixes fp32 for parameters and activations,
 * not the precision of the gradient reduction; fp64 accumulation makes G = fp32(exact sum)
 * up to 2^-53-relative error, independent of summation order).
 * Touched = rows with >= 1 occurrence.  Untouched rows are not written. */
struct GradAcc {
    std::vector<int64_t> order;                         /* rows in first-touch order */
    std::unordered_map<int64_t, std::vector<double>> g; /* row -> G (fp64 accumulator) */
};

static int32_t accumulate_grads(const oracle_model *m, int32_t R, const oracle_batch *batches,
                                std::vector<GradAcc> &acc) {
    acc.assign(m->n_tables, GradAcc());
    for (int32_t r = 0; r < R; ++r) {
        const oracle_batch *bt = &batches[r];
        const int32_t B = bt->batch;
        for (int32_t f = 0; f < m->n_fields; ++f) {
            const int32_t t = m->field_to_table[f];
            const int32_t D = m->table_dim[t];
            for (int32_t b = 0; b < B; ++b) {
                const int32_t s0 = bt->offsets[(int64_t)f * B + b], s1 = bt->offsets[(int64_t)f * B + b + 1];
                const int32_t len = s1 - s0;
                const float *dy = bt->dy + (int64_t)b * bt->dy_stride + m->field_col[f];
                for (int32_t j = s0; j < s1; ++j) {
                    int64_t row;
                    if (oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0,
                                      m->table_rows[t], &row))
                        return OR_ID_RANGE;
                    auto it = acc[t].g.find(row);
                    if (it == acc[t].g.end()) {
                        it = acc[t].g.emplace(row, std::vector<double>(D, 0.0)).first;
                        acc[t].order.push_back(row);
                    }
                    for (int32_t d = 0; d < D; ++d) {
                        float c = dy[d];
                        if (m->pool == OR_POOL_MEAN) c = c / (float)len; /* reading O7 */
                        it->second[d] = it->second[d] + (double)c;
                    }
                }
            }
        }
    }
    return OR_OK;
}

/* One row's optimizer update (readings O9, O10).
 * Adagrad (torch.optim.Adagrad sparse path):  acc = acc + g*g;  w = w - lr*(g/(sqrt(acc)+eps))
 * Lazy Adam (torch.optim.SparseAdam):         m = m + (g-m)*(1-b1);  v = v + (g*g-v)*(1-b2);
 *     w = w - ss*(m/(sqrt(v)+eps)),  ss = (float)(lr*sqrt(1-b2^t)/(1-b1^t)) computed in double. */
static void update_row(const oracle_opt *o, int64_t step, int32_t D, const float *g, float *w,
                       float *s1, float *s2) {
    if (o->kind == OR_OPT_ADAGRAD) {
        for (int32_t d = 0; d < D; ++d) {
            float a = s1[d] + g[d] * g[d];
            s1[d] = a;
            float q = g[d] / (std::sqrt(a) + o->eps);
            w[d] = w[d] - o->lr * q;
        }
    } else {
        const double bc1 = 1.0 - std::pow((double)o->beta1, (double)step);
        const double bc2 = 1.0 - std::pow((double)o->beta2, (double)step);
        const float ss = (float)((double)o->lr * std::sqrt(bc2) / bc1);
        const float omb1 = 1.0f - o->beta1, omb2 = 1.0f - o->beta2;
        for (int32_t d = 0; d < D; ++d) {
            float mo = s1[d], vo = s2[d];
            float mu = (g[d] - mo) * omb1;
            float vu = (g[d] * g[d] - vo) * omb2;
            float mn = mu + mo, vn = vu + vo;
            s1[d] = mn;
            s2[d] = vn;
            float q = mn / (std::sqrt(vn) + o->eps);
            w[d] = w[d] - ss * q;
        }
    }
}

int32_t oracle_backward_update(const oracle_model *m, int32_t R, const oracle_batch *batches,
                               float *const *tables, float *const *state1, float *const *state2,
                               const oracle_opt *opt, int64_t step) {
    std::vector<GradAcc> acc;
    int32_t st = accumulate_grads(m, R, batches, acc);
    if (st) return st;
    for (int32_t t = 0; t < m->n_tables; ++t) {
        const int32_t D = m->table_dim[t];
        for (int64_t row : acc[t].order) {
            const std::vector<double> &g64 = acc[t].g[row];
            std::vector<float> g(g64.begin(), g64.end()); /* one rounding to fp32 */
            update_row(opt, step, D, g.data(), tables[t] + row * D, state1[t] + row * D,
                       state2 ? (state2[t] ? state2[t] + row * D : nullptr) : nullptr);
        }
    }
    return OR_OK;
}

/* G for the whole batch of one table (dense [V_t, D_t], zero for untouched rows) and the
 * per-row occurrence count — small configs only. */
int32_t oracle_table_grad(const oracle_model *m, int32_t R, const oracle_batch *batches, int32_t t,
                          float *G, int64_t *count) {
    std::vector<GradAcc> acc;
    int32_t st = accumulate_grads(m, R, batches, acc);
    if (st) return st;
    const int32_t D = m->table_dim[t];
    std::memset(G, 0, sizeof(float) * (size_t)m->table_rows[t] * D);
    if (count) std::memset(count, 0, sizeof(int64_t) * (size_t)m->table_rows[t]);
    for (int64_t row : acc[t].order) {
        const std::vector<double> &g = acc[t].g[row];
        for (int32_t d = 0; d < D; ++d) G[row * D + d] = (float)g[d];
    }
    if (count) {
        for (int32_t r = 0; r < R; ++r) {
            const oracle_batch *bt = &batches[r];
            for (int32_t f = 0; f < m->n_fields; ++f) {
                if (m->field_to_table[f] != t) continue;
                for (int32_t j = bt->offsets[(int64_t)f * bt->batch]; j < bt->offsets[(int64_t)(f + 1) * bt->batch]; ++j) {
                    int64_t row;
                    oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0, m->table_rows[t], &row);
                    count[row] += 1;
                }
            }
        }
    }
    return OR_OK;
}

/* G for selected (table,row) pairs only (row-sampled parity at full scale).  Same order of
 * summation as accumulate_grads.  G [n_q, ld]; count [n_q] = occurrences (0 = untouched). */
int32_t oracle_row_grads(const oracle_model *m, int32_t R, const oracle_batch *batches, int64_t n_q,
                         const int32_t *q_table, const int64_t *q_row, int64_t ld, float *G,
                         int64_t *count) {
    std::unordered_map<uint64_t, int64_t> where;
    where.reserve((size_t)n_q * 2 + 1);
    std::vector<double> G64((size_t)n_q * ld, 0.0);
    for (int64_t q = 0; q < n_q; ++q) {
        where[((uint64_t)q_table[q] << 48) ^ (uint64_t)q_row[q]] = q;
        count[q] = 0;
    }
    int32_t status = OR_OK;
    /* the all-cores baseline build (-fopenmp, bench.py): every thread scans all occurrences in
     * the order above but accumulates only the queried rows it owns (q mod threads), so each
     * row's sum keeps the sequential order; without OpenMP this is the plain loop (1 thread) */
#pragma omp parallel
    {
        int nth = 1, tid = 0;
#ifdef _OPENMP
        nth = omp_get_num_threads();
        tid = omp_get_thread_num();
#endif
        for (int32_t r = 0; r < R; ++r) {
            const oracle_batch *bt = &batches[r];
            const int32_t B = bt->batch;
            for (int32_t f = 0; f < m->n_fields; ++f) {
                const int32_t t = m->field_to_table[f];
                const int32_t D = m->table_dim[t];
                for (int32_t b = 0; b < B; ++b) {
                    const int32_t s0 = bt->offsets[(int64_t)f * B + b], s1 = bt->offsets[(int64_t)f * B + b + 1];
                    const int32_t len = s1 - s0;
                    for (int32_t j = s0; j < s1; ++j) {
                        int64_t row;
                        if (oracle_row_of(m->id_mode, bt->ids[j], m->table_salt ? m->table_salt[t] : 0,
                                          m->table_rows[t], &row)) {
                            status = OR_ID_RANGE;
                            continue;
                        }
                        auto it = where.find(((uint64_t)t << 48) ^ (uint64_t)row);
                        if (it == where.end() || it->second % nth != tid) continue;
                        const float *dy = bt->dy + (int64_t)b * bt->dy_stride + m->field_col[f];
                        double *g = G64.data() + it->second * ld;
                        for (int32_t d = 0; d < D; ++d) {
                            float c = dy[d];
                            if (m->pool == OR_POOL_MEAN) c = c / (float)len;
                            g[d] = g[d] + (double)c;
                        }
                        count[it->second] += 1;
                    }
                }
            }
        }
    }
    if (status != OR_OK) return status;
    for (size_t i = 0; i < G64.size(); ++i) G[i] = (float)G64[i];
    return OR_OK;
}

/* Apply the optimizer to n rows given G (rows with count 0 are left untouched). */
int32_t oracle_apply_update(const oracle_opt *opt, int64_t step, int64_t n, int32_t D, int64_t ld,
                            const float *G, const int64_t *count, float *w, float *s1, float *s2) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {  /* rows are independent (all-cores build: split over threads) */
        if (count && count[i] == 0) continue;
        update_row(opt, step, D, G + i * ld, w + i * ld, s1 + i * ld, s2 ? s2 + i * ld : nullptr);
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Alg. 1 hot set: top-k(FCounter), k fixed by the size of
 * Hot-storage (L478).  Readings O11-O13: candidates sorted by (count desc, pack asc, key
 * asc); take the longest prefix whose summed row cost fits capacity_bytes (row cost of a
 * key = row_cost_bytes[pack]).  Keys with count 0 are never selected.  order_out receives
 * the selected candidate indices in that order; returns k. */
int64_t oracle_hot_select(int64_t n, const int32_t *pack, const int64_t *key, const uint64_t *count,
                          const int64_t *row_cost_bytes, uint64_t capacity_bytes, int64_t *order_out) {
    std::vector<int64_t> idx;
    for (int64_t i = 0; i < n; ++i)
        if (count[i] > 0) idx.push_back(i);
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
        if (count[a] != count[b]) return count[a] > count[b];
        if (pack[a] != pack[b]) return pack[a] < pack[b];
        if (key[a] != key[b]) return key[a] < key[b];
        return a < b;
    });
    uint64_t used = 0;
    int64_t k = 0;
    for (int64_t i : idx) {
        uint64_t c = (uint64_t)row_cost_bytes[pack[i]];
        if (used + c > capacity_bytes) break;
        used += c;
        order_out[k++] = i;
    }
    return k;
}

/* FCounter update for one rank-step (reading O11: post-unique counting): every distinct key
 * of the rank's pack stream adds 1.  counts is a dense per-pack-key array. */
int32_t oracle_fcounter_add(int64_t n, const int64_t *keys, uint64_t *counts) {
    std::unordered_set<int64_t> s;
    s.reserve((size_t)n * 2 + 1);
    for (int64_t i = 0; i < n; ++i)
        if (s.insert(keys[i]).second) counts[keys[i]] += 1;
    return OR_OK;
}

/* threads of the OpenMP build's parallel loops (the all-cores baseline): set / read; the plain build
 * always runs on 1 (no arithmetic here: the loops' results do not depend on the thread count) */
void oracle_set_threads(int32_t n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int32_t oracle_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

} /* extern "C" */
