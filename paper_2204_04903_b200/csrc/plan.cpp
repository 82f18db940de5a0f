// plan.cpp — picasso_pack_plan: D-Packing with the Eq. 1 split.
// Host-only, pure.  See include/picasso.h for the contract and DESIGN.md (reading O14/O15).
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <vector>

#include "picasso.h"

extern "C" picasso_status picasso_pack_plan(int32_t n_fields, const int32_t *field_to_table, int32_t n_tables,
                                            const int64_t *table_rows, const int32_t *table_dim,
                                            const uint64_t *table_warmup_count, int32_t split,
                                            int32_t *field_to_pack, int32_t *table_to_pack, int64_t *table_base,
                                            int32_t *pack_dim, int64_t *pack_rows, int32_t *n_packs) {
    if (n_fields <= 0 || n_tables <= 0 || !field_to_table || !table_rows || !table_dim || !field_to_pack ||
        !table_to_pack || !table_base || !pack_dim || !pack_rows || !n_packs)
        return PICASSO_ERR_INVALID_ARG;
    for (int32_t t = 0; t < n_tables; ++t)
        if (table_rows[t] <= 0 || table_dim[t] <= 0) return PICASSO_ERR_INVALID_ARG;
    // ID occurrences per table from warm-up statistics (Eq. 1: N * ID_freq summed per table)
    std::vector<double> occ(n_tables, 0.0);
    for (int32_t f = 0; f < n_fields; ++f) {
        const int32_t t = field_to_table[f];
        if (t < 0 || t >= n_tables) return PICASSO_ERR_INVALID_ARG;
        if (!table_warmup_count) occ[t] += 1.0;
    }
    if (table_warmup_count)
        for (int32_t t = 0; t < n_tables; ++t) occ[t] = (double)table_warmup_count[t];

    // one group per distinct dim, ascending
    std::map<int32_t, std::vector<int32_t>> by_dim;
    for (int32_t t = 0; t < n_tables; ++t) by_dim[table_dim[t]].push_back(t);

    // CalcVParam(T) = N * sum_t t_dim * sum_ID ID_freq = sum_t t_dim * occ_t
    std::vector<double> vparam;
    for (auto &kv : by_dim) {
        double v = 0.0;
        for (int32_t t : kv.second) v += (double)kv.first * occ[t];
        vparam.push_back(v);
    }
    const double mean = std::accumulate(vparam.begin(), vparam.end(), 0.0) / (double)vparam.size();
    const double unit = *std::min_element(vparam.begin(), vparam.end());

    int32_t P = 0;
    size_t gi = 0;
    for (auto &kv : by_dim) {
        std::vector<int32_t> members = kv.second;  // ascending table index
        int32_t shards = 1;
        if (split >= 2) {  // K-Interleaving groups: every dim group dealt into `split` packs
            shards = (int32_t)std::min<size_t>(members.size(), (size_t)split);
        } else if (split && vparam[gi] > mean && unit > 0.0) {
            const double want = std::ceil(vparam[gi] / unit);
            shards = (int32_t)std::max(1.0, std::min((double)members.size(), want));
        }
        // deal tables round-robin in descending per-table parameter volume
        std::stable_sort(members.begin(), members.end(), [&](int32_t a, int32_t b) {
            const double va = (double)table_dim[a] * occ[a], vb = (double)table_dim[b] * occ[b];
            return va > vb;  // stable: ties keep ascending table index
        });
        for (size_t i = 0; i < members.size(); ++i) table_to_pack[members[i]] = P + (int32_t)(i % (size_t)shards);
        for (int32_t s = 0; s < shards; ++s) {
            pack_dim[P + s] = kv.first;
            pack_rows[P + s] = 0;
        }
        P += shards;
        ++gi;
    }
    for (int32_t t = 0; t < n_tables; ++t) {  // running row offset, ascending table index
        table_base[t] = pack_rows[table_to_pack[t]];
        pack_rows[table_to_pack[t]] += table_rows[t];
    }
    for (int32_t f = 0; f < n_fields; ++f) field_to_pack[f] = table_to_pack[field_to_table[f]];
    *n_packs = P;
    return PICASSO_OK;
}

// Eq. 3: Capacity_g = min over ops of RBound_op / RParam_op, in parameters
// per step ("we simply treat the parameter volume as the cost", L437-438).  Ops whose RParam is
// 0 never bind; none binding gives +inf (one group).
extern "C" picasso_status picasso_interleave_capacity(int32_t n_ops, const double *rbound, const double *rparam,
                                                      double *capacity) {
    if (n_ops <= 0 || !rbound || !rparam || !capacity) return PICASSO_ERR_INVALID_ARG;
    double c = INFINITY;
    for (int32_t i = 0; i < n_ops; ++i) {
        if (!(rbound[i] >= 0.0) || !(rparam[i] >= 0.0)) return PICASSO_ERR_INVALID_ARG;
        if (rparam[i] > 0.0) c = std::min(c, rbound[i] / rparam[i]);
    }
    *capacity = c;
    return PICASSO_OK;
}

// K-Interleaving plan (reading O22): D-Packing whose dim groups are
// cut into packs of at most Capacity_g parameters per step, packs then joined in order into
// interleaving groups of at most Capacity_g, and the preset-excluded tables' packs ahead of
// every group, outside the chain (group -1).
extern "C" picasso_status picasso_pack_plan_kinterleave(
    int32_t n_fields, const int32_t *field_to_table, int32_t n_tables, const int64_t *table_rows,
    const int32_t *table_dim, const uint64_t *table_warmup_count, double capacity_g, const uint8_t *excluded,
    int32_t *field_to_pack, int32_t *table_to_pack, int64_t *table_base, int32_t *pack_dim, int64_t *pack_rows,
    int32_t *pack_group, int32_t *n_packs, int32_t *n_groups) {
    if (n_fields <= 0 || n_tables <= 0 || !field_to_table || !table_rows || !table_dim || !field_to_pack ||
        !table_to_pack || !table_base || !pack_dim || !pack_rows || !pack_group || !n_packs || !n_groups ||
        std::isnan(capacity_g))
        return PICASSO_ERR_INVALID_ARG;
    for (int32_t t = 0; t < n_tables; ++t)
        if (table_rows[t] <= 0 || table_dim[t] <= 0) return PICASSO_ERR_INVALID_ARG;
    std::vector<double> occ(n_tables, 0.0);
    for (int32_t f = 0; f < n_fields; ++f) {
        const int32_t t = field_to_table[f];
        if (t < 0 || t >= n_tables) return PICASSO_ERR_INVALID_ARG;
        if (!table_warmup_count) occ[t] += 1.0;
    }
    if (table_warmup_count)
        for (int32_t t = 0; t < n_tables; ++t) occ[t] = (double)table_warmup_count[t];
    auto vol = [&](int32_t t) { return (double)table_dim[t] * occ[t]; };  // Eq. 1 per table

    int32_t P = 0;
    std::vector<double> pvol;
    // 1. preset-excluded tables: one pack per dim, ahead of the chain
    std::map<int32_t, std::vector<int32_t>> ex, in;
    for (int32_t t = 0; t < n_tables; ++t) ((excluded && excluded[t]) ? ex : in)[table_dim[t]].push_back(t);
    for (auto &kv : ex) {
        for (int32_t t : kv.second) table_to_pack[t] = P;
        double v = 0.0;
        for (int32_t t : kv.second) v += vol(t);
        pack_dim[P] = kv.first;
        pack_group[P] = -1;
        pvol.push_back(v);
        ++P;
    }
    // 2. the other dim groups, each cut into ceil(vparam / Capacity_g) packs (<= its tables),
    //    tables dealt round-robin by descending volume (ties: ascending index, as Eq. 1's split)
    for (auto &kv : in) {
        std::vector<int32_t> members = kv.second;
        double V = 0.0;
        for (int32_t t : members) V += vol(t);
        int32_t shards = 1;
        if (capacity_g > 0.0 && std::isfinite(capacity_g))
            shards = (int32_t)std::max(1.0, std::min((double)members.size(), std::ceil(V / capacity_g)));
        std::stable_sort(members.begin(), members.end(), [&](int32_t a, int32_t b) { return vol(a) > vol(b); });
        std::vector<double> v(shards, 0.0);
        for (size_t i = 0; i < members.size(); ++i) {
            table_to_pack[members[i]] = P + (int32_t)(i % (size_t)shards);
            v[i % (size_t)shards] += vol(members[i]);
        }
        for (int32_t s = 0; s < shards; ++s) {
            pack_dim[P + s] = kv.first;
            pvol.push_back(v[s]);
        }
        P += shards;
    }
    // 3. interleaving groups: packs joined in order while the group stays within Capacity_g
    int32_t g = -1;
    double cur = 0.0;
    for (int32_t p = 0; p < P; ++p) {
        if (p < (int32_t)ex.size()) continue;  // preset excluded
        if (g < 0 || (cur > 0.0 && cur + pvol[p] > capacity_g)) {
            ++g;
            cur = 0.0;
        }
        pack_group[p] = g;
        cur += pvol[p];
    }
    for (int32_t p = 0; p < P; ++p) pack_rows[p] = 0;
    for (int32_t t = 0; t < n_tables; ++t) {
        table_base[t] = pack_rows[table_to_pack[t]];
        pack_rows[table_to_pack[t]] += table_rows[t];
    }
    for (int32_t f = 0; f < n_fields; ++f) field_to_pack[f] = table_to_pack[field_to_table[f]];
    *n_packs = P;
    *n_groups = g + 1;
    return PICASSO_OK;
}
