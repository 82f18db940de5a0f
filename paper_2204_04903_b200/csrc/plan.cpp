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
