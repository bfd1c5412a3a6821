// Host-side placement planners of libfailsafe_b200 (bit-exact with the
// reference planners; see failsafe_b200.h for the file:line map).
//
// Tables are flat int32 arrays: owner[layer * H + head] = GPU id or
// FS_REPLICATED; shard_owner[shard] = GPU id.  "Rank order" is ascending
// distinct GPU id (placement.py:69-73).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace {

int ranked(const int32_t *alive, int n, std::vector<int32_t> &out) {
    FS_CHECK_ARG(n >= 1 && alive != nullptr, "alive GPU set must be nonempty");
    out.assign(alive, alive + n);
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    for (int32_t g : out) FS_CHECK_ARG(g >= 0, "GPU ids must be nonnegative, got %d", g);
    return FS_OK;
}

// size of block b when `total` items are cut into n contiguous blocks with
// the `total % n` larger blocks first (placement.py:76-84, 94-114)
inline int block_size(int total, int n, int b) { return total / n + (b < total % n ? 1 : 0); }

}  // namespace

extern "C" int fs_plan_placement(int mode, int L, int H, const int32_t *alive, int n_alive,
                                 int32_t *owner) {
    std::vector<int32_t> ranks;
    if (int rc = ranked(alive, n_alive, ranks)) return rc;
    const int n = (int)ranks.size();
    FS_CHECK_ARG(L >= 1 && H >= 1, "num_layers and num_kv_heads must be positive");
    FS_CHECK_ARG(owner != nullptr, "null owner table");
    FS_CHECK_ARG(n <= H, "unsupported configuration: %d GPUs exceed %d KV heads", n, H);
    if (mode == FS_MODE_NAIVE || mode == FS_MODE_CYCLIC) {
        // block b of the contiguous split goes to rank (b + shift) % n
        for (int l = 0; l < L; ++l) {
            const int shift = mode == FS_MODE_CYCLIC ? l % n : 0;
            int head = 0;
            for (int b = 0; b < n; ++b) {
                const int32_t g = ranks[(b + shift) % n];
                for (int k = block_size(H, n, b); k > 0; --k) owner[(int64_t)l * H + head++] = g;
            }
        }
        return FS_OK;
    }
    FS_CHECK_ARG(mode == FS_MODE_HYBRID, "unknown placement mode %d", mode);
    // hybrid: rem = H % n heads starting at (l*rem) % H are replicated; the
    // other heads, in rotated order, are dealt H/n per rank, rank shifted by l
    const int base = H / n, rem = H % n;
    for (int l = 0; l < L; ++l) {
        int32_t *row = owner + (int64_t)l * H;
        const int first = (int)(((int64_t)l * rem) % H);
        for (int j = 0; j < rem; ++j) row[(first + j) % H] = FS_REPLICATED;
        for (int i = 0; i < H - rem; ++i) {
            const int head = (first + rem + i) % H;
            row[head] = ranks[(i / base + l) % n];
        }
    }
    return FS_OK;
}

extern "C" int fs_plan_ffn(int num_shards, const int32_t *alive, int n_alive, int32_t *shard_owner) {
    std::vector<int32_t> ranks;
    if (int rc = ranked(alive, n_alive, ranks)) return rc;
    const int n = (int)ranks.size();
    FS_CHECK_ARG(shard_owner != nullptr, "null shard table");
    FS_CHECK_ARG(num_shards >= n, "num_shards (%d) must be >= world size (%d)", num_shards, n);
    int s = 0;
    for (int b = 0; b < n; ++b)
        for (int k = block_size(num_shards, n, b); k > 0; --k) shard_owner[s++] = ranks[b];
    return FS_OK;
}

extern "C" int fs_plan_on_demand(int L, int H, const int32_t *owner, int num_shards,
                                 const int32_t *shard_owner, const int32_t *survivors, int n_surv,
                                 int32_t *new_owner, int32_t *new_shard_owner) {
    std::vector<int32_t> surv;
    if (int rc = ranked(survivors, n_surv, surv)) return rc;
    FS_CHECK_ARG(owner && new_owner && shard_owner && new_shard_owner, "null table");
    auto alive = [&](int32_t g) { return std::binary_search(surv.begin(), surv.end(), g); };
    for (int64_t i = 0; i < (int64_t)L * H; ++i) {
        const int32_t g = owner[i];
        new_owner[i] = (g == FS_REPLICATED || alive(g)) ? g : FS_REPLICATED;
    }
    // survivors keep their shards; lost shards (ascending) go to the survivor
    // with the fewest shards, lowest id on ties (recovery.py:323-340)
    std::vector<int64_t> count(surv.size(), 0);
    auto idx = [&](int32_t g) { return std::lower_bound(surv.begin(), surv.end(), g) - surv.begin(); };
    for (int s = 0; s < num_shards; ++s)
        if (alive(shard_owner[s])) ++count[idx(shard_owner[s])];
    for (int s = 0; s < num_shards; ++s) {
        if (alive(shard_owner[s])) {
            new_shard_owner[s] = shard_owner[s];
            continue;
        }
        size_t best = 0;
        for (size_t k = 1; k < surv.size(); ++k)
            if (count[k] < count[best]) best = k;
        new_shard_owner[s] = surv[best];
        ++count[best];
    }
    return FS_OK;
}

extern "C" int fs_kv_footprint(int L, int H, const int32_t *owner, const int32_t *alive, int n_alive,
                               const int64_t *tokens, const int32_t *routing, int n_req,
                               int64_t unit, int64_t *out_bytes) {
    FS_CHECK_ARG(owner && alive && out_bytes && n_alive >= 1, "bad arguments");
    FS_CHECK_ARG(n_req == 0 || tokens != nullptr, "null token counts");
    int64_t total = 0;
    for (int r = 0; r < n_req; ++r) total += tokens[r];
    bool has_dp = false;
    for (int64_t i = 0; i < (int64_t)L * H; ++i) has_dp |= owner[i] == FS_REPLICATED;
    FS_CHECK_ARG(!has_dp || n_req == 0 || routing != nullptr,
                 "routing is required for plans with replicated heads");
    for (int a = 0; a < n_alive; ++a) {
        const int32_t g = alive[a];
        int64_t routed = 0;
        if (has_dp)
            for (int r = 0; r < n_req; ++r) routed += routing[r] == g ? tokens[r] : 0;
        int64_t units = 0;
        for (int l = 0; l < L; ++l) {
            int tp = 0, dp = 0;
            for (int h = 0; h < H; ++h) {
                tp += owner[(int64_t)l * H + h] == g;
                dp += owner[(int64_t)l * H + h] == FS_REPLICATED;
            }
            units += tp * total + dp * routed;
        }
        out_bytes[a] = units * unit;
    }
    return FS_OK;
}
