// plan.h — host-side plan of the prefix tree (internal; not part of the C ABI).
//
// Tree: a node at depth t is a list of t active coordinates
// (k_1 < ... < k_t, levels l_m >= 2, node indices j_m); its excess is b = sum (l_m - 1) <= L and it
// IS the Smolyak point whose other coordinates sit at level 1 (the midpoint).  Children append
// (k' > k_t, l' in [2, L+1-b], j' in [0, nl[l'])).  Every node is one point of Eq 2.6 with
// coefficient coef[b]; the root (t = 0) is the all-midpoint point.  With merge (SG_MERGE_MIDPOINT)
// the per-level entries exclude the midpoint x = 1/2 and a node's coefficient is C'(t, b) (below):
// the node then stands for all its copies with extra midpoint coordinates at levels >= 2.
//
// Frontier t (t >= 1) = the extendable depth-t nodes (b <= L-1, k_t <= d-2), stored in segments
// (b, k) in b-major, k-minor order; inside segment (b', k') the children of source segment (b, k)
// sit at  TB[b][b'][k'] + nl[l'] * C_t(b,k) + j' * N_t(b,k) + i   (i = index inside (b, k)).
#pragma once
#include <cstdint>
#include <vector>

#define SG_MAX_L 19        // L + 1 <= 20 levels in the tables
#define SG_CC_MAX_LEVEL 12 // CC weights are O(n^2) quad cosines at plan time: level 12 (n = 2049)
                           // takes ~2 s, level 13 ~8 s, level 20 (n = 524289) hours; the oracle's
                           // independent generator has the same cost, so levels above 12 could
                           // not be checked bit for bit either (SG_EUNSUPPORTED)
#define SG_TRAP_MAX_LEVEL 20 // trapezoidal nodes / weights are exact dyadic rationals (O(n))
#define SG_GL_MAX_N 64
#define SG_GP_MAX_K 6      // Gauss-Patterson rules up to 2^6 - 1 = 63 points (levels <= 48)
#define SG_MAX_D ((1 << 20) - 1)
#define SG_META_KBITS 20
#ifndef GENERIC_POINT_COST
#define GENERIC_POINT_COST 1.0    // shard cost model: a point of a generic pass vs a k_leaf2 point.  With
                                  // pass L-2 concurrent with the fused pass (side stream) the generic
                                  // points overlap the fused ones; A/B of the N = 8 projection (graph
                                  // replays, r02l): config 5 1.8 -> 1.736 ms, 1.0 -> 1.692 ms (with
                                  // LEAF2_MID_COST 0); config 4 0.2878 -> 0.2843 ms
#endif
#ifndef LEAF2_MID_COST
#define LEAF2_MID_COST 0.0        // shard cost model: fixed cost of one k_leaf2 row run, in points
                                  // (r02l A/B on config 5 with GENERIC 1.0: 0 -> 1.692, 5 -> 1.706, 10 -> 1.741 ms)
#endif
#ifndef LEAF2_PPL
#define LEAF2_PPL 3   // parents per lane for a level-2 row that is one conjugate pair (k_leaf2_pairs;
                      // A/B on merged config 5 at 1 CTA/SM: 1 -> 3.51 ms, 2 -> 3.39, 3 -> 3.23, 4 -> 3.37)
#endif
#ifndef LEAF2_PPL3
#define LEAF2_PPL3 3  // parents per lane for the level-2 row {0, 1/2, 1} of the oscillatory kind (k_leaf2_sym3;
                      // A/B on config 5, 3 runs: 1 (k_leaf2, 2 CTAs/SM) 13.105 ms, 2 -> 13.41, 3 -> 13.053)
#endif
#ifndef LEAF2_RESIDENT_WARPS
#define LEAF2_RESIDENT_WARPS (148 * 24)   // persistent k_leaf2 warps (B200: 148 SMs x 16-24 warps)
#endif
#ifndef LEAF2_SPLIT_SHARE
#define LEAF2_SPLIT_SHARE 4   // split long tasks when one is > 1/SHARE of a resident warp's row share
#endif
#ifndef FRONT_SPLIT_MIN_BYTES
#define FRONT_SPLIT_MIN_BYTES (64.0 * 1024 * 1024)   // split a frontier pass writing at least this much
#endif
#ifndef LEAF2_PIECES_PER_WARP
#define LEAF2_PIECES_PER_WARP 2   // split pieces per resident warp on small shards (A/B on config 4 at N = 8:
                                  // 8 -> 0.314 ms, 4 -> 0.296, 2 -> 0.294, 1 -> 0.325; fewer, longer pieces
                                  // amortise the per-task fetch and k_mid prologue)
#endif
#ifndef LEAF2_MAX_PIECE
#define LEAF2_MAX_PIECE 1024      // longest split piece (rows)
#endif
#ifndef LEAF2_MIN_PIECE
#define LEAF2_MIN_PIECE 32        // shortest split piece (rows)
#endif
#ifndef LEAF2_GUIDE
#define LEAF2_GUIDE 1.0           // guided tail: task rows <= GUIDE x remaining rows / resident warps (0: off)
#endif
#ifndef LEAF2_GUIDE_MIN
#define LEAF2_GUIDE_MIN 32        // shortest guided-tail piece (rows)
#endif
#ifndef LEAF2_PRO_COST
#define LEAF2_PRO_COST 2          // schedule cost of one k_mid block's prologue, in rows (guided tail, sort)
#endif
#ifndef LEAF2_TASK_ROWS
#define LEAF2_TASK_ROWS 128   // minimum rows per fused task (grouping of short k_mid rows)
#endif

struct HostPlan {
    int d = 0, L = 0, rule = 0, kind = 0, form = 0;
    int nl[SG_MAX_L + 3] = {0};        // table entries per level (form-dependent)
    // rule entries per level l >= 2, concatenated: node x and weight (dd: hi, lo)
    std::vector<double> X, Whi, Wlo;
    int entry_off[SG_MAX_L + 3] = {0}; // offset of level l in X/W (level 2 at 0)
    int tab_off[SG_MAX_L + 3] = {0};   // offset (entries) of level l in the factor table: d*sum_{2<=m<l} nl[m]
    int tab_entries = 0;               // d * M0
    double coef[SG_MAX_L + 2] = {0};   // coefficient per excess e (combination / delta)
    // Node coefficient per (depth t, excess b), index t * (L + 1) + b, as double-double (hi, lo).
    // merge == 0: coef[b].  merge == 1 (SG_MERGE_MIDPOINT): the merged coefficient
    // C'(t, b) = sum_{e=b}^{L} coef[e] [z^{e-b}] M(z)^{d-t}, M(z) = 1 + sum_{l>=2} w^l(1/2) z^{l-1}.
    int merge = 0;
    std::vector<double> cm_hi, cm_lo;
    int64_t M0 = 0;                    // sum_{l=2}^{L+1} nl[l]
    int64_t range_lo = 0, range_hi = 0;
    bool include_root = true;
    int maxdepth = 0;                  // min(L, d)
    int nfront = 0;                    // deepest frontier depth = min(L-1, d-1) (>= 0)
    // frontier tables, index t = 1..nfront, each [L * d] (b * d + k)
    std::vector<std::vector<int64_t>> N, C, off;
    std::vector<int64_t> total;        // frontier sizes, index t
    std::vector<int64_t> JS;           // depth-1: first j1 of segment (b, k) in the range, [L * d]
    // pass t = 1..nfront-1 (writes frontier t+1): TB [L * L * d]  ((b * L + b') * d + k')
    std::vector<std::vector<int64_t>> TB;
    // pass statistics: index 0 = root pass, t = pass from frontier t
    std::vector<uint64_t> pass_terms, pass_written;
    uint64_t shard_points = 0, total_points = 0;
    // launch geometry
    std::vector<int> pass_nsplit;      // index t
    std::vector<int64_t> pass_ntasks, pass_blocks, pass_partial_off;
    // split frontier pass t (sg_kernels.cu, factor form, large frontiers): a write-only k_pass for the
    // stored children and a concurrent leaf-only k_leaf for the others, pass_blocks[t] slots each
    std::vector<char> pass_split;
    std::vector<int64_t> pass_front_slots;   // split pass t: k_front's chunks (one partial slot each)
    int64_t root_blocks = 0, total_partials = 0;
    size_t ws_front_bytes[2] = {0, 0}; // ping-pong frontier buffers (odd / even depth)
    int64_t ws_front_cap[2] = {0, 0};
    // Fused last two levels (L >= 3, d >= L, level-2 rows of 2 or 3 nodes): frontier L-1 is never
    // stored; the last pass builds each depth-(L-1) prefix from its depth-(L-2) parent (excess L-2,
    // all actives at level 2) on the fly.  Tasks: (k_mid, chunk of 32 parents with k < k_mid).
    bool fuse = false;
    int leaf2_ppl = 1;                 // parents per lane of the fused kernel (2: k_leaf2_pairs)
    int leaf2_groups = 1;              // lane groups of k_leaf2 (real kinds, few parents: 32 / G parents
                                       // per chunk, G k_mid groups per warp); 1 = lane per parent
    bool leaf2_sym3 = false;           // k_leaf2_sym3 (oscillatory, level-2 row {0, 1/2, 1} symmetric)
    // Source tasks: pass L-2 runs k_leaf2_sym3<SRC = true> over all its sources (the prefixes are the
    // stored sources themselves) instead of k_leaf — the excess-(L-1) sources' symmetric level-2
    // rows, the excess-(L-2) sources' level-2 rows (coefficient coef[L-1]) and level-3 rows
    // (SYM3_N3 nodes).  Three int64 per task like T2: first source index, ((-(k+1)) << 32) | (chunk
    // size | flags), (kp0 << 32) | kp1.
    bool leaf2_srctasks = false;
    std::vector<int64_t> T2S;
#define SRC_L3 (1 << 16)      // source task flag: walk the level-3 rows (SYM3_N3 nodes)
#define SRC_CPREV (1 << 17)   // source task flag: children have excess L-1 (coefficient coef[L-1])
#define SYM3_N3 5             // level-3 row length of the level-3 source tasks
#ifndef LEAF2_SRC_ROWS
#define LEAF2_SRC_ROWS 0      // source task rows per piece (0: automatic, see plan.cpp)
#endif
#define SYM3_RESIDENT_WARPS (148 * 8)   // persistent k_leaf2_sym3 warps (1 CTA of 8 warps per SM)
    // Fused tasks: (chunk of 32 parents, k_mid range [ka, kb)).  A chunk's k_mid values whose rows
    // (d - 1 - k_mid each) are short are grouped until a task holds >= LEAF2_TASK_ROWS rows, so the
    // per-task fixed cost (task fetch, parent load, warp reduction, partial store) is amortised.
    // Three int64 per task: first parent index (chunk * 32), (ka << 32) | kb, (kp0 << 32) | kp1 (the
    // row range; [0, d) unless a long single-k_mid task was split); sorted heavy-first.
    std::vector<int64_t> T2;
    // Sub[b * (d + 1) + (k + 1)] = Smolyak points (nonzero coefficient) in the subtree of a node
    // with excess b and last active coordinate k (k = -1: the root), the node itself included
    std::vector<uint64_t> Sub;
};

// K1 unranker: the index-th Smolyak point of the plan's shard in canonical order (the root if the
// shard includes it, then the depth-1 subtrees r1 = lo .. hi-1, each in preorder with children
// ordered by (k', l', j')).  Writes the t active (k, l, j) triples and the Eq 2.6 coefficient.
int host_unrank(const HostPlan &hp, uint64_t index, int *t, int *k, int *l, int *j, double *coef);

// Build rules, counts, shard range and launch geometry. Returns an sg_status code.
int host_plan_build(HostPlan &hp, int d, int L, int rule, int kind, int form, int merge, int rank, int world,
                    long long range_lo, long long range_hi, int fuse_mode = 1);   // 0 never, 1 auto, 2 always

// 1-D rule (level l) on [0,1] as doubles rounded from quad; returns n or -1.
int host_rule(int rule, int l, double *x, double *w);
int host_node_count(int rule, int l);
