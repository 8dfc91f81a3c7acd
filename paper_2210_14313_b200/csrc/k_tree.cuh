// k_tree.cuh — K2/K3: the prefix-tree passes (root, frontier writer, generic / single-level / fused leaf kernels)
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

// ---------------------------------------------------------------------------------------------
// Root pass: every depth-1 point (k1, l1, j1) of this shard, one thread each.
// ---------------------------------------------------------------------------------------------
// One depth-1 point r1 (lexicographic rank in [R.lo, R.hi)): its term, and its frontier-1 record if
// it is extendable.
template <bool CPLX>
__device__ __forceinline__ dd root_node(const DevPlan &P, const RootArgs &R, long long r1) {
    dd tot = {0.0, 0.0};
    if (r1 < R.hi) {
        const int k1 = (int)(r1 / P.M0);
        int rem = (int)(r1 - (long long)k1 * P.M0);
        int l1 = 2;
        while (rem >= P.nl[l1]) {
            rem -= P.nl[l1];
            ++l1;
        }
        const int j1 = rem;
        const int ti = P.tab_off[l1] + k1 * P.nl[l1] + j1;
        const dd Br = {P.base[0], P.base[1]};
        const double2 fr = P.Fre[ti];
        dd cr, ci = {0.0, 0.0};
        if (CPLX) {
            const dd Bi = {P.base[2], P.base[3]};
            const double2 fi = P.Fim[ti];
            cdd ch = cdd_mul(cdd{Br, Bi}, cdd{dd{fr.x, fr.y}, dd{fi.x, fi.y}});
            cr = ch.re;
            ci = ch.im;
        } else {
            cr = dd_mul(Br, dd{fr.x, fr.y});
        }
        const int b1 = l1 - 1;
        tot = coef_mul(P, cr, 1, b1);
        if (P.nfront >= 1 && b1 <= P.L - 1 && k1 <= P.d - 2) {
            const long long seg = (long long)b1 * P.d + k1;
            const long long o = R.off1[seg] + j1 - R.JS[seg];
            SG_DST(R, dst_re, o) = make_double2(cr.hi, cr.lo);
            if (CPLX) SG_DST(R, dst_im, o) = make_double2(ci.hi, ci.lo);
            SG_DST(R, dst_meta, o) = ((uint32_t)b1 << SG_META_KBITS) | (uint32_t)k1;
        }
    }
    return tot;
}

template <bool CPLX>
__global__ void __launch_bounds__(256) k_root(const DevPlan P, const RootArgs R) {
    const long long r1 = R.lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    dd s = block_reduce_dd<8>(root_node<CPLX>(P, R, r1));
    if (threadIdx.x == 0) SG_PART(R.partials, blockIdx.x) = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// Pass t >= 1 (K3 leaf + K2 frontier): warp task = (32 consecutive frontier-t nodes, a k' range).
// Lane = one parent prefix, held in registers; the loop over its children (k', l', j') reads the
// factor table at warp-uniform addresses (one broadcast transaction per load).
// ---------------------------------------------------------------------------------------------
#ifndef LEAF_ROW_UNROLL
#define LEAF_ROW_UNROLL 2   // row-loop unrolling in k_leaf (A/B: c5 pass 2 0.629 -> 0.602 ms with NJ = 5)
#endif
constexpr int kRowUnroll = LEAF_ROW_UNROLL;
#ifndef LEAF_SYM_FOLD
#define LEAF_SYM_FOLD 4   // rows between folds in the symmetric-row path (A/B on c5: error 5.1e-21 at 4, 1.4e-20 at 16; time +0.2%)
#endif
#ifndef FOLD
#define FOLD 16   // rows between folds of acc_lo onto the grid (A/B: 32 is 0.8% faster on c5 but triples its error, 3e-20 vs 1e-20)
#endif
#ifndef LEAF_MINB
#define LEAF_MINB 3
#endif

struct LeafAcc {
    double h, l;
};

// Biased grid accumulator (all leaf kernels).  The lane's high accumulator a.h starts at sigma =
// 1.5 * 2^m (2^m > 2 * bound on the sum of |P F| over the lane's children) and stays inside the
// binade [2^m, 2^(m+1)), where the double grid is u = ulp(sigma).  fma(P.hi, F.hi, a.h) therefore adds
// P.hi * F.hi rounded ONCE to the grid, exactly; the grid part h = new - old is exact (Sterbenz), and
// the remainder P.hi*F.hi - h (|.| <= u/2) and the cross terms P.hi*F.lo + P.lo*F.hi go to a.l by
// FMAs.  The lane result is (a.h - sigma) + a.l.  One FP64 instruction per product fewer than
// forming h = fma(P.hi, F.hi, sigma) - sigma and adding it.
template <bool CPLX>
__device__ __forceinline__ void leaf_term(const dd &er, const dd &ei, const double2 f, const double2 fi,
                                          LeafAcc &a) {
    if (!CPLX) {
        const double a1 = fma(er.hi, f.x, a.h);
        const double h = a1 - a.h;
        a.h = a1;
        a.l += fma(er.hi, f.x, -h);
        a.l = fma(er.hi, f.y, a.l);
        a.l = fma(er.lo, f.x, a.l);
    } else {
        // Re((er + i ei)(f + i fi)) = er f - ei fi, both grid parts added to a.h in turn
        const double a1 = fma(er.hi, f.x, a.h);
        const double h1 = a1 - a.h;
        const double a2 = fma(-ei.hi, fi.x, a1);
        const double h2 = a2 - a1;
        a.h = a2;
        a.l += fma(er.hi, f.x, -h1) + fma(-ei.hi, fi.x, -h2);
        a.l = fma(er.hi, f.y, a.l);
        a.l = fma(er.lo, f.x, a.l);
        a.l = fma(-ei.hi, fi.y, a.l);
        a.l = fma(-ei.lo, fi.x, a.l);
    }
}

__device__ __forceinline__ void leaf_fold(LeafAcc &a, double sigma) {
    const double t = (a.l + sigma) - sigma;
    a.h += t;
    a.l -= t;
}

// Leaf term for a node whose factor is REAL (imaginary part exactly 0): the midpoint node x = 1/2 of
// a level (E_k(1/2) = 1 for every kind, so F = w exactly real).  Re(P F) = P.re F: 7 FP64
// instructions instead of 14 for the oscillatory kind; bitwise the same value the general formula
// gives with F.im = 0 (every dropped term is an exact zero).
// CZ: the factor's low part is exactly 0 (combination form: F = w * 1), its cross term drops.
template <bool CZ = false>
__device__ __forceinline__ void leaf_real_factor_term(const dd &er, const double2 f, double &ah, double &al) {
    const double a1 = fma(er.hi, f.x, ah);   // biased accumulator (leaf_term)
    const double h = a1 - ah;
    ah = a1;
    double c = fma(er.lo, f.x, fma(er.hi, f.x, -h));
    if (!CZ) c = fma(er.hi, f.y, c);
    al += c;
}

// Symmetric pair (x_0 = 1 - x_2, w_0 = w_2; oscillatory): F_0 = conj(F_2) exactly, so the two
// points' terms Re(P F_0) = A + B and Re(P F_2) = A - B share the products A = P.re F_2.re and
// B = P.im F_2.im (their grid parts, remainders and cross terms); each point's term is still formed
// and accumulated on its own: node 0 adds the grid parts of A and B in turn (biased accumulator,
// leaf_term), node 2 forms h_A - h_B and adds it.  16 FP64 instructions for the two points.
__device__ __forceinline__ void leaf_sym_pair_terms(const dd &er, const dd &ei, const double2 f, const double2 g,
                                                    double &ah, double &al) {
    const double a1 = fma(er.hi, f.x, ah);
    const double h1 = a1 - ah;
    const double a2 = fma(ei.hi, g.x, a1);   // node 0: A + B
    const double h2 = a2 - a1;
    const double cA = fma(er.lo, f.x, fma(er.hi, f.y, fma(er.hi, f.x, -h1)));
    const double cB = fma(ei.lo, g.x, fma(ei.hi, g.y, fma(ei.hi, g.x, -h2)));
    al += cA + cB;
    ah = a2 + (h1 - h2);                     // node 2: A - B
    al += cA - cB;
}


// One level of the frontier writer's children for a lane: rows kp in [kb, ks1) (kp > k), the NJ
// nodes of each row unrolled (NJ = 0: runtime n).  Every child is a Smolyak point (biased grid
// accumulator term); children with excess bp <= L-1 and kp <= d-2 are also stored to frontier t+1
// (dd product P F; coalesced: consecutive lanes = consecutive records of a segment).
struct PassLevel {
    int kb, ks1, k;
    bool lv, wr;
    int b, bp;
    long long wbase, Nseg;
    const double2 *Fr, *Fi;
};

template <bool CPLX, bool WRITE, int NJ>
__device__ __forceinline__ void pass_level(const DevPlan &P, const PassArgs &A, const PassLevel &V, const dd &pr,
                                           const dd &pim, double sigma, LeafAcc &acc, int nrt = 0) {
    const int n = NJ > 0 ? NJ : nrt;
    const int d = P.d, L = P.L;
    int nfold = 0;
    for (int kp = V.kb; kp < V.ks1; ++kp) {
        const bool kv = V.lv && (kp > V.k);
        const dd er = kv ? pr : dd{0.0, 0.0};
        const dd ei = kv ? pim : dd{0.0, 0.0};
        const bool wk = WRITE && V.wr && kv && (kp <= d - 2);
        long long tb = 0;
        if (WRITE && wk) tb = A.TB[((long long)V.b * L + V.bp) * d + kp] + V.wbase;
        const double2 *fr_row = V.Fr + (long long)kp * n;
        const double2 *fi_row = CPLX ? V.Fi + (long long)kp * n : nullptr;
#pragma unroll
        for (int j = 0; j < (NJ > 0 ? NJ : n); ++j) {
            const double2 f = fr_row[j];
            const double2 fi = CPLX ? fi_row[j] : make_double2(0.0, 0.0);
            leaf_term<CPLX>(er, ei, f, fi, acc);
            if (WRITE && wk) {
                // the stored child product P F in dd (complex for the oscillatory kind)
                const long long o = tb + (long long)j * V.Nseg;
                double p1, e1;
                dd_mul_pe(er, dd{f.x, f.y}, p1, e1);
                if (!CPLX) {
                    const dd ch = dd_norm(p1, e1);
                    SG_DST(A, dst_re, o) = make_double2(ch.hi, ch.lo);
                } else {
                    double p2, e2, p3, e3, p4, e4;
                    dd_mul_pe(ei, dd{fi.x, fi.y}, p2, e2);
                    dd_mul_pe(er, dd{fi.x, fi.y}, p3, e3);
                    dd_mul_pe(ei, dd{f.x, f.y}, p4, e4);
                    const dd cre = dd_combine_pe(p1, e1, -p2, -e2), cim = dd_combine_pe(p3, e3, p4, e4);
                    SG_DST(A, dst_re, o) = make_double2(cre.hi, cre.lo);
                    SG_DST(A, dst_im, o) = make_double2(cim.hi, cim.lo);
                }
                SG_DST(A, dst_meta, o) = ((uint32_t)V.bp << SG_META_KBITS) | (uint32_t)kp;
            }
        }
        if (++nfold == FOLD) {
            nfold = 0;
            leaf_fold(acc, sigma);
        }
    }
}

// Symmetric oscillatory row (P.symmask): conjugate node pairs share the products of their terms
// (leaf_sym_pair_terms) and of their stored child products (cdd_mul_conj_pair); the midpoint
// (odd NJ) has a real factor.
template <bool WRITE, int NJ>
__device__ __forceinline__ void pass_level_sym(const DevPlan &P, const PassArgs &A, const PassLevel &V, const dd &pr,
                                               const dd &pim, double sigma, LeafAcc &acc) {
    constexpr int NP = NJ / 2;
    const int d = P.d, L = P.L;
    int nfold = 0;
    for (int kp = V.kb; kp < V.ks1; ++kp) {
        const bool kv = V.lv && (kp > V.k);
        const dd er = kv ? pr : dd{0.0, 0.0};
        const dd ei = kv ? pim : dd{0.0, 0.0};
        const bool wk = WRITE && V.wr && kv && (kp <= d - 2);
        long long tb = 0;
        if (WRITE && wk) tb = A.TB[((long long)V.b * L + V.bp) * d + kp] + V.wbase;
        const double2 *fr_row = V.Fr + (long long)kp * NJ;
        const double2 *fi_row = V.Fi + (long long)kp * NJ;
        const uint32_t meta = ((uint32_t)V.bp << SG_META_KBITS) | (uint32_t)kp;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int ju = NJ - 1 - q;
            const double2 f = fr_row[ju], g = fi_row[ju];
            leaf_sym_pair_terms(er, ei, f, g, acc.h, acc.l);
            if (WRITE && wk) {
                cdd cu, cl;
                cdd_mul_conj_pair(cdd{er, ei}, cdd{dd{f.x, f.y}, dd{g.x, g.y}}, cu, cl);
                const long long ou = tb + (long long)ju * V.Nseg, ol = tb + (long long)q * V.Nseg;
                SG_DST(A, dst_re, ou) = make_double2(cu.re.hi, cu.re.lo);
                SG_DST(A, dst_im, ou) = make_double2(cu.im.hi, cu.im.lo);
                SG_DST(A, dst_meta, ou) = meta;
                SG_DST(A, dst_re, ol) = make_double2(cl.re.hi, cl.re.lo);
                SG_DST(A, dst_im, ol) = make_double2(cl.im.hi, cl.im.lo);
                SG_DST(A, dst_meta, ol) = meta;
            }
        }
        if constexpr (NJ % 2 == 1) {
            const double2 w = fr_row[NP];
            leaf_real_factor_term<false>(er, w, acc.h, acc.l);
            if (WRITE && wk) {
                const long long oc = tb + (long long)NP * V.Nseg;
                const dd cr = dd_mul(er, dd{w.x, w.y}), ci = dd_mul(ei, dd{w.x, w.y});
                SG_DST(A, dst_re, oc) = make_double2(cr.hi, cr.lo);
                SG_DST(A, dst_im, oc) = make_double2(ci.hi, ci.lo);
                SG_DST(A, dst_meta, oc) = meta;
            }
        }
        if (++nfold == LEAF_SYM_FOLD) {
            nfold = 0;
            leaf_fold(acc, sigma);
        }
    }
}

#ifndef PASS_MINB
#define PASS_MINB 3   // CTAs/SM bound of k_pass
#endif
template <bool CPLX, bool WRITE>
__global__ void __launch_bounds__(PASS_THREADS, PASS_MINB) k_pass(const DevPlan P, const PassArgs A) {
    // factor levels 2 .. A.stage_lmax staged in shared memory (same layout as the table: level l at
    // tab_off[l] - tab_off[2]); the row loads of the level loop then cost shared-memory latency
    // instead of an L1/L2 round trip per row (ncu r02p: long-scoreboard stalls on those loads were the
    // first limiter of this kernel)
    extern __shared__ double2 fsm[];
    if (A.stage_lmax >= 2) {
        const double2 *gr = P.Fre + P.tab_off[2];
        const double2 *gi = CPLX ? P.Fim + P.tab_off[2] : nullptr;
        for (int i = threadIdx.x; i < A.stage_entries; i += blockDim.x) {
            fsm[i] = gr[i];
            if (CPLX) fsm[A.stage_entries + i] = gi[i];
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * WPB + wib;
    dd tot = {0.0, 0.0};
    if (task < A.ntasks) {
        const int d = P.d, L = P.L;
        const long long chunk = task / A.nsplit;
        const int split = (int)(task - chunk * A.nsplit);
        const long long g = chunk * 32 + lane;
        const bool valid = g < A.nsrc;
        int b = L, k = d;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (valid) {
            const uint32_t m = SG_SRC(A, src_meta, g);
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = SG_SRC(A, src_re, g);
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = SG_SRC(A, src_im, g);
                pim = dd{vi.x, vi.y};
            }
        }
        const int ks0 = (int)((long long)split * d / A.nsplit);
        const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
        const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
        const int bmin = __reduce_min_sync(0xffffffffu, b);
        long long iseg = 0, Nseg = 0, Cseg = 0;
        if (WRITE && valid) {
            const long long s = (long long)b * d + k;
            iseg = g - A.offT[s];
            Nseg = A.NT[s];
            Cseg = A.CT[s];
        }
        const double pabs = fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0);
        const int kb = max(ks0, kmin + 1);
        for (int lp = 2; lp <= L + 1 - bmin; ++lp) {
            const bool lv = valid && (lp <= L + 1 - b);
            const int n = P.nl[lp];
            const int bp = b + lp - 1;
            const bool staged = lp <= A.stage_lmax;
            const double2 *Fr = staged ? fsm + (P.tab_off[lp] - P.tab_off[2]) : P.Fre + P.tab_off[lp];
            const double2 *Fi = CPLX ? (staged ? fsm + A.stage_entries + (P.tab_off[lp] - P.tab_off[2])
                                               : P.Fim + P.tab_off[lp])
                                     : nullptr;
            const bool wr = WRITE && lv && (bp <= L - 1);
            const long long wbase = (long long)n * Cseg + iseg;
            // biased grid accumulator (leaf_term): sigma = 1.5 * 2^m > 2 * bound on the lane's
            // children of this level, from the suffix table SA
            const double bound = lv ? pabs * P.SA[(long long)lp * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20) : 0.0;
            const double sigma = grid_sigma(bound);
            LeafAcc acc = {sigma, 0.0};
            PassLevel L0 = {kb, ks1, k, lv, wr, b, bp, wbase, Nseg, Fr, Fi};
            const bool sym = CPLX && ((P.symmask >> lp) & 1);
            if (sym && n == 3) pass_level_sym<WRITE, 3>(P, A, L0, pr, pim, sigma, acc);
            else if (sym && n == 5) pass_level_sym<WRITE, 5>(P, A, L0, pr, pim, sigma, acc);
            else if (sym && n == 2) pass_level_sym<WRITE, 2>(P, A, L0, pr, pim, sigma, acc);
            else switch (n) {
            case 2: pass_level<CPLX, WRITE, 2>(P, A, L0, pr, pim, sigma, acc); break;
            case 3: pass_level<CPLX, WRITE, 3>(P, A, L0, pr, pim, sigma, acc); break;
            case 5: pass_level<CPLX, WRITE, 5>(P, A, L0, pr, pim, sigma, acc); break;
            default: pass_level<CPLX, WRITE, 0>(P, A, L0, pr, pim, sigma, acc, n); break;
            }
            if (lv) tot = dd_add(tot, coef_mul(P, dd_norm(acc.h - sigma, acc.l), A.t + 1, bp));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) SG_PART(A.partials, blockIdx.x) = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// Leaf-only pass (no extendable children), generic levels: k_leaf (config 5 pass 2: 7.2e8 points).
//
// Same task mapping as k_pass; the accumulation is the biased grid accumulator (leaf_term): every
// product P.hi F.hi is rounded once onto the grid of the lane's sigma and added exactly; the
// remainder and the cross terms go to acc_lo by FMAs (folded back onto the grid every FOLD rows).
// 6 FP64 instructions per real leaf and 12 per oscillatory leaf (symmetric rows: 7-8 via shared
// conjugate-pair products), against 12 / 24 with TwoSum + dd products.
// Children (k', j') are walked row by row (k'), NJ nodes per row unrolled with one accumulator pair
// per node (or per symmetric pair) for ILP; rows with k' <= max lane k of the warp are predicated
// (segment boundaries).
// ---------------------------------------------------------------------------------------------

template <bool CPLX, int NJ>
__device__ __forceinline__ void leaf_rows(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                          int n, int kp0, int kp1, int klane, bool pred, const dd &pr,
                                          const dd &pim, double sigma, LeafAcc (&acc)[NJ > 0 ? NJ : 1]) {
    const int nj = NJ > 0 ? NJ : n;
    for (int kp = kp0; kp < kp1;) {
        const int ke = min(kp1, kp + FOLD);
        #pragma unroll kRowUnroll
        for (; kp < ke; ++kp) {
            const bool kv = !pred || kp > klane;
            const dd er = kv ? pr : dd{0.0, 0.0};
            const dd ei = (CPLX && kv) ? pim : dd{0.0, 0.0};
            const double2 *fr = Fr + (long long)kp * nj;
            const double2 *fi = CPLX ? Fi + (long long)kp * nj : nullptr;
            if (NJ > 0) {
#pragma unroll
                for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) {
                    const double2 f = __ldg(fr + j);
                    const double2 g = CPLX ? __ldg(fi + j) : make_double2(0.0, 0.0);
                    leaf_term<CPLX>(er, ei, f, g, acc[j]);
                }
            } else {
                for (int j = 0; j < nj; ++j) {
                    const double2 f = __ldg(fr + j);
                    const double2 g = CPLX ? __ldg(fi + j) : make_double2(0.0, 0.0);
                    leaf_term<CPLX>(er, ei, f, g, acc[0]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) leaf_fold(acc[j], sigma);
    }
}

template <bool CPLX, int NJ>
__device__ __forceinline__ dd leaf_level(const double2 *Fr, const double2 *Fi, int n, int kb, int kmain,
                                         int ks1, int k, const dd &pr, const dd &pim, double sigma) {
    LeafAcc acc[NJ > 0 ? NJ : 1];
#pragma unroll
    for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) acc[j] = LeafAcc{sigma, 0.0};   // biased accumulator
    // boundary rows (some lanes of the warp have k >= k'), then the unpredicated main rows
    leaf_rows<CPLX, NJ>(Fr, Fi, n, kb, min(kmain, ks1), k, true, pr, pim, sigma, acc);
    leaf_rows<CPLX, NJ>(Fr, Fi, n, max(kb, kmain), ks1, k, false, pr, pim, sigma, acc);
    dd s = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) s = dd_add(s, dd_norm(acc[j].h - sigma, acc[j].l));
    return s;
}

// Symmetric oscillatory row of NJ nodes: pairs (j, NJ-1-j) share their products
// (leaf_sym_pair_terms, F_j = conj(F_{NJ-1-j})), the midpoint's factor (odd NJ) is real; one biased
// accumulator pair per pair plus one for the midpoint.  8 FP64 instructions per point for even NJ
// (midpoint-merged rows), 7.0 for NJ = 3, 7.4 for NJ = 5, instead of 12.
#ifndef LEAF_SYM_SPLIT
#define LEAF_SYM_SPLIT 0   // 1: the two nodes of a pair in separate accumulators (shorter chains)
#endif
#define LEAF_SYM_NACC(NJ) (LEAF_SYM_SPLIT ? NJ : (NJ + 1) / 2)
// node 0 (A + B) into accumulator a, node 2 (A - B) into b
__device__ __forceinline__ void leaf_sym_pair_split(const dd &er, const dd &ei, const double2 f, const double2 g,
                                                    LeafAcc &a, LeafAcc &b) {
    const double u1 = fma(er.hi, f.x, a.h);
    const double h1 = u1 - a.h;
    a.h = fma(ei.hi, g.x, u1);
    const double h2 = a.h - u1;
    const double cA = fma(er.lo, f.x, fma(er.hi, f.y, fma(er.hi, f.x, -h1)));
    const double cB = fma(ei.lo, g.x, fma(ei.hi, g.y, fma(ei.hi, g.x, -h2)));
    a.l += cA + cB;
    b.h += h1 - h2;
    b.l += cA - cB;
}

template <int NJ>
__device__ __forceinline__ void leaf_rows_sym(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                              int kp0, int kp1, int klane, bool pred, const dd &pr, const dd &pim,
                                              double sigma, LeafAcc (&acc)[LEAF_SYM_NACC(NJ)]) {
    constexpr int NP = NJ / 2;
    for (int kp = kp0; kp < kp1;) {
        const int ke = min(kp1, kp + LEAF_SYM_FOLD);
        #pragma unroll kRowUnroll
        for (; kp < ke; ++kp) {
            const bool kv = !pred || kp > klane;
            const dd er = kv ? pr : dd{0.0, 0.0};
            const dd ei = kv ? pim : dd{0.0, 0.0};
            const double2 *fr = Fr + (long long)kp * NJ;
            const double2 *fi = Fi + (long long)kp * NJ;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                if constexpr (LEAF_SYM_SPLIT)
                    leaf_sym_pair_split(er, ei, __ldg(fr + NJ - 1 - q), __ldg(fi + NJ - 1 - q), acc[q], acc[NJ - 1 - q]);
                else
                    leaf_sym_pair_terms(er, ei, __ldg(fr + NJ - 1 - q), __ldg(fi + NJ - 1 - q), acc[q].h, acc[q].l);
            }
            if constexpr (NJ % 2 == 1) leaf_real_factor_term<false>(er, __ldg(fr + NP), acc[NP].h, acc[NP].l);
        }
#pragma unroll
        for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) leaf_fold(acc[q], sigma);
    }
}

template <int NJ>
__device__ __forceinline__ dd leaf_level_sym(const double2 *Fr, const double2 *Fi, int kb, int kmain, int ks1,
                                             int k, const dd &pr, const dd &pim, double sigma) {
    LeafAcc acc[LEAF_SYM_NACC(NJ)];
#pragma unroll
    for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) acc[q] = LeafAcc{sigma, 0.0};   // biased accumulator
    leaf_rows_sym<NJ>(Fr, Fi, kb, min(kmain, ks1), k, true, pr, pim, sigma, acc);
    leaf_rows_sym<NJ>(Fr, Fi, max(kb, kmain), ks1, k, false, pr, pim, sigma, acc);
    dd s = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) s = dd_add(s, dd_norm(acc[q].h - sigma, acc[q].l));
    return s;
}

// SKIPW: the leaf-only kernel of a split frontier pass — the children the write-only k_pass stores
// (levels with bp <= L-1, rows k' <= d-2) are skipped: for such a level a lane only walks the row
// k' = d-1 (its effective last coordinate becomes max(k, d-2)).
template <bool CPLX, bool SKIPW = false>
__global__ void __launch_bounds__(PASS_THREADS, LEAF_MINB) k_leaf(const DevPlan P, const PassArgs A) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * WPB + wib;
    dd tot = {0.0, 0.0};
    if (task < A.ntasks) {
        const int d = P.d, L = P.L;
        const long long chunk = task / A.nsplit;
        const int split = (int)(task - chunk * A.nsplit);
        const long long g = chunk * 32 + lane;
        const bool valid = g < A.nsrc;
        int b = L, k = d;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (valid) {
            const uint32_t m = SG_SRC(A, src_meta, g);
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = SG_SRC(A, src_re, g);
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = SG_SRC(A, src_im, g);
                pim = dd{vi.x, vi.y};
            }
        }
        const int ks0 = (int)((long long)split * d / A.nsplit);
        const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
        const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
        const int kmax = __reduce_max_sync(0xffffffffu, valid ? k : -1);
        const int bmin = __reduce_min_sync(0xffffffffu, b);
        const int kb0 = max(ks0, kmin + 1), kmain0 = kmax + 1, k0 = k;
        const double pabs = fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0);
        for (int lp = 2; lp <= L + 1 - bmin; ++lp) {
            const bool lv = valid && (lp <= L + 1 - b);
            const dd er = lv ? pr : dd{0.0, 0.0};
            const dd ei = lv ? pim : dd{0.0, 0.0};
            const int n = P.nl[lp];
            // sigma = 1.5 * 2^m with 2^m >= 2 * bound on sum |p| over this lane's children
            const double bound = lv ? pabs * P.SA[(long long)lp * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20) : 0.0;
            const double sigma = grid_sigma(bound);
            const double2 *Fr = P.Fre + P.tab_off[lp];
            const double2 *Fi = CPLX ? P.Fim + P.tab_off[lp] : nullptr;
            int kb = kb0, kmain = kmain0, k = k0;
            if (SKIPW) {
                // stored children of this level belong to the write-only kernel
                if (lv && b + lp - 1 <= L - 1) k = max(k0, d - 2);
                const int kmn = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
                const int kmx = __reduce_max_sync(0xffffffffu, valid ? k : -1);
                kb = max(ks0, kmn + 1);
                kmain = kmx + 1;
            }
            dd s;
            const bool sym = CPLX && ((P.symmask >> lp) & 1);
            if (sym && n == 3) s = leaf_level_sym<3>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 5) s = leaf_level_sym<5>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 2) s = leaf_level_sym<2>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 4) s = leaf_level_sym<4>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else switch (n) {
            case 2: s = leaf_level<CPLX, 2>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            case 3: s = leaf_level<CPLX, 3>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            case 4: s = leaf_level<CPLX, 4>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            case 5: s = leaf_level<CPLX, 5>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            default: s = leaf_level<CPLX, 0>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            }
            if (lv) tot = dd_add(tot, coef_mul(P, s, A.t + 1, b + lp - 1));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) SG_PART(A.partials, blockIdx.x) = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// k_leaf1: the last pass when every source prefix has excess L-1 (t = L-1), so every child has
// level 2 and coefficient coef[L]: the dominant kernel of configs 4-5 (c4: 99.6%, c5: 97.4% of the
// points) when the last two levels are not fused (SG_B200_NOFUSE=1 or plans that cannot fuse).
// One biased accumulator pair per lane, LEAF1_ROWS rows per iteration for ILP.  Oscillatory leaf =
// 12 FP64 instructions (two grid adds + their exact grid parts, remainder + cross-term FMA chain,
// acc_lo), real leaf = 6.
// ---------------------------------------------------------------------------------------------
template <bool CPLX>
__device__ __forceinline__ void leaf1_term(const dd &er, const dd &ei, const double2 f, const double2 fi,
                                           double &ah, double &al) {
    // biased accumulator ah (see leaf_term); the remainder t = P.hi F.hi - h (one rounding) seeds the
    // FMA chain of the cross terms.  Real: 6 FP64 instructions (4 DFMA + 2 DADD); oscillatory: 12.
    if (!CPLX) {
        const double a1 = fma(er.hi, f.x, ah);
        const double h = a1 - ah;
        ah = a1;
        double c = fma(er.lo, f.x, fma(er.hi, f.x, -h));
        c = fma(er.hi, f.y, c);
        al += c;
    } else {
        const double a1 = fma(er.hi, f.x, ah);
        const double h1 = a1 - ah;
        const double a2 = fma(-ei.hi, fi.x, a1);
        const double h2 = a2 - a1;
        ah = a2;
        double c = fma(er.lo, f.x, fma(er.hi, f.x, -h1));
        c = fma(er.hi, f.y, c);
        c = fma(-ei.lo, fi.x, c);
        c = fma(-ei.hi, fi.y, c);
        al += c + fma(-ei.hi, fi.x, -h2);
    }
}

#ifdef SG_TAILPROF
// experiment build only (-DSG_TAILPROF, tools/tail_profile.py): per-warp start / exit times (globaltimer,
// ns), SM id and task count of the persistent fused kernel
#define TAILPROF_MAX 16384
__device__ unsigned long long g_tp_t0[TAILPROF_MAX], g_tp_t1[TAILPROF_MAX];
__device__ unsigned g_tp_sm[TAILPROF_MAX], g_tp_n[TAILPROF_MAX], g_tp_rows[TAILPROF_MAX];
__device__ __forceinline__ unsigned long long tp_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned tp_smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#endif
#ifndef LEAF1_MINB
#define LEAF1_MINB 4
#endif
#ifndef LEAF1_THREADS
#define LEAF1_THREADS PASS_THREADS   // k_leaf1 CTA size
#endif
#ifndef LEAF1_PERJ
#define LEAF1_PERJ 0   // 1 = one accumulator pair per node j of the row (measured slower)
#endif
#ifndef LEAF1_ROWS
#define LEAF1_ROWS 4   // rows k' per loop iteration (A/B: 4 > 2 > 1)
#endif

template <bool CPLX, int NJ, int NA, bool SMEM>
__device__ __forceinline__ void leaf1_row(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi, int kp,
                                          const dd &er, const dd &ei, double (&ah)[NA], double (&al)[NA]) {
    double2 f[NJ], g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        f[j] = SMEM ? Fr[kp * NJ + j] : __ldg(Fr + kp * NJ + j);
        g[j] = CPLX ? (SMEM ? Fi[kp * NJ + j] : __ldg(Fi + kp * NJ + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) leaf1_term<CPLX>(er, ei, f[j], g[j], ah[j % NA], al[j % NA]);
}

// One warp task of the single-level leaf pass: returns this lane's coefficient-free sum.
template <bool CPLX, int NJ, bool SMEM>
__device__ __forceinline__ dd leaf1_task(const DevPlan &P, const PassArgs &A, long long task,
                                         const double2 *Fr, const double2 *Fi) {
    constexpr int NA = LEAF1_PERJ ? NJ : 1;
    const int lane = threadIdx.x & 31;
    const int d = P.d;
    const long long chunk = task / A.nsplit;
    const int split = (int)(task - chunk * A.nsplit);
    const long long g = chunk * 32 + lane;
    const bool valid = g < A.nsrc;
    int k = d;
    dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
    if (valid) {
        k = (int)(SG_SRC(A, src_meta, g) & META_KMASK);
        const double2 v = SG_SRC(A, src_re, g);
        pr = dd{v.x, v.y};
        if (CPLX) {
            const double2 vi = SG_SRC(A, src_im, g);
            pim = dd{vi.x, vi.y};
        }
    }
    const int ks0 = (int)((long long)split * d / A.nsplit);
    const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
    const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
    const int kmax = __reduce_max_sync(0xffffffffu, valid ? k : -1);
    const int kb = max(ks0, kmin + 1);
    const double bound = valid ? (fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0)) *
                                     P.SA[2LL * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20)
                               : 0.0;
    const double sigma = grid_sigma(bound);
    double ah[NA], al[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        ah[a] = sigma;   // biased accumulator
        al[a] = 0.0;
    }
    // boundary rows: lanes whose prefix ends at k >= k' contribute zero
    const int kmid = min(kmax + 1, ks1);
    for (int kp = kb; kp < kmid; ++kp) {
        const bool kv = kp > k;
        const dd er = kv ? pr : dd{0.0, 0.0};
        const dd ei = kv ? pim : dd{0.0, 0.0};
        leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp, er, ei, ah, al);
    }
    // main rows, LEAF1_ROWS per iteration, folded back onto the grid every FOLD rows
    int kp = max(kb, kmid);
    while (kp < ks1) {
        const int ke = min(ks1, kp + FOLD);
        for (; kp + LEAF1_ROWS - 1 < ke; kp += LEAF1_ROWS) {
#pragma unroll
            for (int r = 0; r < LEAF1_ROWS; ++r)
                leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp + r, pr, pim, ah, al);
        }
        for (; kp < ke; ++kp) leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp, pr, pim, ah, al);
#pragma unroll
        for (int a = 0; a < NA; ++a) {
            const double t = (al[a] + sigma) - sigma;
            ah[a] += t;
            al[a] -= t;
        }
    }
    dd s = {0.0, 0.0};
    if (valid) {
#pragma unroll
        for (int a = 0; a < NA; ++a) s = dd_add(s, dd_from_sum(ah[a] - sigma, al[a]));
    }
    return s;
}

// Persistent: gridDim.x = resident CTAs; CTA c's warp w runs tasks (c*WPB + w) + i*gridDim.x*WPB
// (static round robin over tasks sorted heavy-first, so partials stay deterministic).  With SMEM the
// level-2 factor slice (d x NJ entries) is staged once per CTA in shared memory, so the warp-uniform
// row loads are broadcast LDS instead of LDG through the L1 data path.
template <bool CPLX, int NJ, bool SMEM>
__global__ void __launch_bounds__(LEAF1_THREADS, LEAF1_MINB) k_leaf1(const DevPlan P, const PassArgs A) {
    extern __shared__ double2 fsm[];
    const int wib = threadIdx.x >> 5;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = CPLX ? P.Fim + P.tab_off[2] : nullptr;
    if (SMEM) {
        const int n = P.d * NJ;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            if (CPLX) fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = CPLX ? fsm + n : nullptr;
    }
    (void)wib;
    const int lane = threadIdx.x & 31;
    // dynamic scheduling: warps pull tasks (sorted heavy-first) from a global counter; every task
    // writes its own partial, so the fixed-order reduction keeps results bitwise reproducible
#ifdef SG_TAILPROF
    const unsigned long long tp_start = tp_now();
    unsigned tp_tasks = 0;
#endif
    for (;;) {
        unsigned long long task = 0;
        if (lane == 0) task = atomicAdd(A.counter, 1ull);
        task = __shfl_sync(0xffffffffu, task, 0);
        if ((long long)task >= A.ntasks) break;
        dd v = warp_reduce_dd(leaf1_task<CPLX, NJ, SMEM>(P, A, (long long)task, Fr, Fi));
        if (lane == 0) {
            v = dd_mul_d(v, P.coef[P.L]);
            SG_PART(A.partials, task) = make_double2(v.hi, v.lo);
        }
#ifdef SG_TAILPROF
        ++tp_tasks;
#endif
    }
#ifdef SG_TAILPROF
    const int tp_w = (int)(blockIdx.x * (blockDim.x >> 5) + wib);
    if (lane == 0 && tp_w < TAILPROF_MAX) {
        g_tp_t0[tp_w] = tp_start;
        g_tp_t1[tp_w] = tp_now();
        g_tp_sm[tp_w] = tp_smid();
        g_tp_n[tp_w] = tp_tasks;
        g_tp_rows[tp_w] = 0;
    }
#endif
}

// ---------------------------------------------------------------------------------------------
// k_leaf2: fused last two levels.  The depth-(L-1) prefixes are never stored: a warp task is
// (k_mid, 32 stored depth-(L-2) parents of excess L-2 whose last active coordinate is < k_mid);
// each lane forms P' = P * F[2][k_mid][j_mid] in full double-double for every node j_mid, then
// walks the rows k' > k_mid of its level-2 children exactly like k_leaf1.  All lanes share k_mid,
// so every row is warp-uniform (no boundary predication).  Saves the write + read of frontier
// L-1 (config 5: 119 M nodes, 4.3 GB each way).
// ---------------------------------------------------------------------------------------------
struct Leaf2Args {
    const double2 *src_re, *src_im;   // frontier L-2
    long long base;                   // offset of segment (b = L-2, k = 0) in frontier L-2
    const long long *Cmid;            // C_{L-2}(L-2, k): parents of excess L-2 with k_last < k
    const long long *T2;              // task descriptors: first parent, (ka << 32) | kb, (kp0 << 32) | kp1 (plan.h)
    long long ntasks;
    double2 *partials;             // one per task
    unsigned long long *counter;   // dynamic task counter, zeroed per launch
    int prefetch;                  // software-pipelined task fetch (>= 16 tasks per resident warp)
    SG_CHK_FIELDS
};

#ifndef LEAF2_ROWS
#define LEAF2_ROWS 1        // rows per iteration, real kinds (A/B on config 4: 1 > 2)
#endif
#ifndef LEAF2_ROWS_CPLX
#define LEAF2_ROWS_CPLX 4   // rows per iteration, oscillatory (A/B on config 5: 4 = 6 = 8 > 2 > 1)
#endif
// Real kinds: ONE CTA of 24 warps per SM (80 registers), not three CTAs of 8.  With three, the warp
// schedulers' age priority starves the youngest CTA of every SM (tools/tail_profile.py, config 4 at
// N = 1: rows per warp 9925 / 2625 / 810 by CTA age) and its warps, still holding early-claimed tasks
// when the list runs dry, finish alone over the last 8% (N = 1) to 20% (N = 8) of the launch; in one
// CTA the 24 warps share the pipe evenly (rows per warp 4212-4756, warp-busy 0.947 -> 0.994).
#ifndef LEAF2_MINB
#define LEAF2_MINB 1        // CTAs/SM bound, real kinds
#endif
#ifndef LEAF2_REAL_THREADS
#define LEAF2_REAL_THREADS 768   // k_leaf2 CTA size, real kinds
#endif
#ifndef LEAF2_MINB_CPLX
#define LEAF2_MINB_CPLX 2   // CTAs/SM bound, oscillatory (108 regs, 16 warps/SM: 26.14 ms vs 27.52)
#endif

// CJ = index of the midpoint node in the level-2 row (-1: none), fixed per launch by the host;
// SYM: nodes 0 and 2 form a symmetric pair (CJ == 1, NJ == 3, oscillatory), or nodes 0 and 1 do
// (CJ == -1, NJ == 2: the midpoint-merged Clenshaw-Curtis level-2 row {0, 1}).
#ifndef LEAF2_PREFETCH
#define LEAF2_PREFETCH 1   // prefetch the next task's index and descriptor
#endif
#ifndef LEAF2_SPLITR
#define LEAF2_SPLITR 0  // same split for the real kinds' NJ = 3 row with midpoint
#endif
#ifndef LEAF2_SPLIT2
#define LEAF2_SPLIT2 1  // same split for the midpoint-merged NJ = 2 symmetric row (merged c5 -0.6%)
#endif
#ifndef LEAF2_SPLIT
#define LEAF2_SPLIT 1   // second accumulator pair per mid (node 2 + midpoint): shorter chains, c5 -1%
#endif
template <bool CPLX, int NJ, bool SMEM, int CJ, bool SYM = false, bool CZ = false>
__device__ __forceinline__ void leaf2_row_multi(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                                int kp, const dd (&er)[NJ], const dd (&ei)[NJ],
                                                double (&ah)[NJ], double (&al)[NJ], double (&bh)[NJ],
                                                double (&bl)[NJ]) {
    if constexpr (LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) {
        const double2 f2 = SMEM ? Fr[kp * 3 + 2] : __ldg(Fr + kp * 3 + 2);
        const double2 g2 = SMEM ? Fi[kp * 3 + 2] : __ldg(Fi + kp * 3 + 2);
        const double2 f1 = SMEM ? Fr[kp * 3 + 1] : __ldg(Fr + kp * 3 + 1);
#pragma unroll
        for (int jm = 0; jm < 3; ++jm) {
            // node 0 (A + B) into accumulator a, node 2 (A - B) and the midpoint into b
            const double u1 = fma(er[jm].hi, f2.x, ah[jm]);
            const double h1 = u1 - ah[jm];
            ah[jm] = fma(ei[jm].hi, g2.x, u1);
            const double h2 = ah[jm] - u1;
            const double cA = fma(er[jm].lo, f2.x, fma(er[jm].hi, f2.y, fma(er[jm].hi, f2.x, -h1)));
            const double cB = fma(ei[jm].lo, g2.x, fma(ei[jm].hi, g2.y, fma(ei[jm].hi, g2.x, -h2)));
            al[jm] += cA + cB;
            bh[jm] += h1 - h2;
            bl[jm] += cA - cB;
            leaf_real_factor_term<CZ>(er[jm], f1, bh[jm], bl[jm]);
        }
        return;
    }
    if constexpr (SYM && CPLX && NJ == 3 && CJ == 1) {
        const double2 f2 = SMEM ? Fr[kp * 3 + 2] : __ldg(Fr + kp * 3 + 2);
        const double2 g2 = SMEM ? Fi[kp * 3 + 2] : __ldg(Fi + kp * 3 + 2);
        const double2 f1 = SMEM ? Fr[kp * 3 + 1] : __ldg(Fr + kp * 3 + 1);
#pragma unroll
        for (int jm = 0; jm < 3; ++jm) {
            leaf_sym_pair_terms(er[jm], ei[jm], f2, g2, ah[jm], al[jm]);
            leaf_real_factor_term<CZ>(er[jm], f1, ah[jm], al[jm]);
        }
        return;
    }
    if constexpr (SYM && CPLX && NJ == 2 && CJ == -1) {
        const double2 f1 = SMEM ? Fr[kp * 2 + 1] : __ldg(Fr + kp * 2 + 1);
        const double2 g1 = SMEM ? Fi[kp * 2 + 1] : __ldg(Fi + kp * 2 + 1);
#pragma unroll
        for (int jm = 0; jm < 2; ++jm) {
            if constexpr (LEAF2_SPLIT2) {
                // node 0 (A + B) into accumulator a, node 1 (A - B) into b: shorter chains
                const double u1 = fma(er[jm].hi, f1.x, ah[jm]);
                const double h1 = u1 - ah[jm];
                ah[jm] = fma(ei[jm].hi, g1.x, u1);
                const double h2 = ah[jm] - u1;
                const double cA = fma(er[jm].lo, f1.x, fma(er[jm].hi, f1.y, fma(er[jm].hi, f1.x, -h1)));
                const double cB = fma(ei[jm].lo, g1.x, fma(ei[jm].hi, g1.y, fma(ei[jm].hi, g1.x, -h2)));
                al[jm] += cA + cB;
                bh[jm] += h1 - h2;
                bl[jm] += cA - cB;
            } else {
                leaf_sym_pair_terms(er[jm], ei[jm], f1, g1, ah[jm], al[jm]);
            }
        }
        return;
    }
    double2 f[NJ], g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        f[j] = SMEM ? Fr[kp * NJ + j] : __ldg(Fr + kp * NJ + j);
        g[j] = (CPLX && j != CJ) ? (SMEM ? Fi[kp * NJ + j] : __ldg(Fi + kp * NJ + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int jm = 0; jm < NJ; ++jm) {
            if constexpr (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1) {
                // real kinds: node 0 and the midpoint into accumulator a, node 2 into b
                if (j == CJ) leaf_real_factor_term<CZ>(er[jm], f[j], ah[jm], al[jm]);
                else if (j == 0) leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], ah[jm], al[jm]);
                else leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], bh[jm], bl[jm]);
                continue;
            }
            if (j == CJ) leaf_real_factor_term<CZ>(er[jm], f[j], ah[jm], al[jm]);
            else leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], ah[jm], al[jm]);
        }
}

// G (lane groups, small shards): a task's chunk holds 32 / G parents and lane = (parent lane % (32/G),
// k_mid group lane / (32/G)); group g walks the task's k_mids ka + g, ka + g + G, ... < kb (rows
// [max(k_mid + 1, kp0), kp1) each), so a shard with few parents (config 4 on 8 GPUs: 132 on rank 0)
// fills its lanes.  G = 1 is the lane = parent mapping (every k_mid of the task on every lane).
template <bool CPLX, int NJ, bool SMEM, int CJ, bool SYM = false, bool CZ = false, int G = 1>
__global__ void __launch_bounds__(CPLX ? PASS_THREADS : LEAF2_REAL_THREADS, CPLX ? LEAF2_MINB_CPLX : LEAF2_MINB) k_leaf2(const DevPlan P, const Leaf2Args A) {
    extern __shared__ double2 fsm[];
    static_assert(G == 1 || G == 2 || G == 4 || G == 8, "lane groups");
    constexpr int PCH = 32 / G;   // parents per task chunk
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int plane = G == 1 ? lane : lane % PCH, lgrp = G == 1 ? 0 : lane / PCH;
    const int d = P.d;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = CPLX ? P.Fim + P.tab_off[2] : nullptr;
    if (SMEM) {
        const int n = d * NJ;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            if (CPLX) fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = CPLX ? fsm + n : nullptr;
    }
    (void)wib;
#ifdef SG_TAILPROF
    const int tp_w = (int)(blockIdx.x * (blockDim.x >> 5) + wib);
    const unsigned long long tp_start = tp_now();
    unsigned tp_tasks = 0, tp_rows = 0;
#endif
#if LEAF2_PREFETCH
    // software-pipelined task fetch: the next task's index and descriptor are requested before the
    // current task's rows run, so their latency (atomic + L2 loads) is hidden behind the FP64 work
    auto fetch = [&]() -> long long {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(A.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, u, 0);
    };
    long long task = fetch();
    long long first = 0, kk = 0, rr = 0;
    if (task < A.ntasks) {
        first = A.T2[3 * task];
        kk = A.T2[3 * task + 1];
        rr = A.T2[3 * task + 2];
    }
    for (;;) {
        if (task >= A.ntasks) break;
        // prefetch only with many tasks per warp: a reserved next task cannot be stolen by an idle
        // warp, which lengthens the tail when each warp runs only a few tasks (config 3)
        long long next = 0, nfirst = 0, nkk = 0, nrr = 0;
        if (A.prefetch) {
            next = fetch();
            if (next < A.ntasks) {
                nfirst = A.T2[3 * next];
                nkk = A.T2[3 * next + 1];
                nrr = A.T2[3 * next + 2];
            }
        }
#else
    for (;;) {
        unsigned long long utask = 0;
        if (lane == 0) utask = atomicAdd(A.counter, 1ull);
        utask = __shfl_sync(0xffffffffu, utask, 0);
        const long long task = (long long)utask;
        if (task >= A.ntasks) break;
        // task = (chunk of 32 parents starting at `first`, k_mid range [ka, kb), rows [kp0, kp1)),
        // plan.h T2
        const long long first = A.T2[3 * task], kk = A.T2[3 * task + 1], rr = A.T2[3 * task + 2];
#endif
        const int ka = task_hi32(kk), kb = task_lo32(kk);
        const int kp0 = task_hi32(rr), kp1 = task_lo32(rr);
#ifdef SG_TAILPROF
        ++tp_tasks;
#endif
        const long long i = first + plane;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (i < A.Cmid[kb - 1]) {   // Cmid is nondecreasing: valid for the last k_mid
            const double2 v = SG_SRC(A, src_re, A.base + i);
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = SG_SRC(A, src_im, A.base + i);
                pim = dd{vi.x, vi.y};
            }
        }
        dd lane_sum = {0.0, 0.0};
        for (int km = ka + lgrp; km < kb; km += G) {
            const bool valid = i < A.Cmid[km];
            const dd prv = valid ? pr : dd{0.0, 0.0};
            const dd pimv = valid ? pim : dd{0.0, 0.0};
            const double sa = P.SA[2LL * (d + 1) + km + 1] * (1.0 + 0x1p-20);
            // all NJ mid prefixes of the lane at once: NJ independent accumulator chains that share
            // every row load (ILP x NJ, shared-memory loads / leaf / NJ)
            dd er[NJ], ei[NJ];
            double sg[NJ], ah[NJ], al[NJ], bh[NJ], bl[NJ];
            if constexpr (CPLX && SYM && NJ == 3 && CJ == 1) {
                // mids 0 and 2 are conjugate (F_0 = conj(F_2)): P F_2 and P conj(F_2) share their
                // four products; mid 1 (the midpoint) is real
                const double2 f = Fr[km * 3 + 2], g = Fi[km * 3 + 2], w1 = Fr[km * 3 + 1];
                cdd c2, c0;
                cdd_mul_conj_pair(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}}, c2, c0);
                er[0] = c0.re;
                ei[0] = c0.im;
                er[2] = c2.re;
                ei[2] = c2.im;
                er[1] = CZ ? dd_mul_d(prv, w1.x) : dd_mul(prv, dd{w1.x, w1.y});
                ei[1] = CZ ? dd_mul_d(pimv, w1.x) : dd_mul(pimv, dd{w1.x, w1.y});
            } else if constexpr (CPLX && SYM && NJ == 2 && CJ == -1) {
                const double2 f = Fr[km * 2 + 1], g = Fi[km * 2 + 1];
                cdd c1, c0;
                cdd_mul_conj_pair(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}}, c1, c0);
                er[0] = c0.re;
                ei[0] = c0.im;
                er[1] = c1.re;
                ei[1] = c1.im;
            } else {
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {
                    const double2 f = Fr[km * NJ + jm];
                    if (CPLX) {
                        const double2 g = Fi[km * NJ + jm];
                        cdd c = cdd_mul_fast(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}});
                        er[jm] = c.re;
                        ei[jm] = c.im;
                    } else {
                        er[jm] = dd_mul(prv, dd{f.x, f.y});
                        ei[jm] = dd{0.0, 0.0};
                    }
                }
            }
#pragma unroll
            for (int jm = 0; jm < NJ; ++jm) {
                const double bound = (fabs(er[jm].hi) + (CPLX ? fabs(ei[jm].hi) : 0.0)) * sa;
                sg[jm] = grid_sigma_frexp(bound);   // (grid_sigma measured 2% slower here: c4 1.78 vs 1.74 ms)
                ah[jm] = sg[jm];   // biased accumulator
                al[jm] = 0.0;
                bh[jm] = sg[jm];
                bl[jm] = 0.0;
            }
            SG_CHK(km, d - 1, 6);                               // mid row (its factors, Cmid, SA)
            SG_CHK(kp1 - 1, d, 5);                              // last leaf row of the table slice
            int kp = max(km + 1, kp0);
#ifdef SG_TAILPROF
            tp_rows += (unsigned)max(0, kp1 - kp);
#endif
            while (kp < kp1) {
                const int ke = min(kp1, kp + FOLD);
                constexpr int RW = CPLX ? LEAF2_ROWS_CPLX : LEAF2_ROWS;
                for (; kp + RW - 1 < ke; kp += RW) {
#pragma unroll
                    for (int r = 0; r < RW; ++r)
                        leaf2_row_multi<CPLX, NJ, SMEM, CJ, SYM, CZ>(Fr, Fi, kp + r, er, ei, ah, al, bh, bl);
                }
                for (; kp < ke; ++kp) leaf2_row_multi<CPLX, NJ, SMEM, CJ, SYM, CZ>(Fr, Fi, kp, er, ei, ah, al, bh, bl);
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {
                    if ((LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) ||
                        (LEAF2_SPLIT2 && SYM && CPLX && NJ == 2 && CJ == -1) ||
                        (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1))
                        al[jm] += bl[jm], bl[jm] = 0.0;
                    const double t = (al[jm] + sg[jm]) - sg[jm];
                    ah[jm] += t;
                    al[jm] -= t;
                }
            }
            // lane value = sum_jm (ah - sigma) + al: exact grid parts via TwoSum, low parts in FP64
            if ((LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) ||
                (LEAF2_SPLIT2 && SYM && CPLX && NJ == 2 && CJ == -1) ||
                (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1)) {
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {   // same grid, |sum| < 2^m: exact
                    ah[jm] += bh[jm] - sg[jm];
                    al[jm] += bl[jm];
                }
            }
            double hs = ah[0] - sg[0], ls = al[0];
#pragma unroll
            for (int jm = 1; jm < NJ; ++jm) {
                double e;
                two_sum(hs, ah[jm] - sg[jm], hs, e);
                ls += al[jm] + e;
            }
            lane_sum = dd_add_fast(lane_sum, dd_norm(hs, ls));
        }
        dd v = warp_reduce_dd_fast(lane_sum);
        if (lane == 0) {
            v = dd_mul_d(v, P.coef[P.L]);
            SG_PART(A.partials, task) = make_double2(v.hi, v.lo);
        }
#if LEAF2_PREFETCH
        if (!A.prefetch) {
            next = fetch();
            if (next < A.ntasks) {
                nfirst = A.T2[3 * next];
                nkk = A.T2[3 * next + 1];
                nrr = A.T2[3 * next + 2];
            }
        }
        task = next;
        first = nfirst;
        kk = nkk;
        rr = nrr;
#endif
    }
#ifdef SG_TAILPROF
    if (lane == 0 && tp_w < TAILPROF_MAX) {
        g_tp_t0[tp_w] = tp_start;
        g_tp_t1[tp_w] = tp_now();
        g_tp_sm[tp_w] = tp_smid();
        g_tp_n[tp_w] = tp_tasks;
        g_tp_rows[tp_w] = tp_rows;
    }
#endif
}


// ---------------------------------------------------------------------------------------------
// k_leaf2_pairs: the fused last two levels for a level-2 row that is one conjugate pair (the
// midpoint-merged Clenshaw-Curtis row {0, 1}, oscillatory kind).  Each lane carries PPL parents
// (first + 32 p + lane), i.e. 2 PPL mid prefixes, so every row load and loop step feeds 16 PPL FP64
// instructions instead of 32 and the warp has twice the independent accumulator chains.  Same
// arithmetic per point as k_leaf2's split symmetric pair (node 0 into a, node 1 into b).
// ---------------------------------------------------------------------------------------------
#ifndef SYM3_LAST_FOLD
#define SYM3_LAST_FOLD 0   // 1: fold after the last row chunk too (A/B)
#endif
#ifndef SYM3_THREADS
#define SYM3_THREADS 256   // k_leaf2_sym3 CTA size (A/B knob)
#endif
#ifndef SYM3_MINB
#define SYM3_MINB 1        // k_leaf2_sym3 CTAs per SM bound (A/B knob)
#endif
#ifndef LEAF2_PAIRS_MINB
#define LEAF2_PAIRS_MINB 1   // 1 CTA (8 warps) per SM, up to 255 registers: ILP over occupancy
#endif
template <int PPL, bool SMEM>
__global__ void __launch_bounds__(PASS_THREADS, LEAF2_PAIRS_MINB) k_leaf2_pairs(const DevPlan P, const Leaf2Args A) {
    constexpr int NM = 2 * PPL;   // mid prefixes per lane
    extern __shared__ double2 fsm[];
    const int lane = threadIdx.x & 31;
    const int d = P.d;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = P.Fim + P.tab_off[2];
    if (SMEM) {
        const int n = d * 2;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = fsm + n;
    }
    auto fetch = [&]() -> long long {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(A.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, u, 0);
    };
    long long task = fetch();
    long long first = 0, kk = 0, rr = 0;
    if (task < A.ntasks) {
        first = A.T2[3 * task];
        kk = A.T2[3 * task + 1];
        rr = A.T2[3 * task + 2];
    }
    while (task < A.ntasks) {
        long long next = 0, nfirst = 0, nkk = 0, nrr = 0;
        if (A.prefetch) {
            next = fetch();
            if (next < A.ntasks) {
                nfirst = A.T2[3 * next];
                nkk = A.T2[3 * next + 1];
                nrr = A.T2[3 * next + 2];
            }
        }
        const int ka = task_hi32(kk), kb = task_lo32(kk);
        const int kp0 = task_hi32(rr), kp1 = task_lo32(rr);
        long long ip[PPL];
        dd pr[PPL], pim[PPL];
        const long long cend = A.Cmid[kb - 1];
#pragma unroll
        for (int q = 0; q < PPL; ++q) {
            ip[q] = first + 32LL * q + lane;
            pr[q] = dd{0.0, 0.0};
            pim[q] = dd{0.0, 0.0};
            if (ip[q] < cend) {
                const double2 v = SG_SRC(A, src_re, A.base + ip[q]), vi = SG_SRC(A, src_im, A.base + ip[q]);
                pr[q] = dd{v.x, v.y};
                pim[q] = dd{vi.x, vi.y};
            }
        }
        dd lane_sum = {0.0, 0.0};
        for (int km = ka; km < kb; ++km) {
            const long long cm = A.Cmid[km];
            const double sa = P.SA[2LL * (d + 1) + km + 1] * (1.0 + 0x1p-20);
            const double2 fm = Fr[km * 2 + 1], gm = Fi[km * 2 + 1];
            dd er[NM], ei[NM];
            double sg[NM], ah[NM], al[NM], bh[NM], bl[NM];
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                const bool valid = ip[q] < cm;
                cdd c1, c0;
                cdd_mul_conj_pair(cdd{valid ? pr[q] : dd{0.0, 0.0}, valid ? pim[q] : dd{0.0, 0.0}},
                                  cdd{dd{fm.x, fm.y}, dd{gm.x, gm.y}}, c1, c0);
                er[2 * q] = c0.re;
                ei[2 * q] = c0.im;
                er[2 * q + 1] = c1.re;
                ei[2 * q + 1] = c1.im;
            }
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                const double bound = (fabs(er[m].hi) + fabs(ei[m].hi)) * sa;
                sg[m] = grid_sigma(bound);
                ah[m] = bh[m] = sg[m];   // biased accumulators (node 0 -> a, node 1 -> b)
                al[m] = bl[m] = 0.0;
            }
            SG_CHK(km, d - 1, 6);
            SG_CHK(kp1 - 1, d, 5);
            int kp = max(km + 1, kp0);
            while (kp < kp1) {
                const int ke = min(kp1, kp + FOLD);
            for (; kp < ke; ++kp) {
                const double2 f1 = SMEM ? Fr[kp * 2 + 1] : __ldg(Fr + kp * 2 + 1);
                const double2 g1 = SMEM ? Fi[kp * 2 + 1] : __ldg(Fi + kp * 2 + 1);
#pragma unroll
                for (int m = 0; m < NM; ++m) {
                    const double u1 = fma(er[m].hi, f1.x, ah[m]);
                    const double h1 = u1 - ah[m];
                    ah[m] = fma(ei[m].hi, g1.x, u1);
                    const double h2 = ah[m] - u1;
                    const double cA = fma(er[m].lo, f1.x, fma(er[m].hi, f1.y, fma(er[m].hi, f1.x, -h1)));
                    const double cB = fma(ei[m].lo, g1.x, fma(ei[m].hi, g1.y, fma(ei[m].hi, g1.x, -h2)));
                    al[m] += cA + cB;
                    bh[m] += h1 - h2;
                    bl[m] += cA - cB;
                }
            }
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                al[m] += bl[m];
                bl[m] = 0.0;
                const double t = (al[m] + sg[m]) - sg[m];
                ah[m] += t;
                al[m] -= t;
            }
        }
        double hs = (ah[0] + (bh[0] - sg[0])) - sg[0], ls = al[0] + bl[0];
#pragma unroll
        for (int m = 1; m < NM; ++m) {
            double e;
            two_sum(hs, (ah[m] + (bh[m] - sg[m])) - sg[m], hs, e);
            ls += al[m] + bl[m] + e;
        }
        lane_sum = dd_add_fast(lane_sum, dd_norm(hs, ls));
    }
    dd v = warp_reduce_dd_fast(lane_sum);
    if (lane == 0) {
        v = dd_mul_d(v, P.coef[P.L]);
        SG_PART(A.partials, task) = make_double2(v.hi, v.lo);
    }
    if (!A.prefetch) {
        next = fetch();
        if (next < A.ntasks) {
            nfirst = A.T2[3 * next];
            nkk = A.T2[3 * next + 1];
            nrr = A.T2[3 * next + 2];
        }
    }
    task = next;
    first = nfirst;
    kk = nkk;
    rr = nrr;
}
}

// ---------------------------------------------------------------------------------------------
// k_leaf2_sym3: the fused last two levels for a level-2 row {0, 1/2, 1} (symmetric pair + real
// midpoint, oscillatory: the Clenshaw-Curtis / trapezoidal combination-form row of configs 2, 5)
// with PPL parents per lane (3 PPL mid prefixes), 1 CTA per SM: k_leaf2's per-point arithmetic
// (split symmetric pair: node 0 into a, node 2 and the midpoint into b) with more independent
// accumulator chains per warp.
// ---------------------------------------------------------------------------------------------
// One k_leaf2_sym3 task for one lane.  MODE 0: a fused task (the lane's PPL parents times the three
// level-2 factors of each k_mid in [ka, kb), each prefix walking the symmetric level-2 rows).
// MODE 1 / 2: a source task: NM stored sources of frontier L-2 with last coordinate -ka - 1 (kb of
// them in the chunk) are the prefixes themselves; MODE 1 walks their symmetric level-2 rows, MODE 2
// their level-3 rows (SYM3_N3 nodes, general complex leaf terms).  One instantiation per mode, so the
// fused tasks' loop nest is compiled as if the source tasks did not exist.
template <int PPL, bool SMEM, bool CZ, int MODE>
__device__ __forceinline__ dd sym3_task(const DevPlan &P, const Leaf2Args &A, const double2 *Fr,
                                        const double2 *Fi, int lane, long long first, int ka, int kb,
                                        int kp0, int kp1) {
    constexpr bool SRCT = MODE != 0;
    constexpr int NM = 3 * PPL;
    const int d = P.d;
    const int km0 = SRCT ? -ka - 1 : ka, km1 = SRCT ? km0 + 1 : kb;
    long long ip[PPL];
    dd pr[PPL], pim[PPL];
    const long long cend = SRCT ? 0 : A.Cmid[kb - 1];
#pragma unroll
    for (int q = 0; q < PPL; ++q) {
        ip[q] = first + 32LL * q + lane;
        pr[q] = dd{0.0, 0.0};
        pim[q] = dd{0.0, 0.0};
        if (ip[q] < cend) {
            const double2 v = SG_SRC(A, src_re, A.base + ip[q]), vi = SG_SRC(A, src_im, A.base + ip[q]);
            pr[q] = dd{v.x, v.y};
            pim[q] = dd{vi.x, vi.y};
        }
    }
    dd lane_sum = {0.0, 0.0};
    for (int km = km0; km < km1; ++km) {
        const double sa = P.SA[(MODE >= 2 ? 3LL : 2LL) * (d + 1) + km + 1] * (1.0 + 0x1p-20);
        dd er[NM], ei[NM];
        double sg[NM], ah[NM], al[NM], bh[NM], bl[NM];
        if constexpr (SRCT) {
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                const int is = 32 * m + lane;
                er[m] = ei[m] = dd{0.0, 0.0};
                if (is < kb) {
                    const double2 v = SG_SRC(A, src_re, first + is), vi = SG_SRC(A, src_im, first + is);
                    er[m] = dd{v.x, v.y};
                    ei[m] = dd{vi.x, vi.y};
                }
            }
        } else {
            const long long cm = A.Cmid[km];
            const double2 fm = Fr[km * 3 + 2], gm = Fi[km * 3 + 2], wm = Fr[km * 3 + 1];
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                const bool valid = ip[q] < cm;
                const dd vr = valid ? pr[q] : dd{0.0, 0.0}, vi = valid ? pim[q] : dd{0.0, 0.0};
                cdd c2, c0;
                cdd_mul_conj_pair(cdd{vr, vi}, cdd{dd{fm.x, fm.y}, dd{gm.x, gm.y}}, c2, c0);
                er[3 * q] = c0.re;
                ei[3 * q] = c0.im;
                er[3 * q + 2] = c2.re;
                ei[3 * q + 2] = c2.im;
                er[3 * q + 1] = CZ ? dd_mul_d(vr, wm.x) : dd_mul(vr, dd{wm.x, wm.y});
                ei[3 * q + 1] = CZ ? dd_mul_d(vi, wm.x) : dd_mul(vi, dd{wm.x, wm.y});
            }
        }
#pragma unroll
        for (int m = 0; m < NM; ++m) {
            const double bound = (fabs(er[m].hi) + fabs(ei[m].hi)) * sa;
            sg[m] = grid_sigma(bound);
            ah[m] = bh[m] = sg[m];   // biased accumulators (node 0 -> a, node 1 -> b)
            al[m] = bl[m] = 0.0;
        }
        SG_CHK(km, d, 6);
        SG_CHK(kp1 - 1, d, 5);
        int kp = max(km + 1, kp0);
        while (kp < kp1) {
            const int ke = min(kp1, kp + FOLD);
            if constexpr (MODE == 2) {
                const double2 *F3r = P.Fre + P.tab_off[3], *F3i = P.Fim + P.tab_off[3];
                for (; kp < ke; ++kp) {
#pragma unroll
                    for (int j = 0; j < SYM3_N3; ++j) {
                        const double2 f = __ldg(F3r + kp * SYM3_N3 + j), g = __ldg(F3i + kp * SYM3_N3 + j);
#pragma unroll
                        for (int m = 0; m < NM; ++m) {
                            LeafAcc a = {ah[m], al[m]};
                            leaf_term<true>(er[m], ei[m], f, g, a);
                            ah[m] = a.h;
                            al[m] = a.l;
                        }
                    }
                }
            }
            if constexpr (MODE >= 3) {
                // level-3 row {0, x1, 1/2, x3, 1} with x = 0 and 1 an exactly conjugate pair and an
                // exactly real midpoint (MODE 3: nodes x1, x3 general terms; MODE 4: x1 = 1 - x3
                // exactly, a second conjugate pair): 46 resp. 38 FP64 per 5 points instead of 60
                const double2 *F3r = P.Fre + P.tab_off[3], *F3i = P.Fim + P.tab_off[3];
                for (; kp < ke; ++kp) {
                    const double2 f4 = __ldg(F3r + kp * 5 + 4), g4 = __ldg(F3i + kp * 5 + 4);
                    const double2 f3 = __ldg(F3r + kp * 5 + 3), g3 = __ldg(F3i + kp * 5 + 3);
                    const double2 f2 = __ldg(F3r + kp * 5 + 2);
                    double2 f1 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
                    if constexpr (MODE == 3) {
                        f1 = __ldg(F3r + kp * 5 + 1);
                        g1 = __ldg(F3i + kp * 5 + 1);
                    }
#pragma unroll
                    for (int m = 0; m < NM; ++m) {
                        leaf_sym_pair_terms(er[m], ei[m], f4, g4, ah[m], al[m]);   // nodes 0 and 4
                        if constexpr (MODE == 4) {
                            leaf_sym_pair_terms(er[m], ei[m], f3, g3, bh[m], bl[m]);   // nodes 1 and 3
                        } else {
                            LeafAcc b = {bh[m], bl[m]};
                            leaf_term<true>(er[m], ei[m], f1, g1, b);
                            leaf_term<true>(er[m], ei[m], f3, g3, b);
                            bh[m] = b.h;
                            bl[m] = b.l;
                        }
                        leaf_real_factor_term<false>(er[m], f2, ah[m], al[m]);   // the midpoint
                    }
                }
            }
            if constexpr (MODE < 2) {
            for (; kp < ke; ++kp) {
                const double2 f1 = SMEM ? Fr[kp * 3 + 2] : __ldg(Fr + kp * 3 + 2);
                const double2 g1 = SMEM ? Fi[kp * 3 + 2] : __ldg(Fi + kp * 3 + 2);
                const double2 w1 = SMEM ? Fr[kp * 3 + 1] : __ldg(Fr + kp * 3 + 1);
#pragma unroll
                for (int m = 0; m < NM; ++m) {
                    const double u1 = fma(er[m].hi, f1.x, ah[m]);
                    const double h1 = u1 - ah[m];
                    ah[m] = fma(ei[m].hi, g1.x, u1);
                    const double h2 = ah[m] - u1;
                    const double cA = fma(er[m].lo, f1.x, fma(er[m].hi, f1.y, fma(er[m].hi, f1.x, -h1)));
                    const double cB = fma(ei[m].lo, g1.x, fma(ei[m].hi, g1.y, fma(ei[m].hi, g1.x, -h2)));
                    al[m] += cA + cB;
                    bh[m] += h1 - h2;
                    bl[m] += cA - cB;
                    leaf_real_factor_term<CZ>(er[m], w1, bh[m], bl[m]);   // the midpoint node
                }
            }
            }
            // fold the low accumulators onto the grid between row chunks; after the last chunk the
            // lane epilogue below takes them as they are
            if (SYM3_LAST_FOLD || kp < kp1) {
#pragma unroll
                for (int m = 0; m < NM; ++m) {
                    al[m] += bl[m];
                    bl[m] = 0.0;
                    const double t = (al[m] + sg[m]) - sg[m];
                    ah[m] += t;
                    al[m] -= t;
                }
            }
        }
        double hs = (ah[0] + (bh[0] - sg[0])) - sg[0], ls = al[0] + bl[0];
#pragma unroll
        for (int m = 1; m < NM; ++m) {
            double e;
            two_sum(hs, (ah[m] + (bh[m] - sg[m])) - sg[m], hs, e);
            ls += al[m] + bl[m] + e;
        }
        lane_sum = dd_add_fast(lane_sum, dd_norm(hs, ls));
    }
    return lane_sum;
}

// SRC = false: the fused tasks (pass L-1); SRC = true: the source tasks (pass L-2, its own task list
// T2 and partial slots), a separate kernel so the fused loop nest's code is not disturbed (measured:
// sharing one kernel slowed the fused tasks by 1.6-4% through code layout alone).
template <int PPL, bool SMEM, bool CZ, bool SRC, int L3S = 0>
__global__ void __launch_bounds__(SYM3_THREADS, SYM3_MINB) k_leaf2_sym3(const DevPlan P, const Leaf2Args A) {
    constexpr int NM = 3 * PPL;   // mid prefixes per lane
    extern __shared__ double2 fsm[];
    const int lane = threadIdx.x & 31;
    const int d = P.d;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = P.Fim + P.tab_off[2];
    if (SMEM) {
        const int n = d * 3;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = fsm + n;
    }
#ifdef SG_TAILPROF
    const unsigned long long tp_start = tp_now();
    unsigned tp_tasks = 0;
#endif
    auto fetch = [&]() -> long long {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(A.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, u, 0);
    };
    long long task = fetch();
    long long first = 0, kk = 0, rr = 0;
    if (task < A.ntasks) {
        first = A.T2[3 * task];
        kk = A.T2[3 * task + 1];
        rr = A.T2[3 * task + 2];
    }
    while (task < A.ntasks) {
        long long next = 0, nfirst = 0, nkk = 0, nrr = 0;
        if (A.prefetch) {
            next = fetch();
            if (next < A.ntasks) {
                nfirst = A.T2[3 * next];
                nkk = A.T2[3 * next + 1];
                nrr = A.T2[3 * next + 2];
            }
        }
        const int ka = task_hi32(kk), kb = task_lo32(kk);
        const int kp0 = task_hi32(rr), kp1 = task_lo32(rr);
        // source tasks: ka = -(k + 1), kb = chunk size | SRC_L3 | SRC_CPREV
        dd lane_sum;
        if constexpr (SRC) {
            const int cnt = kb & 0xffff;
            lane_sum = (kb & SRC_L3) ? sym3_task<PPL, SMEM, CZ, 2 + L3S>(P, A, Fr, Fi, lane, first, ka, cnt, kp0, kp1)
                                     : sym3_task<PPL, SMEM, CZ, 1>(P, A, Fr, Fi, lane, first, ka, cnt, kp0, kp1);
        } else {
            lane_sum = sym3_task<PPL, SMEM, CZ, 0>(P, A, Fr, Fi, lane, first, ka, kb, kp0, kp1);
        }
        dd v = warp_reduce_dd_fast(lane_sum);
        if (lane == 0) {
            v = dd_mul_d(v, P.coef[SRC && (kb & SRC_CPREV) ? P.L - 1 : P.L]);
            SG_PART(A.partials, task) = make_double2(v.hi, v.lo);
        }
        if (!A.prefetch) {
            next = fetch();
            if (next < A.ntasks) {
                nfirst = A.T2[3 * next];
                nkk = A.T2[3 * next + 1];
                nrr = A.T2[3 * next + 2];
            }
        }
#ifdef SG_TAILPROF
        ++tp_tasks;
#endif
        task = next;
        first = nfirst;
        kk = nkk;
        rr = nrr;
    }
#ifdef SG_TAILPROF
    const int tp_w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    if (!SRC && lane == 0 && tp_w < TAILPROF_MAX) {
        g_tp_t0[tp_w] = tp_start;
        g_tp_t1[tp_w] = tp_now();
        g_tp_sm[tp_w] = tp_smid();
        g_tp_n[tp_w] = tp_tasks;
        g_tp_rows[tp_w] = 0;
    }
#endif
}

// ---------------------------------------------------------------------------------------------
// k_front: the write-only frontier kernel of a split pass (HBM-bound by design).  A CTA takes a chunk
// of up to FRONT_THREADS consecutive sources of one frontier-t segment (b, k) — one source per thread,
// read once, coalesced — and writes all their stored children: for every child level l' with
// b' = b + l' - 1 <= L-1, every row k' in (k, d-2] and node j', the chunk's children are consecutive
// records at TB[b][b'][k'] + n_l' C_t(b, k) + j' N_t(b, k) + i (plan.h layout), so each (k', j')
// store is one contiguous block of up to FRONT_THREADS records (re, im, meta).  The factor and the TB
// offset of a row are CTA-uniform (broadcast loads).  Each stored child's own Smolyak term, the real
// part of its product, is accumulated (times C(t+1, b')).  The other children of the pass are
// evaluated by k_leaf<CPLX, true> concurrently.  Chunks are assigned dynamically (sorted
// heavy-first, pulled from an atomic counter): one partial per chunk, fixed reduction order.
// ---------------------------------------------------------------------------------------------
struct FrontChunk {
    long long src0;   // first source record (frontier t index)
    int i0, cnt;      // index of the first source inside its segment, sources in the chunk
    int b, k;         // the segment
    long long C, N;   // C_t(b, k), N_t(b, k)
};

#ifndef FRONT_THREADS
#define FRONT_THREADS 256
#endif
template <bool CPLX>
__device__ __forceinline__ dd front_product(const dd &pr, const dd &pim, const double2 f, const double2 fi,
                                            dd &cim) {
    if (!CPLX) {
        cim = dd{0.0, 0.0};
        return dd_mul(pr, dd{f.x, f.y});
    }
    double p1, e1, p2, e2, p3, e3, p4, e4;
    dd_mul_pe(pr, dd{f.x, f.y}, p1, e1);
    dd_mul_pe(pim, dd{fi.x, fi.y}, p2, e2);
    dd_mul_pe(pr, dd{fi.x, fi.y}, p3, e3);
    dd_mul_pe(pim, dd{f.x, f.y}, p4, e4);
    cim = dd_combine_pe(p3, e3, p4, e4);
    return dd_combine_pe(p1, e1, -p2, -e2);
}

#ifndef FRONT_SPT
#define FRONT_SPT 4   // sources per thread: a (row, node) store block is FRONT_THREADS * FRONT_SPT records
#endif
template <bool CPLX>
__global__ void __launch_bounds__(FRONT_THREADS) k_front(const DevPlan P, const PassArgs A, const FrontChunk *chunks,
                                                         long long nchunks) {
    const int d = P.d, L = P.L;
    __shared__ long long cnext;
    for (;;) {
        if (threadIdx.x == 0) cnext = (long long)atomicAdd(A.counter, 1ull);
        __syncthreads();
        const long long c = cnext;
        __syncthreads();
        if (c >= nchunks) break;
        dd tot = {0.0, 0.0};
        const FrontChunk C = chunks[c];
        // sources s = threadIdx.x + FRONT_THREADS u of the chunk (u < FRONT_SPT), loaded once
        dd pr[FRONT_SPT], pim[FRONT_SPT];
#pragma unroll
        for (int u = 0; u < FRONT_SPT; ++u) {
            const int sidx = threadIdx.x + FRONT_THREADS * u;
            pr[u] = pim[u] = dd{0.0, 0.0};
            if (sidx < C.cnt) {
                const double2 v = SG_SRC(A, src_re, C.src0 + sidx);
                pr[u] = dd{v.x, v.y};
                if (CPLX) {
                    const double2 vi = SG_SRC(A, src_im, C.src0 + sidx);
                    pim[u] = dd{vi.x, vi.y};
                }
            }
        }
        for (int lp = 2; lp <= L - C.b; ++lp) {   // stored child levels: b' = b + lp - 1 <= L - 1
            const int bp = C.b + lp - 1, n = P.nl[lp];
            const double2 *__restrict__ Fr = P.Fre + P.tab_off[lp];
            const double2 *__restrict__ Fi = CPLX ? P.Fim + P.tab_off[lp] : nullptr;
            const long long *__restrict__ tbrow = A.TB + ((long long)C.b * L + bp) * d;
            const long long base = (long long)n * C.C + C.i0 + threadIdx.x;
            double ah = 0.0, al = 0.0;
            long long tbn = __ldg(tbrow + C.k + 1);
            for (int kp = C.k + 1; kp <= d - 2; ++kp) {
                const long long tb = tbn + base;
                if (kp + 1 <= d - 2) tbn = __ldg(tbrow + kp + 1);
                const uint32_t meta = ((uint32_t)bp << SG_META_KBITS) | (uint32_t)kp;
                for (int j = 0; j < n; ++j) {
                    const double2 f = __ldg(Fr + (long long)kp * n + j);
                    const double2 fi = CPLX ? __ldg(Fi + (long long)kp * n + j) : make_double2(0.0, 0.0);
#pragma unroll
                    for (int u = 0; u < FRONT_SPT; ++u) {
                        if ((int)threadIdx.x + FRONT_THREADS * u < C.cnt) {
                            const long long o = tb + (long long)j * C.N + FRONT_THREADS * u;
                            dd cim;
                            const dd cre = front_product<CPLX>(pr[u], pim[u], f, fi, cim);
                            SG_DST(A, dst_re, o) = make_double2(cre.hi, cre.lo);
                            if (CPLX) SG_DST(A, dst_im, o) = make_double2(cim.hi, cim.lo);
                            SG_DST(A, dst_meta, o) = meta;
                            acc_add(ah, al, cre.hi, cre.lo);
                        }
                    }
                }
            }
            tot = dd_add(tot, coef_mul(P, dd_norm(ah, al), A.t + 1, bp));
        }
        dd s = block_reduce_dd<FRONT_THREADS / 32>(tot);
        if (threadIdx.x == 0) SG_PART(A.partials, c) = make_double2(s.hi, s.lo);
        __syncthreads();   // block_reduce's shared scratch is reused by the next chunk
    }
}
