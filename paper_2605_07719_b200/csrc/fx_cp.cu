// fx_cp.cu -- context-parallel decode (config C5): the global budgeted top-k
// of topk_blocks (block_index.cpp:55-83) and the LSE merge of merge_into
// (attention.cpp:89-104), split over cpu-segment shards.
//
// Why the two exchanges reproduce the single-device selection bit-exactly:
// a block in the global top-k of a head is beaten by fewer than k blocks
// overall, hence by fewer than k blocks of its own shard, so it is in that
// shard's local top-k (candidates).  If shard r holds >= k blocks, its k-th
// local score t_r is <= the global k-th score, so T = max_r t_r is a lower
// bound: only entries with score >= T can be selected, and the shard that
// attains T contributes k of them.  The global rank of an entry under the
// reference's strict total order (score desc, id asc) is the sum over shards
// of the entries that precede it -- one binary search per shard list, since
// every list is sorted by that same order.
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
int cp_sort_n(int64_t nblk16);
double approx_eps_scale(const fx_layout& L);
namespace {

constexpr int kT = 256;

struct MetaLevels {
    const void* p[4];  // blk 16 / 32 / 64 / 128
};

// Local candidates of one head: the ids of the shard's selected blocks, exact
// reference scores as keys, bitonic-sorted in smem by (key desc, id asc).
template <int DT>
__global__ void __launch_bounds__(kT) k_cp_candidates(
    const MetaLevels meta_levels, const float* __restrict__ q,
    const int32_t* __restrict__ blk_arr, const int32_t* __restrict__ kblocks,
    const uint32_t* __restrict__ sel_bits, int sel_words, int Hkv, int G, int D, int64_t l_cpu,
    int64_t cpu_offset, int64_t cap, int sort_n, uint64_t* __restrict__ keys_out,
    uint32_t* __restrict__ ids_out, int32_t* __restrict__ count_out, uint64_t* __restrict__ kth_out) {
    using T = typename Elem<DT>::T;
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(dsm);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + sort_n);
    __shared__ int s_wpos[kT + 1];
    __shared__ double s_q[256];
    const int64_t head = blockIdx.x;
    const int64_t H = (int64_t)Hkv * G;
    const int b = (int)(head / H), h = (int)(head % H);
    const int bg = b * Hkv + h / G;
    const int t = threadIdx.x;
    const int blk = blk_arr[bg];
    const int64_t k = kblocks[head];
    const int64_t nblk = blk > 0 ? cdiv_dev(l_cpu, blk) : 0;
    const int W = (int)cdiv_dev(nblk, 32);
    const uint32_t* bits = sel_bits + head * sel_words;
    // 1. compact the selected ids (thread-contiguous word ranges, block scan)
    const int per = (W + kT - 1) / kT;
    const int w0 = min(W, t * per), w1 = min(W, w0 + per);
    int c = 0;
    for (int w = w0; w < w1; ++w) c += __popc(bits[w]);
    s_wpos[t + 1] = c;
    __syncthreads();
    if (t == 0) {
        s_wpos[0] = 0;
        for (int i = 1; i <= kT; ++i) s_wpos[i] += s_wpos[i - 1];
    }
    __syncthreads();
    const int n = s_wpos[kT];  // = min(k, nblk) by the selection
    int pos = s_wpos[t];
    for (int w = w0; w < w1; ++w) {
        uint32_t u = bits[w];
        while (u) {
            const int l = __ffs(u) - 1;
            u &= u - 1;
            si[pos++] = (uint32_t)(w * 32 + l);
        }
    }
    __syncthreads();
    // 2. exact scores (block_index.cpp:41-53) -> keys; pad to sort_n
    const T* mbase = blk > 0 ? static_cast<const T*>(meta_levels.p[blk == 16 ? 0 : blk == 32 ? 1 : blk == 64 ? 2 : 3]) +
                                   (int64_t)bg * nblk * 2 * D
                             : nullptr;
    const float* qh = q + head * D;
    for (int d = t; d < D; d += kT) s_q[d] = (double)qh[d];
    __syncthreads();
    const int64_t off_blk = blk > 0 ? cpu_offset / blk : 0;
    for (int i = t; i < sort_n; i += kT) {
        if (i < n) {
            const uint32_t id = si[i];
            const T* row = mbase + (int64_t)id * 2 * D;
            double sc;
            if constexpr (DT == FX_BF16) {
                sc = D == 128 ? exact_score_row<128>(s_q, row)
                   : D == 64  ? exact_score_row<64>(s_q, row)
                              : exact_score(qh, row, row + D, D);
            } else {
                sc = exact_score(qh, row, row + D, D);
            }
            sk[i] = f64_key(sc);
            si[i] = (uint32_t)(id + off_blk);  // global block id
        } else {
            sk[i] = 0;
            si[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    // 3. bitonic sort, (key desc, id asc) first, over the smallest power of two
    //    holding the n real entries (the padding sorts last and stays in place)
    int len = 32;
    while (len < n) len <<= 1;
    len = len < sort_n ? len : sort_n;
    for (int kk = 2; kk <= len; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = t; i < len; i += kT) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & kk) == 0;
                    const uint64_t a = sk[i], e = sk[p];
                    const uint32_t ia = si[i], ie = si[p];
                    if (up ? first_of(e, ie, a, ia) : first_of(a, ia, e, ie)) {
                        sk[i] = e;
                        sk[p] = a;
                        si[i] = ie;
                        si[p] = ia;
                    }
                }
            }
            __syncthreads();
        }
    // 4. emit
    for (int64_t i = t; i < cap; i += kT) {
        keys_out[head * cap + i] = i < n ? sk[i] : 0ull;
        ids_out[head * cap + i] = i < n ? si[i] : 0xffffffffu;
    }
    if (t == 0) {
        count_out[head] = n;
        kth_out[head] = (k > 0 && n >= k) ? sk[k - 1] : 0ull;
    }
}

__global__ void k_cp_threshold(int R, int64_t n, int64_t cap, const uint64_t* __restrict__ keys,
                               const uint64_t* __restrict__ kth_all, uint64_t* __restrict__ thresh,
                               int32_t* __restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t T = 0;
    for (int r = 0; r < R; ++r) {
        const uint64_t v = kth_all[(int64_t)r * n + i];
        T = v > T ? v : T;
    }
    // sorted descending, zero-filled: entries with key >= max(T, 1)
    const uint64_t lim = T > 0 ? T : 1ull;
    const uint64_t* kh = keys + i * cap;
    int64_t lo = 0, hi = cap;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (kh[mid] >= lim) lo = mid + 1;
        else hi = mid;
    }
    thresh[i] = T;
    keep[i] = (int32_t)lo;
}

// Global rank of each own entry; bits for rank < k.
__global__ void __launch_bounds__(kT) k_cp_select(
    int R, int self, int64_t n, int64_t m, const uint64_t* __restrict__ gkeys,
    const uint32_t* __restrict__ gids, const uint64_t* __restrict__ thresh,
    const int32_t* __restrict__ kblocks, const int32_t* __restrict__ blk_arr, int G,
    int64_t cpu_offset, uint32_t* __restrict__ sel_out, int sel_words) {
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x;
    uint32_t* bits = sel_out + head * sel_words;
    for (int w = t; w < sel_words; w += kT) bits[w] = 0u;
    __syncthreads();
    const int blk = blk_arr[head / G];
    const int64_t k = kblocks[head];
    if (blk <= 0 || k <= 0) return;
    const uint64_t lim = thresh[head] > 0 ? thresh[head] : (uint64_t)1;
    const int64_t off_blk = cpu_offset / blk;
    const uint64_t* own_k = gkeys + ((int64_t)self * n + head) * m;
    const uint32_t* own_i = gids + ((int64_t)self * n + head) * m;
    for (int64_t j = t; j < m; j += kT) {
        const uint64_t ke = own_k[j];
        if (ke < lim) continue;  // below the bound (or an empty slot)
        const uint32_t ie = own_i[j];
        int64_t rank = j;         // own entries before j precede it
        for (int r = 0; r < R && rank < k; ++r) {
            if (r == self) continue;
            const uint64_t* kr = gkeys + ((int64_t)r * n + head) * m;
            const uint32_t* ir = gids + ((int64_t)r * n + head) * m;
            int64_t lo = 0, hi = m;  // entries of list r that come first
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (kr[mid] >= lim && first_of(kr[mid], ir[mid], ke, ie)) lo = mid + 1;
                else hi = mid;
            }
            rank += lo;
        }
        if (rank < k) {
            const int64_t local = (int64_t)ie - off_blk;
            atomicOr(&bits[local >> 5], 1u << (local & 31));
        }
    }
}

__global__ void k_cp_combine(int R, int64_t n, int D, const float* __restrict__ op,
                             const float* __restrict__ lp, float* __restrict__ o,
                             float* __restrict__ lse) {
    const int64_t i = blockIdx.x;
    float M = -INFINITY;
    for (int r = 0; r < R; ++r) M = fmaxf(M, lp[(int64_t)r * n + i]);
    float den = 0.f;
    for (int r = 0; r < R; ++r) {
        const float l = lp[(int64_t)r * n + i];
        den += (l == -INFINITY) ? 0.f : expf(l - M);
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float num = 0.f;
        for (int r = 0; r < R; ++r) {
            const float l = lp[(int64_t)r * n + i];
            if (l != -INFINITY) num += expf(l - M) * op[((int64_t)r * n + i) * D + d];
        }
        o[i * D + d] = den > 0.f ? num / den : 0.f;
    }
    if (threadIdx.x == 0 && lse) lse[i] = den > 0.f ? M + logf(den) : -INFINITY;
}

// ---------------------------------------------------------------------------
// exchanges over peer memory
// ---------------------------------------------------------------------------
struct PeerSet {
    fx_cp_peer p[FX_CP_MAX_RANKS];
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* a) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

// thread 0 waits until every rank's flag[slot] reached `stamp`; the acquire
// loads make the peers' preceding writes visible to the whole CTA after the
// barrier
__device__ void wait_peers(const PeerSet& ps, int R, int slot, uint64_t stamp) {
    if (threadIdx.x == 0)
        for (int r = 0; r < R; ++r)
            while (ld_acquire_sys(ps.p[r].flags + slot) < stamp) __nanosleep(64);
    __syncthreads();
}

__global__ void k_cp_signal(uint64_t* flags, int slot, uint64_t stamp) {
    __threadfence_system();  // everything this stream wrote before is visible first
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags + slot), "l"(stamp) : "memory");
}

// threshold (max over ranks of the local k-th key) + global rank of each own
// entry by binary search in every peer's sorted list -- the fx_cp_threshold /
// fx_cp_select pair reading the peers' lists where they are
__global__ void __launch_bounds__(kT) k_cp_select_peer(
    const __grid_constant__ PeerSet ps, int R, int self, int64_t n, uint64_t stamp,
    const int32_t* __restrict__ kblocks, const int32_t* __restrict__ blk_arr, int G,
    int64_t cpu_offset, uint32_t* __restrict__ sel_out, int sel_words) {
    pdl_wait();
    pdl_trigger();
    wait_peers(ps, R, 0, stamp);
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x;
    uint32_t* bits = sel_out + head * sel_words;
    for (int w = t; w < sel_words; w += kT) bits[w] = 0u;
    __syncthreads();
    const int blk = blk_arr[head / G];
    const int64_t k = kblocks[head];
    if (blk <= 0 || k <= 0) return;
    uint64_t T = 0;
    for (int r = 0; r < R; ++r) {
        const uint64_t v = ps.p[r].kth[head];
        T = v > T ? v : T;
    }
    const uint64_t lim = T > 0 ? T : 1ull;
    const int64_t off_blk = cpu_offset / blk;
    const fx_cp_peer& me = ps.p[self];
    const uint64_t* own_k = me.keys + head * me.cap;
    const uint32_t* own_i = me.ids + head * me.cap;
    for (int64_t j = t; j < me.cap; j += kT) {
        const uint64_t ke = own_k[j];
        if (ke < lim) break;  // sorted descending: the rest is below the bound
        const uint32_t ie = own_i[j];
        int64_t rank = j;
        for (int r = 0; r < R && rank < k; ++r) {
            if (r == self) continue;
            const uint64_t* kr = ps.p[r].keys + head * ps.p[r].cap;
            const uint32_t* ir = ps.p[r].ids + head * ps.p[r].cap;
            int64_t lo = 0, hi = ps.p[r].cap;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (kr[mid] >= lim && first_of(kr[mid], ir[mid], ke, ie)) lo = mid + 1;
                else hi = mid;
            }
            rank += lo;
        }
        if (rank < k) {
            const int64_t local = (int64_t)ie - off_blk;
            atomicOr(&bits[local >> 5], 1u << (local & 31));
        }
    }
}

// merge_into over the ranks' (o, lse) partials, read from their memory
__global__ void k_cp_combine_peer(const __grid_constant__ PeerSet ps, int R, int64_t n, int D,
                                  uint64_t stamp, float* __restrict__ o, float* __restrict__ lse) {
    pdl_wait();
    pdl_trigger();
    wait_peers(ps, R, 3, stamp);
    const int64_t i = blockIdx.x;
    float M = -INFINITY;
    for (int r = 0; r < R; ++r) M = fmaxf(M, ps.p[r].lse[i]);
    float den = 0.f;
    for (int r = 0; r < R; ++r) {
        const float l = ps.p[r].lse[i];
        den += (l == -INFINITY) ? 0.f : expf(l - M);
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float num = 0.f;
        for (int r = 0; r < R; ++r) {
            const float l = ps.p[r].lse[i];
            if (l != -INFINITY) num += expf(l - M) * ps.p[r].o[i * D + d];
        }
        o[i * D + d] = den > 0.f ? num / den : 0.f;
    }
    if (threadIdx.x == 0 && lse) lse[i] = den > 0.f ? M + logf(den) : -INFINITY;
}

// ---------------------------------------------------------------------------
// the bracket selection distributed over the ranks
// ---------------------------------------------------------------------------
constexpr int kDBins = 2048;

struct DistArgs {
    int R, self, Hkv, G, D;
    int64_t l_cpu, l_total, cpu_offset, astride;
    double eps_scale;
    const float* approx;
    const float* q;
    const float* absmax;
    MetaLevels meta;
    const int32_t* blk;
    const int32_t* kblocks;
    uint32_t* sel;
    int sel_words, sort_n;
    double* stats;     // own tables
    int32_t* hist;
    uint64_t* keys;
    uint32_t* ids;
    int32_t* defc;
    int64_t cap;
    uint64_t stamp;
};

struct HeadInfo {
    int blk;
    int64_t nblk_local, nblk_total, k;
};
__device__ __forceinline__ HeadInfo head_info(const DistArgs& a, int64_t head) {
    HeadInfo h;
    h.blk = a.blk[head / a.G];
    h.k = a.kblocks[head];
    h.nblk_local = h.blk > 0 ? cdiv_dev(a.l_cpu, h.blk) : 0;
    h.nblk_total = h.blk > 0 ? cdiv_dev(a.l_total, h.blk) : 0;
    return h;
}

// phase 0: min, max, finiteness of the local approximate scores; error bound
__global__ void __launch_bounds__(kT) k_cpd_stats(const DistArgs a) {
    __shared__ float rmx[kT / 32], rmn[kT / 32];
    __shared__ double s_eps;
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const HeadInfo hi = head_info(a, head);
    const float* sc = a.approx + head * a.astride;
    float mx = -INFINITY, mn = INFINITY;
    bool fin = true;
    for (int64_t i = t; i < hi.nblk_local; i += kT) {
        const float x = sc[i];
        if (isfinite(x)) {
            mx = fmaxf(mx, x);
            mn = fminf(mn, x);
        } else {
            fin = false;
        }
    }
    if (warp == 0) {  // eps = c * sum_d |q_d| absmax_d (fx_topk.cu)
        const int64_t bg = head / a.G;
        double e = 0.0;
        for (int d = lane; d < a.D; d += 32)
            e += fabs((double)a.q[head * a.D + d]) * (double)a.absmax[bg * a.D + d];
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) s_eps = e * a.eps_scale * 1.01 + 1e-30;
    }
    mx = warp_max(mx);
    mn = -warp_max(-mn);
    if (lane == 0) {
        rmx[warp] = mx;
        rmn[warp] = mn;
    }
    const bool allfin = __syncthreads_and(fin);
    if (t == 0) {
        for (int w = 0; w < kT / 32; ++w) {
            mx = fmaxf(mx, rmx[w]);
            mn = fminf(mn, rmn[w]);
        }
        double* st = a.stats + head * 4;
        st[0] = mn;
        st[1] = mx;
        st[2] = s_eps;
        st[3] = (allfin && isfinite(s_eps)) ? 0.0 : 1.0;
    }
}

// global range / bound / sanity of a head over all ranks
struct Global {
    float gmn, gmx;
    double eps;
    bool sane;
};
__device__ Global global_of(const PeerSet& ps, int R, int64_t head) {
    Global g{INFINITY, -INFINITY, 0.0, true};
    for (int r = 0; r < R; ++r) {
        const double* st = ps.p[r].stats + head * 4;
        g.gmn = fminf(g.gmn, (float)st[0]);
        g.gmx = fmaxf(g.gmx, (float)st[1]);
        g.eps = fmax(g.eps, st[2]);
        g.sane = g.sane && st[3] == 0.0;
    }
    return g;
}

// phase 1: local histogram over the global range (the single-device bin map)
__global__ void __launch_bounds__(kT) k_cpd_hist(const __grid_constant__ PeerSet ps, const DistArgs a) {
    pdl_wait();
    pdl_trigger();
    wait_peers(ps, a.R, 0, a.stamp);
    __shared__ int hist[kDBins];
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x;
    const HeadInfo hi = head_info(a, head);
    const Global g = global_of(ps, a.R, head);
    for (int i = t; i < kDBins; i += kT) hist[i] = 0;
    __syncthreads();
    if (hi.blk > 0 && g.sane && g.gmx > g.gmn) {
        const float scale = (float)kDBins / (g.gmx - g.gmn);
        const float* sc = a.approx + head * a.astride;
        for (int64_t i = t; i < hi.nblk_local; i += kT) {
            const float f = (sc[i] - g.gmn) * scale;
            atomicAdd(&hist[f >= (float)(kDBins - 1) ? kDBins - 1 : (f <= 0.f ? 0 : (int)f)], 1);
        }
    }
    __syncthreads();
    for (int i = t; i < kDBins; i += kT) a.hist[head * kDBins + i] = hist[i];
}

// phase 2: bracket from the summed histogram; definite bits; exact, sorted band
// Bitonic sort of n entries (score desc, id asc) in the "flip" form: every
// stage sorts ascending and its first step pairs i with the mirror i ^ (kk - 1),
// so a pair always has its larger index on the later side and the virtual
// entries past n (+inf) never move -- no padding to a power of two.  Shared or
// global memory, one CTA.
__device__ void sort_band(uint64_t* k, uint32_t* id, int64_t n) {
    int64_t len = 1;
    while (len < n) len <<= 1;
    for (int64_t kk = 2; kk <= len; kk <<= 1)
        for (int64_t j = kk >> 1; j > 0; j >>= 1) {
            const int64_t m = j == (kk >> 1) ? kk - 1 : j;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                if (i & j) continue;
                const int64_t p2 = i ^ m;
                if (p2 >= n) continue;
                const uint64_t x1 = k[i], x2 = k[p2];
                const uint32_t i1 = id[i], i2 = id[p2];
                if (first_of(x2, i2, x1, i1)) {
                    k[i] = x2;
                    k[p2] = x1;
                    id[i] = i2;
                    id[p2] = i1;
                }
            }
            __syncthreads();
        }
}

template <int DT>
__global__ void __launch_bounds__(kT) k_cpd_band(const __grid_constant__ PeerSet ps, const DistArgs a) {
    pdl_wait();
    pdl_trigger();
    wait_peers(ps, a.R, 1, a.stamp);
    using T = typename Elem<DT>::T;
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* s_k = reinterpret_cast<uint64_t*>(dsm);  // the band when it fits (a.sort_n entries)
    uint32_t* s_i = reinterpret_cast<uint32_t*>(s_k + a.sort_n);
    uint64_t* sk = s_k;
    uint32_t* si = s_i;
    __shared__ int hist[kDBins];
    __shared__ int s_cnt[2][kT / 32];
    __shared__ int s_bin;
    __shared__ double s_q[256];
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const HeadInfo hi = head_info(a, head);
    uint32_t* bits = a.sel + head * a.sel_words;
    const int W = (int)cdiv_dev(hi.nblk_local, 32);
    for (int j = t; j < a.sel_words; j += kT) bits[j] = 0u;
    int64_t ndef = 0, nband = 0;
    const bool all = hi.blk > 0 && hi.k >= hi.nblk_total;  // clamped: every block
    const bool none = hi.blk <= 0 || hi.k <= 0;
    __syncthreads();
    if (all) {
        for (int j = t; j < W; j += kT) {
            const int64_t rem = hi.nblk_local - (int64_t)j * 32;
            bits[j] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        }
        ndef = hi.nblk_local;
    } else if (!none) {
        const Global g = global_of(ps, a.R, head);
        double e_lo = -INFINITY, e_hi = INFINITY;  // insane: everything is band
        if (g.sane && !(g.gmx > g.gmn)) {
            e_lo = e_hi = (double)g.gmx;
        } else if (g.sane) {
            for (int i = t; i < kDBins; i += kT) {
                int c = 0;
                for (int r = 0; r < a.R; ++r) c += ps.p[r].hist[head * kDBins + i];
                hist[i] = c;
            }
            __syncthreads();
            constexpr int PB = kDBins / kT;
            int c = 0;
#pragma unroll
            for (int i = 0; i < PB; ++i) c += hist[t * PB + i];
            int x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            if (lane == 0) s_cnt[0][warp] = x;
            __syncthreads();
            int S = x;
            for (int w = warp + 1; w < kT / 32; ++w) S += s_cnt[0][w];
            if (S >= hi.k && S - c < hi.k) {
                int above = S - c;
                for (int i = PB - 1; i >= 0; --i) {
                    above += hist[t * PB + i];
                    if (above >= hi.k) {
                        s_bin = t * PB + i;
                        break;
                    }
                }
            }
            __syncthreads();
            const double wdt = ((double)g.gmx - (double)g.gmn) / kDBins;
            e_lo = (double)g.gmn + (s_bin - 1) * wdt;
            e_hi = (double)g.gmn + (s_bin + 2) * wdt;
        }
        const double up = e_hi + 2.0 * g.eps, lo = e_lo - 2.0 * g.eps;
        const float* sc = a.approx + head * a.astride;
        // definite-in bits and the band ids (compacted in block order)
        int wdef = 0, wband = 0;
        for (int j = warp; j < W; j += kT / 32) {
            const int64_t i = (int64_t)j * 32 + lane;
            const bool in = i < hi.nblk_local;
            const double x = in ? (double)sc[i] : 0.0;
            const uint32_t bd = __ballot_sync(0xffffffffu, in && x > up);
            const uint32_t bc = __ballot_sync(0xffffffffu, in && !(x > up) && x >= lo);
            if (lane == 0) bits[j] = bd;
            wdef += __popc(bd);
            wband += __popc(bc);
        }
        if (lane == 0) {
            s_cnt[0][warp] = wdef;
            s_cnt[1][warp] = wband;
        }
        __syncthreads();
        int64_t base = 0;
        for (int w = 0; w < kT / 32; ++w) {
            ndef += s_cnt[0][w];
            nband += s_cnt[1][w];
            if (w < warp) base += s_cnt[1][w];
        }
        // a band larger than the shared stage (degenerate data: ties, NaN)
        // is built and sorted in place in the own table row (cap >= nblk)
        const bool big = nband > a.sort_n;
        if (big) {
            sk = a.keys + head * a.cap;
            si = a.ids + head * a.cap;
        }
        for (int j = warp; j < W; j += kT / 32) {
            const int64_t i = (int64_t)j * 32 + lane;
            const bool in = i < hi.nblk_local;
            const double x = in ? (double)sc[i] : 0.0;
            const bool cand = in && !(x > up) && x >= lo;
            const uint32_t bc = __ballot_sync(0xffffffffu, cand);
            if (cand) si[base + __popc(bc & ((1u << lane) - 1u))] = (uint32_t)i;
            base += __popc(bc);
        }
        for (int d = t; d < a.D; d += kT) s_q[d] = (double)a.q[head * a.D + d];
        __syncthreads();
        const int64_t bgi = head / a.G;
        const T* mbase = static_cast<const T*>(a.meta.p[hi.blk == 16 ? 0 : hi.blk == 32 ? 1 : hi.blk == 64 ? 2 : 3]) +
                         bgi * hi.nblk_local * 2 * a.D;
        const int64_t off_blk = a.cpu_offset / hi.blk;
        for (int64_t i = t; i < nband; i += kT) {
            const uint32_t id = si[i];
            const T* row = mbase + (int64_t)id * 2 * a.D;
            double v;
            if constexpr (DT == FX_BF16) {
                v = a.D == 128 ? exact_score_row<128>(s_q, row)
                  : a.D == 64  ? exact_score_row<64>(s_q, row)
                               : exact_score(a.q + head * a.D, row, row + a.D, a.D);
            } else {
                v = exact_score(a.q + head * a.D, row, row + a.D, a.D);
            }
            sk[i] = f64_key(v);
            si[i] = (uint32_t)(id + off_blk);
        }
        __syncthreads();
        sort_band(sk, si, nband);
    }
    __syncthreads();
    if (sk == s_k)
        for (int64_t i = t; i < nband; i += kT) {
            a.keys[head * a.cap + i] = sk[i];
            a.ids[head * a.cap + i] = si[i];
        }
    if (t == 0) {
        a.defc[head * 2] = (int32_t)ndef;
        a.defc[head * 2 + 1] = (int32_t)nband;
    }
}

// phase 3: global ranks of the own band entries among all ranks' bands.  The
// peers' bands (sorted, usually tens of entries) are staged in shared memory
// with one coalesced pass each; a band too large for the stage is searched in
// place.
constexpr int kRankStage = 3840;  // entries (12 B each; static smem under 48 KB)
__global__ void __launch_bounds__(kT) k_cpd_rank(const __grid_constant__ PeerSet ps, const DistArgs a) {
    pdl_wait();
    pdl_trigger();
    wait_peers(ps, a.R, 2, a.stamp);
    __shared__ uint64_t s_k[kRankStage];
    __shared__ uint32_t s_i[kRankStage];
    __shared__ int s_off[FX_CP_MAX_RANKS + 1];
    __shared__ int s_len[FX_CP_MAX_RANKS];
    const int64_t head = blockIdx.x;
    const int t = threadIdx.x;
    const HeadInfo hi = head_info(a, head);
    if (hi.blk <= 0 || hi.k <= 0 || hi.k >= hi.nblk_total) return;
    if (t == 0) {
        int off = 0;
        for (int r = 0; r < a.R; ++r) {
            const int n = ps.p[r].defc[head * 2 + 1];
            s_len[r] = n;
            s_off[r] = off;
            off += (r != a.self && off + n <= kRankStage) ? n : 0;  // staged, or searched in place
        }
        s_off[a.R] = off;
    }
    __syncthreads();
    int64_t need = hi.k;
    for (int r = 0; r < a.R; ++r) need -= ps.p[r].defc[head * 2];
    for (int r = 0; r < a.R; ++r) {
        const int n = s_off[r + 1] - s_off[r];
        const uint64_t* kr = ps.p[r].keys + head * ps.p[r].cap;
        const uint32_t* ir = ps.p[r].ids + head * ps.p[r].cap;
        for (int j = t; j < n; j += kT) {
            s_k[s_off[r] + j] = kr[j];
            s_i[s_off[r] + j] = ir[j];
        }
    }
    __syncthreads();
    uint32_t* bits = a.sel + head * a.sel_words;
    const int64_t off_blk = a.cpu_offset / hi.blk;
    const fx_cp_peer& me = ps.p[a.self];
    const uint64_t* own_k = me.keys + head * me.cap;
    const uint32_t* own_i = me.ids + head * me.cap;
    const int own_n = s_len[a.self];
    for (int64_t j = t; j < own_n; j += kT) {
        const uint64_t ke = own_k[j];
        const uint32_t ie = own_i[j];
        int64_t rank = j;
        for (int r = 0; r < a.R && rank < need; ++r) {
            if (r == a.self) continue;
            const int n = s_len[r];
            const bool staged = s_off[r + 1] - s_off[r] == n;
            const uint64_t* kr = staged ? s_k + s_off[r] : ps.p[r].keys + head * ps.p[r].cap;
            const uint32_t* ir = staged ? s_i + s_off[r] : ps.p[r].ids + head * ps.p[r].cap;
            int lo = 0, hi2 = n;
            while (lo < hi2) {
                const int mid = (lo + hi2) >> 1;
                if (first_of(kr[mid], ir[mid], ke, ie)) lo = mid + 1;
                else hi2 = mid;
            }
            rank += lo;
        }
        if (rank < need) {
            const int64_t local = (int64_t)ie - off_blk;
            atomicOr(&bits[local >> 5], 1u << (local & 31));
        }
    }
}

}  // namespace

void launch_cp_dist_phase(const fx_layout& L, int phase, int R, int self, const fx_cp_peer* peers,
                          uint64_t stamp, const float* approx, int64_t astride, const float* q,
                          const float* absmax, const void* const meta[4], const int32_t* blk,
                          const int32_t* kblocks, int64_t l_total, int64_t cpu_offset, uint32_t* sel,
                          int sel_words, cudaStream_t s) {
    FX_REQUIRE(R >= 1 && R <= FX_CP_MAX_RANKS && self >= 0 && self < R, FX_ERR_INVALID,
               "bad-shape: rank / rank count");
    FX_REQUIRE(L.head_dim <= 256 && L.group_size <= 8, FX_ERR_INVALID,
               "bad-shape: head_dim must be <= 256 and group_size <= 8");
    PeerSet ps{};
    for (int r = 0; r < R; ++r) ps.p[r] = peers[r];
    const fx_cp_peer& me = peers[self];
    // a band never outgrows the tables: cap covers every local block at size 16
    FX_REQUIRE(me.cap >= cdiv(L.l_cpu, 16) && me.stats && me.hist && me.defc && me.keys && me.ids,
               FX_ERR_INVALID, "bad-shape: own exchange tables missing or cap below the shard's 16-blocks");
    DistArgs a{};
    a.R = R;
    a.self = self;
    a.Hkv = L.kv_heads;
    a.G = L.group_size;
    a.D = L.head_dim;
    a.l_cpu = L.l_cpu;
    a.l_total = l_total;
    a.cpu_offset = cpu_offset;
    a.astride = astride;
    a.eps_scale = approx_eps_scale(L);
    a.approx = approx;
    a.q = q;
    a.absmax = absmax;
    for (int i = 0; i < 4; ++i) a.meta.p[i] = meta[i];
    a.blk = blk;
    a.kblocks = kblocks;
    a.sel = sel;
    a.sel_words = sel_words;
    a.cap = me.cap;
    a.sort_n = (int)std::min<int64_t>(cp_sort_n(std::max<int64_t>(1, me.cap)), 4096);
    a.stats = const_cast<double*>(me.stats);
    a.hist = const_cast<int32_t*>(me.hist);
    a.keys = const_cast<uint64_t*>(me.keys);
    a.ids = const_cast<uint32_t*>(me.ids);
    a.defc = const_cast<int32_t*>(me.defc);
    a.stamp = stamp;
    const int64_t n = (int64_t)L.batch * L.kv_heads * L.group_size;
    if (n <= 0) return;
    if (phase == 0) {
        k_cpd_stats<<<(unsigned)n, kT, 0, s>>>(a);
    } else if (phase == 1) {
        launch_pdl(k_cpd_hist, (unsigned)n, kT, 0, s, ps, a);
    } else if (phase == 2) {
        const size_t smem = (size_t)a.sort_n * 12;  // larger bands sort in the own table row
        if (L.dtype == FX_BF16) {
            FX_CUDA(cudaFuncSetAttribute(k_cpd_band<FX_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            launch_pdl(k_cpd_band<FX_BF16>, (unsigned)n, kT, smem, s, ps, a);
        } else {
            FX_CUDA(cudaFuncSetAttribute(k_cpd_band<FX_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            launch_pdl(k_cpd_band<FX_F32>, (unsigned)n, kT, smem, s, ps, a);
        }
    } else {
        launch_pdl(k_cpd_rank, (unsigned)n, kT, 0, s, ps, a);
    }
    FX_CUDA(cudaGetLastError());
}

void launch_cp_signal(uint64_t* flags, int slot, uint64_t stamp, cudaStream_t s) {
    k_cp_signal<<<1, 1, 0, s>>>(flags, slot, stamp);
    FX_CUDA(cudaGetLastError());
}

void launch_cp_select_peer(const fx_layout& L, int R, int self, const fx_cp_peer* peers, uint64_t stamp,
                           const int32_t* kblocks, const int32_t* blk, int64_t cpu_offset,
                           uint32_t* sel_out, int sel_words, cudaStream_t s) {
    FX_REQUIRE(R >= 1 && R <= FX_CP_MAX_RANKS && self >= 0 && self < R, FX_ERR_INVALID,
               "bad-shape: rank / rank count");
    PeerSet ps{};
    for (int r = 0; r < R; ++r) ps.p[r] = peers[r];
    const int64_t n = (int64_t)L.batch * L.kv_heads * L.group_size;
    if (n <= 0) return;
    launch_pdl(k_cp_select_peer, (unsigned)n, kT, 0, s, ps, R, self, n, stamp, kblocks, blk,
               L.group_size, cpu_offset, sel_out, sel_words);
    FX_CUDA(cudaGetLastError());
}

void launch_cp_combine_peer(int R, int64_t n, int dim, const fx_cp_peer* peers, uint64_t stamp, float* o,
                            float* lse, cudaStream_t s) {
    FX_REQUIRE(R >= 1 && R <= FX_CP_MAX_RANKS, FX_ERR_INVALID, "bad-shape: rank count");
    PeerSet ps{};
    for (int r = 0; r < R; ++r) ps.p[r] = peers[r];
    if (n <= 0) return;
    launch_pdl(k_cp_combine_peer, (unsigned)n, 128, 0, s, ps, R, n, dim, stamp, o, lse);
    FX_CUDA(cudaGetLastError());
}

int cp_sort_n(int64_t nblk16) {
    int64_t s = 1;
    while (s < nblk16) s <<= 1;
    return (int)std::max<int64_t>(s, 32);
}

void launch_cp_candidates(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, const uint32_t* sel_bits,
                          int sel_words, int64_t cpu_offset, int64_t cap, uint64_t* keys,
                          uint32_t* ids, int32_t* count, uint64_t* kth, cudaStream_t s) {
    const int64_t heads = (int64_t)L.batch * L.kv_heads * L.group_size;
    FX_REQUIRE(L.head_dim <= 256, FX_ERR_INVALID, "bad-shape: head_dim must be <= 256");
    const int sort_n = cp_sort_n(std::max<int64_t>(1, level_blocks(L.l_cpu, 16)));
    const size_t smem = (size_t)sort_n * 12;
    FX_REQUIRE(smem <= 200 * 1024, FX_ERR_INVALID,
               "bad-shape: context-parallel shard too long (more than 16384 blocks of 16, i.e. 262144 cpu rows per rank; use more ranks)");
    const MetaLevels ml{{meta[0], meta[1], meta[2], meta[3]}};
    if (L.dtype == FX_BF16) {
        auto kern = k_cp_candidates<FX_BF16>;
        FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)heads, kT, smem, s>>>(
            ml, q, blk, kblocks, sel_bits,
            sel_words, L.kv_heads, L.group_size, L.head_dim, L.l_cpu, cpu_offset, cap, sort_n,
            keys, ids, count, kth);
    } else {
        auto kern = k_cp_candidates<FX_F32>;
        FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)heads, kT, smem, s>>>(
            ml, q, blk, kblocks, sel_bits, sel_words,
            L.kv_heads, L.group_size, L.head_dim, L.l_cpu, cpu_offset, cap, sort_n, keys, ids,
            count, kth);
    }
    FX_CUDA(cudaGetLastError());
}

void launch_cp_threshold(int R, int64_t n, int64_t cap, const uint64_t* keys,
                         const uint64_t* kth_all, uint64_t* thresh, int32_t* keep, cudaStream_t s) {
    if (n <= 0) return;
    k_cp_threshold<<<(unsigned)cdiv(n, 128), 128, 0, s>>>(R, n, cap, keys, kth_all, thresh, keep);
    FX_CUDA(cudaGetLastError());
}

void launch_cp_select(const fx_layout& L, int R, int self, int64_t m, const uint64_t* gkeys,
                      const uint32_t* gids, const uint64_t* thresh, const int32_t* kblocks,
                      const int32_t* blk, int64_t cpu_offset, uint32_t* sel_out, int sel_words,
                      cudaStream_t s) {
    const int64_t n = (int64_t)L.batch * L.kv_heads * L.group_size;
    if (n <= 0) return;
    k_cp_select<<<(unsigned)n, kT, 0, s>>>(R, self, n, m, gkeys, gids, thresh, kblocks, blk,
                                           L.group_size, cpu_offset, sel_out, sel_words);
    FX_CUDA(cudaGetLastError());
}

void launch_cp_combine(int R, int64_t n, int dim, const float* o_parts, const float* lse_parts,
                       float* o, float* lse, cudaStream_t s) {
    if (n <= 0) return;
    k_cp_combine<<<(unsigned)n, 128, 0, s>>>(R, n, dim, o_parts, lse_parts, o, lse);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
