// extern "C" boundary of libbdeg.so (include/bdeg.h): planning, device
// workspace, launches, overflow re-runs, re-lifting and the exact combine.
#include "../../include/bdeg.h"
#include "bdeg_internal.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>

using namespace bdeg;

// The work queue of a plan (build_queue): a pure function of the plan's
// shape (K, N, base depth, world, SMs, resident warps), so plans of one shape
// share it (cached; the split table is uploaded once per device).
struct WorkQueue {
    std::vector<uint64_t> split;          // split items (depth << 58 | colex id), largest first
    std::vector<uint64_t> grp_u, grp_cum; // grouped base-depth items
    uint64_t nitems = 0, nstatic_steal = 0, grab = 1;
};

struct bdeg_plan_s {
    // inputs
    bool points_mode = false;
    int n = 0, m = 0;
    std::vector<int64_t> A;
    std::vector<double> bre, bim;
    bool user_lift = false;
    std::vector<int64_t> lift;        // n+1 (system) or N (points) values in use
    bdeg_options opt{};
    // front end
    FrontEnd fe;
    int K = 0, N = 0, origin_index = -1;
    std::vector<int64_t> V, w;        // point-major N x K, and N lifts
    std::vector<int> point_of_var;
    std::vector<int> order;          // system plans: plan point t = configuration point order[t]
    int tier = 0, S = 0, T = 0, D = 0;
    int bits_v = 30, bits_l = 31;
    bool big = false;                 // N > 64: walk only (rank space beyond uint64 / lane slots)
    bool v_safe = false;              // every V-minor < 2^31 - 1 by Hadamard's bound (tier-0 kernels skip V checks)
    bool dead_full = false;           // full mode: detect cell-dead subtrees (degenerate configurations)
    unsigned long long *steal = nullptr;   // cross-GPU item counters (2, by step parity), IPC-mapped
    int steal_parity = 0;
    uint64_t basis_lo = 0, basis_hi = 0;   // basis-seeded start cell (N > 64, generated lifting)
    uint64_t nblocks = 0, total = 0;      // base-depth items (colex range mode), C(N,K)
    std::shared_ptr<const WorkQueue> q = std::make_shared<WorkQueue>();   // work queue (build_queue;
                                                                          // shared by plans of one shape)
    uint64_t seed_used = 0;
    int relifts = 0;
    double plan_ms = 0;
    std::string err;
    // device
    bool dev_ready = false, own_ws = false, l_dirty = true;
    char *ws = nullptr;
    size_t ws_bytes = 0;
    unsigned long long *d_slots = nullptr, *d_ctr = nullptr, *d_ovfq = nullptr;
    uint64_t *d_split = nullptr, *d_gu = nullptr, *d_gc = nullptr;
    int64_t *d_L = nullptr;
    uint64_t *d_B = nullptr;
    uint64_t ovf_words = 1;               // re-run bitmap: one bit per work-queue position
    int grid = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<uint64_t> binom;
};

namespace {

thread_local std::string g_err;

// NVTX range for the scope (plan / enumerate / replays / walk level / finalize)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bdeg_status fail(bdeg_plan_t p, bdeg_status s, const std::string &msg) {
    if (p) p->err = msg;
    g_err = msg;
    return s;
}

uint64_t C(const std::vector<uint64_t> &B, int n, int k) {
    if (n < 0 || k < 0 || k > n) return 0;
    return B[(size_t)n * kBinomCols + k];
}

void fill_binom(std::vector<uint64_t> &B) {
    B.assign((size_t)kBinomRows * kBinomCols, 0);
    for (int n = 0; n < kBinomRows; ++n) {
        B[(size_t)n * kBinomCols] = 1;
        for (int k = 1; k < kBinomCols && k <= n; ++k)
            B[(size_t)n * kBinomCols + k] = B[(size_t)(n - 1) * kBinomCols + k - 1] +
                                            (k <= n - 1 ? B[(size_t)(n - 1) * kBinomCols + k] : 0);
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace layout
constexpr int kMaxGroups = 66;
constexpr uint64_t kMaxOvfWords = 1ull << 21;   // base-depth item groups (one per smallest top index u)
struct Layout {
    size_t slots, ctr, L, B, q, gu, gc, total;
};
Layout layout(const bdeg_plan_s *p) {
    Layout l;
    size_t off = 0;
    l.slots = off; off = align256(off + kNSlots * 8);
    l.ctr = off;   off = align256(off + 8 * 8);
    l.L = off;     off = align256(off + (((size_t)(p->K + 1) * p->N * 8 + 15) & ~(size_t)15));
    l.B = off;     off = align256(off + (size_t)kBinomRows * kBinomCols * 8);
    l.q = off;     off = align256(off + 2 * p->ovf_words * 8);   // bitmaps A (narrow -> int64), B (-> int128)
    l.gu = off;    off = align256(off + kMaxGroups * 8);
    l.gc = off;    off = align256(off + kMaxGroups * 8);
    l.total = off;
    return l;
}

void gen_lifting(uint64_t seed, int count, int bits, std::vector<int64_t> &out) {
    SplitMix64 g(seed);
    out.resize(count);
    const int sh = 64 - std::max(1, std::min(bits, 62));
    for (int i = 0; i < count; ++i) out[i] = (int64_t)(g.next() >> sh);
}

// colex unrank (host planner)
void unrank(const std::vector<uint64_t> &B, uint64_t r, int K, std::vector<int> &c) {
    c.assign(K, 0);
    for (int i = K - 1; i >= 0; --i) {
        int x = i;
        while (C(B, x + 1, i + 1) <= r) ++x;
        c[i] = x;
        r -= C(B, x, i + 1);
    }
}

// work item (D-tuple of the largest indices, colex id) containing `rank`
uint64_t block_of(const bdeg_plan_s *p, uint64_t rank) {
    if (p->D == 0) return 0;
    std::vector<int> c;
    unrank(p->binom, rank, p->K, c);
    const int kd = p->K - p->D;
    uint64_t b = 0;
    for (int t = 0; t < p->D; ++t) b += C(p->binom, c[kd + t] - kd, t + 1);
    return b;
}

// Largest magnitudes (bits) of the fraction-free elimination values of the
// V rows and of the lift row along sampled prefixes, as the kernel computes
// them — steers the choice of the starting tier only (the kernel checks every
// stored value against its tier's bounds and re-runs offending blocks).
// Exact division by d != 0 (the quotient is known to be an integer): in int64
// shift out d's 2-adic part and multiply by the odd part's inverse mod 2^64
// (Newton); int128 divides.
inline uint64_t odd_inverse(int64_t d, int &tz) {
    tz = __builtin_ctzll((uint64_t)d);
    const uint64_t o = (uint64_t)(d >> tz);          // odd part (arithmetic shift keeps the sign)
    uint64_t x = o;                                  // correct to 3 bits
    for (int i = 0; i < 5; ++i) x *= 2 - o * x;
    return x;
}
inline uint64_t odd_inverse(i128, int &tz) { tz = 0; return 0; }
inline int64_t exact_div(int64_t n, int64_t, uint64_t inv, int tz) {
    return (int64_t)((uint64_t)(n >> tz) * inv);
}
inline i128 exact_div(i128 n, i128 d, uint64_t, int) { return n / d; }

// One sampled elimination order (perm) in the integer type T; returns false
// when a product leaves T (the caller retries in the wider type, or gives up).
template <typename T>
bool sample_one(const bdeg_plan_s *p, const std::vector<int> &perm, i128 &mv, i128 &ml) {
    const int K = p->K, N = p->N;
    std::vector<T> M((size_t)(K + 1) * N);          // row i, column l at M[i*N + l]
    for (int l = 0; l < N; ++l) {
        for (int i = 0; i < K; ++i) M[(size_t)i * N + l] = p->V[(size_t)l * K + i];
        M[(size_t)K * N + l] = p->w[l];
    }
    std::vector<char> alive(K, 1);
    T prev = 1;
    T lv = 0, ll = 0;
    for (int t = 0; t < K - 1; ++t) {
        const int piv_c = perm[t];
        int r = -1;
        for (int i = 0; i < K; ++i) if (alive[i] && M[(size_t)i * N + piv_c] != 0) { r = i; break; }
        if (r < 0) break;
        const T piv = M[(size_t)r * N + piv_c];
        int dtz = 0;
        const uint64_t dinv = odd_inverse(prev, dtz);
        for (int i = 0; i <= K; ++i) {
            if (i == r || (i < K && !alive[i])) continue;
            T *row = &M[(size_t)i * N];
            const T *prow = &M[(size_t)r * N];
            const T ci = row[piv_c];
            for (int l = 0; l < N; ++l) {
                T a, b2, num;
                if (__builtin_mul_overflow(piv, row[l], &a) || __builtin_mul_overflow(ci, prow[l], &b2) ||
                    __builtin_sub_overflow(a, b2, &num) || (sizeof(T) == 8 && num == (T)INT64_MIN))
                    return false;
                row[l] = exact_div(num, prev, dinv, dtz);   // exact (Sylvester)
                const T v = row[l] < 0 ? -row[l] : row[l];
                if (i < K) { if (v > lv) lv = v; } else { if (v > ll) ll = v; }
            }
        }
        alive[r] = 0;
        prev = piv;
    }
    if ((i128)lv > mv) mv = lv;
    if ((i128)ll > ml) ml = ll;
    return true;
}

void sample_bits(const bdeg_plan_s *p, int &bv, int &bl) {
    const int K = p->K, N = p->N;
    SplitMix64 g(0x5eed ^ p->seed_used);
    i128 mv = 1, ml = 1;
    bool big = false;
    std::vector<int> perm(N);
    static const int nsamp = [] {            // tuning knob (A/B of planning time vs tier accuracy)
        const char *e = std::getenv("BDEG_TIER_SAMPLES");
        return e ? std::max(1, std::atoi(e)) : 32;
    }();
    for (int s = 0; s < nsamp && !big; ++s) {
        for (int i = 0; i < N; ++i) perm[i] = i;
        for (int i = N - 1; i > 0; --i) std::swap(perm[i], perm[g.next() % (uint64_t)(i + 1)]);
        // int64 first (C5, master spaces), checked int128 when a product leaves it
        if (!sample_one<int64_t>(p, perm, mv, ml) && !sample_one<i128>(p, perm, mv, ml)) big = true;
    }
    auto nbits = [](i128 x) { int b = 0; while (x > 0) { ++b; x >>= 1; } return b; };
    bv = big ? 127 : nbits(mv);
    bl = big ? 127 : nbits(ml);
    for (int l = 0; l < N; ++l) {      // the level-0 values themselves
        int64_t a = p->w[l] < 0 ? -p->w[l] : p->w[l];
        bl = std::max(bl, nbits((i128)a));
        for (int i = 0; i < K; ++i) {
            int64_t v = p->V[(size_t)l * K + i];
            bv = std::max(bv, nbits((i128)(v < 0 ? -v : v)));
        }
    }
}

// A narrow tier (forced by a flag, or chosen before a re-lift) still needs
// the RAW values inside its bounds: the shared-memory prefix multiplies them
// in int64 before any range check, and the narrow walk stores them as int32.
void raw_tier_bounds(bdeg_plan_s *p) {
    int64_t mv = 0, mw = 0;
    for (int64_t v : p->V) mv = std::max(mv, v < 0 ? -v : v);
    for (int64_t v : p->w) mw = std::max(mw, v < 0 ? -v : v);
    if (p->tier == 0 && (mv >= INT32_MAX || mw >= INT32_MAX)) p->tier = 1;
    if (p->tier == 1 && (mv >= ((int64_t)1 << p->bits_v) || mw >= ((int64_t)1 << p->bits_l))) p->tier = 2;
}

// Per-device properties (queried once per process) and a small pool of
// device workspaces, so that planning a new problem does not pay
// cudaGetDeviceProperties / cudaMalloc / cudaFree every time.
struct DevInfo { bool ok = false; int sms = 0, major = 0; };
std::mutex g_mu;
constexpr int kMaxDevices = 64;
DevInfo g_dev[kMaxDevices];
std::vector<std::pair<size_t, void *>> g_pool[kMaxDevices];
std::map<std::string, void *> g_steal_local;   // IPC handles exported by this process

DevInfo g_dev_none;

const DevInfo &dev_info(int d) {
    if (d < 0 || d >= kMaxDevices) return g_dev_none;   // ok = false
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_dev[d].ok) {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, d) == cudaSuccess) {
            g_dev[d].sms = prop.multiProcessorCount;
            g_dev[d].major = prop.major;
            g_dev[d].ok = true;
        }
    }
    return g_dev[d];
}

// ------------------------------------------------------------ work queue
// SURVEY §8.e.  Items are tuples of the largest subset indices (c_{K-d} <
// ... < c_{K-1}); an item of depth d whose smallest index is u holds the
// C(u, K-d) candidates below it (a contiguous colex rank interval).  The
// queue lists the items largest-first: (1) items split to a finer depth (only
// for world > 1: base-depth items larger than a quarter of a warp's share are
// cut one level deeper, recursively), sorted by size; (2) the other base-depth
// items grouped by u, u descending (group g = every (D-1)-subset of
// {u+1..N-1} above u, in colex order).  Positions [0, nstatic) are
// interleaved over the ranks; with cross-GPU stealing the rest is taken from
// one global counter, `grab` positions per atomic.
inline uint64_t colex_id(const std::vector<uint64_t> &B, const int *c, int d, int shift) {
    uint64_t id = 0;
    for (int t = 0; t < d; ++t) id += C(B, c[t] - shift, t + 1);
    return id;
}

int warps_per_sm_estimate(const bdeg_plan_s *p) {
    const int ctas_lb = 4;                               // __launch_bounds__ of k_enumerate
    const size_t smem = enumerate_smem_bytes(p->K, p->N, kernel_warps_per_cta());
    const int ctas_sm = (int)std::max<size_t>(1, (228 * 1024) / (smem + 1024));
    return std::min(ctas_lb, ctas_sm) * kernel_warps_per_cta();
}

std::mutex g_qmu;
std::map<std::vector<int64_t>, std::shared_ptr<const WorkQueue>> g_queue_cache;

void build_queue(bdeg_plan_s *p) {
    const int K = p->K, N = p->N, D = p->D;
    const auto &B = p->binom;
    const int world = std::max(1, p->opt.world);
    const DevInfo &di = dev_info(p->opt.device);
    const double sms = di.ok ? di.sms : 148.0;
    const int wps = warps_per_sm_estimate(p);
    const double warps = sms * wps;
    double frac = 0.25;                                   // largest item <= frac x a warp's share
    if (const char *e = std::getenv("BDEG_SPLIT_SHARE")) frac = std::atof(e);
    const bool do_split = (world > 1 || std::getenv("BDEG_SPLIT_1GPU")) && D > 0 && frac > 0;
    const double cap = std::max(1.0, (double)p->total / (world * warps) * frac);
    int64_t capbits;
    std::memcpy(&capbits, &cap, 8);
    const std::vector<int64_t> key{K, N, D, world, (int64_t)sms, wps, capbits, do_split ? 1 : 0};
    {
        std::lock_guard<std::mutex> lk(g_qmu);
        auto it = g_queue_cache.find(key);
        if (it != g_queue_cache.end()) { p->q = it->second; return; }
    }
    auto Q = std::make_shared<WorkQueue>();
    // split items, bucketed by (depth, smallest index): every item of a bucket
    // has the same size C(u, K-d), so ordering the buckets orders the items
    std::map<std::pair<int, int>, std::vector<uint64_t>> buckets;
    int c[kMaxK + 1];                                     // c[K-d .. K-1]: an item's top indices
    // depth-first split of the node whose indices are c[K-d..K-1]
    auto expand = [&](auto &&self, int d) -> void {
        const int u = c[K - d];
        const uint64_t size = C(B, u, K - d);
        if ((double)size <= cap || d >= K - 1) {
            buckets[{d, u}].push_back(((uint64_t)d << 58) | colex_id(B, c + (K - d), d, K - d));
            return;
        }
        for (int u2 = K - d - 1; u2 < u; ++u2) {
            c[K - d - 1] = u2;
            self(self, d + 1);
        }
    };
    if (D == 0) {
        Q->grp_u.push_back(N);
        Q->grp_cum = {0, 1};
    } else {
        uint64_t cum = 0;
        for (int u = N - D; u >= K - D; --u) {
            const uint64_t cnt = C(B, N - 1 - u, D - 1), sz = C(B, u, K - D);
            if (cnt == 0) continue;
            if (!do_split || (double)sz <= cap || D >= K - 1) {
                Q->grp_u.push_back(u);
                Q->grp_cum.push_back(cum);
                cum += cnt;
                continue;
            }
            // every item of the group: u, then a (D-1)-subset of {u+1..N-1} (colex successor)
            int top[kMaxK];
            top[0] = u;
            for (int t = 1; t < D; ++t) top[t] = u + t;
            for (;;) {
                for (int t = 0; t < D; ++t) c[K - D + t] = top[t];
                expand(expand, D);
                int t = 1;                                // next (D-1)-subset of {u+1..N-1}
                while (t < D && (t + 1 < D ? top[t] + 1 >= top[t + 1] : top[t] + 1 >= N)) ++t;
                if (t >= D) break;
                ++top[t];
                for (int q = 1; q < t; ++q) top[q] = u + q;
            }
        }
        Q->grp_cum.push_back(cum);
    }
    std::vector<std::pair<uint64_t, const std::vector<uint64_t> *>> order;   // (size, bucket)
    size_t nsplit = 0;
    for (const auto &kv : buckets) {
        order.push_back({C(B, kv.first.second, K - kv.first.first), &kv.second});
        nsplit += kv.second.size();
    }
    std::stable_sort(order.begin(), order.end(), [](const auto &x, const auto &y) { return x.first > y.first; });
    Q->split.clear();
    Q->split.reserve(nsplit);
    std::vector<uint64_t> split_size;                    // per split position (for the static share)
    split_size.reserve(nsplit);
    for (const auto &o : order) {
        Q->split.insert(Q->split.end(), o.second->begin(), o.second->end());
        split_size.insert(split_size.end(), o.second->size(), o.first);
    }
    Q->nitems = Q->split.size() + Q->grp_cum.back();
    // static share: the positions holding the first ~80% of the candidates
    // (balanced by the interleave); the rest is the stealing tail
    uint64_t acc = 0, pos = 0;
    const double want = 0.8 * (double)p->total;
    for (size_t i = 0; i < split_size.size() && acc < want; ++i, ++pos) acc += split_size[i];
    for (size_t g = 0; g + 1 < Q->grp_cum.size() && acc < want; ++g) {
        const uint64_t cnt = Q->grp_cum[g + 1] - Q->grp_cum[g];
        const uint64_t sz = D == 0 ? p->total : C(B, Q->grp_u[g], K - D);
        const uint64_t need = sz ? (uint64_t)std::ceil((want - (double)acc) / (double)sz) : cnt;
        const uint64_t take = std::min(cnt, need);
        acc += take * sz;
        pos += take;
    }
    Q->nstatic_steal = world > 1 ? std::min(pos, Q->nitems) : Q->nitems;
    const uint64_t tail = Q->nitems - Q->nstatic_steal;
    Q->grab = std::max<uint64_t>(1, tail / (uint64_t)std::max(1.0, world * warps * 4));
    {
        std::lock_guard<std::mutex> lk(g_qmu);
        if (g_queue_cache.size() > 64) g_queue_cache.clear();   // plans keep their own reference
        g_queue_cache[key] = Q;
    }
    p->q = Q;
}

// queue position -> (depth, tuple of the largest indices, smallest first)
void decode_position(const bdeg_plan_s *p, uint64_t pos, int &d, std::vector<int> &top) {
    const auto &B = p->binom;
    const int K = p->K;
    top.clear();
    if (pos < p->q->split.size()) {
        d = (int)(p->q->split[pos] >> 58);
        uint64_t r = p->q->split[pos] & ((1ull << 58) - 1);
        top.assign(d, 0);
        for (int t = d - 1; t >= 0; --t) {
            int x = t;
            while (C(B, x + 1, t + 1) <= r) ++x;
            r -= C(B, x, t + 1);
            top[t] = x + K - d;
        }
        return;
    }
    d = p->D;
    if (d == 0) return;
    const uint64_t q = pos - p->q->split.size();
    size_t g = 0;
    while (g + 2 < p->q->grp_cum.size() && p->q->grp_cum[g + 1] <= q) ++g;
    const int u = p->q->grp_u[g];
    uint64_t r = q - p->q->grp_cum[g];
    top.assign(d, 0);
    top[0] = u;
    for (int t = d - 2; t >= 0; --t) {
        int x = t;
        while (C(B, x + 1, t + 1) <= r) ++x;
        r -= C(B, x, t + 1);
        top[t + 1] = x + u + 1;
    }
}

// Fraction of singular K-subsets among `samples` random ones (det mod the
// prime 2^31 - 1; a det divisible by p counts as singular: a heuristic).
// Degenerate configurations (master spaces: 60-93 % singular) have many
// cell-dead subtrees, which full mode then detects; random
// configurations (C5: 0.04 %) skip the per-node test.
double sampled_singular_fraction(const bdeg_plan_s *p, int samples) {
    const int K = p->K, N = p->N;
    const uint64_t P = 2147483647ull;                     // Mersenne: x mod P by shifts
    auto red = [P](uint64_t x) { x = (x & P) + (x >> 31); x = (x & P) + (x >> 31); return x >= P ? x - P : x; };
    SplitMix64 g(0xdeadull ^ p->seed_used);
    std::vector<int> idx(N);
    std::vector<uint64_t> M((size_t)K * K);
    int sing = 0;
    for (int s = 0; s < samples; ++s) {
        for (int i = 0; i < N; ++i) idx[i] = i;
        for (int i = 0; i < K; ++i) std::swap(idx[i], idx[i + (int)(g.next() % (uint64_t)(N - i))]);
        for (int r = 0; r < K; ++r)
            for (int c = 0; c < K; ++c) {
                int64_t v = p->V[(size_t)idx[c] * K + r] % (int64_t)P;
                M[(size_t)r * K + c] = (uint64_t)(v < 0 ? v + (int64_t)P : v);
            }
        bool zero = false;
        for (int c = 0; c < K && !zero; ++c) {
            int pr = -1;
            for (int r = c; r < K; ++r) if (M[(size_t)r * K + c]) { pr = r; break; }
            if (pr < 0) { zero = true; break; }
            if (pr != c) for (int t = 0; t < K; ++t) std::swap(M[(size_t)pr * K + t], M[(size_t)c * K + t]);
            // division-free step (row_r <- piv row_r - f row_c): the rank is all that matters
            const uint64_t piv = M[(size_t)c * K + c];
            for (int r = c + 1; r < K; ++r) {
                const uint64_t f = M[(size_t)r * K + c];
                if (!f) continue;
                for (int t = c; t < K; ++t)
                    M[(size_t)r * K + t] = red(red(piv * M[(size_t)r * K + t]) + P - red(f * M[(size_t)c * K + t]));
            }
        }
        sing += zero;
    }
    return samples ? (double)sing / samples : 0.0;
}

void choose_tier_and_blocks(bdeg_plan_s *p) {
    p->total = C(p->binom, p->N, p->K);
    // Register-DFS depth S (deep: the DFS does one fraction-free step per
    // tree node) and smem prefix T = K-1-S
    const int smax = std::min(kMaxInner, p->K - 1);
    // measured (tools/sweep_libs.sh): S = 3 for K = 8, 4-5 for K = 12, 6 for K >= 14
    const int sauto = std::min(smax, std::max(3, p->K / 2 - 1));
    p->S = p->opt.inner_levels >= 0 ? std::min(p->opt.inner_levels, smax) : sauto;
    p->T = p->K - 1 - p->S;
    int bv = 0, bl = 0;
    sample_bits(p, bv, bl);
    p->bits_v = std::min(30, std::max(bv + 2, 8));
    p->bits_l = 61 - p->bits_v;
    if (bv <= 28 && bl <= 28) p->tier = 0;
    else if (bv + 2 <= 30 && bl < p->bits_l) p->tier = 1;
    else p->tier = 2;
    // Hadamard: |det| <= prod of the column norms, so every V-minor (any rows,
    // <= K columns; every V-row value of the elimination is one, by Sylvester's
    // identity) is at most sqrt(product of the K largest squared column norms)
    {
        std::vector<u128> n2(p->N, 0);
        const u128 cap = (u128)1 << 124;
        for (int l = 0; l < p->N; ++l)
            for (int i = 0; i < p->K; ++i) {
                const int64_t v = p->V[(size_t)l * p->K + i];
                const u128 a = (u128)(v < 0 ? -(i128)v : (i128)v);
                n2[l] = std::min(cap, n2[l] + (a > ((u128)1 << 62) ? cap : a * a));
            }
        std::sort(n2.begin(), n2.end(), [](u128 x, u128 y) { return x > y; });
        u128 prod = 1;
        for (int i = 0; i < std::min(p->K, p->N) && prod < cap; ++i) {
            const u128 f = n2[i] == 0 ? 1 : n2[i];
            prod = (f > cap / prod) ? cap : prod * f;
        }
        const u128 lim = (u128)INT32_MAX * (u128)INT32_MAX;
        p->v_safe = prod < lim && !std::getenv("BDEG_NO_VSAFE");
    }
    if (p->opt.flags & BDEG_FLAG_FORCE_TIER0) p->tier = 0;
    if (p->opt.flags & BDEG_FLAG_FORCE_TIER1) p->tier = 1;
    if (p->opt.flags & BDEG_FLAG_FORCE_TIER2) p->tier = 2;
    raw_tier_bounds(p);
    if (const char *e = std::getenv("BDEG_DEAD_FULL")) p->dead_full = std::atoi(e) != 0;   // A/B knob
    else p->dead_full = sampled_singular_fraction(p, 32) > 0.25;
    // The work-item depth D >= T chosen
    // so that the largest item C(N-D, K-D) is a small fraction of the
    // per-warp share (items are processed largest-first).
    const double warps = 148.0 * 16.0;
    double factor = 0.25;
    if (const char *e = std::getenv("BDEG_ITEM_FACTOR")) factor = std::atof(e);   // tuning knob
    const double limit = std::max(1.0, (double)p->total / (warps * factor));
    int D = p->T;
    while (D < p->K - 1 && (double)C(p->binom, p->N - D, p->K - D) > limit) ++D;
    p->D = D;
    p->nblocks = C(p->binom, p->N - p->K + p->D, p->D);
    build_queue(p);
}

// Greedy basis of the point vectors (first K linearly independent points,
// exact rank test by fraction-free elimination in __int128).
bool greedy_basis(const bdeg_plan_s *p, std::vector<int> &basis) {
    const int K = p->K;
    std::vector<std::vector<i128>> rows;   // reduced basis vectors (echelon)
    std::vector<int> lead;
    basis.clear();
    for (int l = 0; l < p->N && (int)basis.size() < K; ++l) {
        std::vector<i128> v(K);
        for (int i = 0; i < K; ++i) v[i] = p->V[(size_t)l * K + i];
        for (size_t r = 0; r < rows.size(); ++r) {
            const int c = lead[r];
            if (v[c] == 0) continue;
            const i128 a = rows[r][c], b = v[c];
            for (int i = 0; i < K; ++i) {
                i128 t1, t2;
                if (__builtin_mul_overflow(a, v[i], &t1) || __builtin_mul_overflow(b, rows[r][i], &t2)) return false;
                v[i] = t1 - t2;
            }
            i128 g = 0;                           // keep entries small
            for (int i = 0; i < K; ++i) { i128 x = v[i] < 0 ? -v[i] : v[i]; while (x) { i128 t = g % x; g = x; x = t; } }
            if (g > 1) for (int i = 0; i < K; ++i) v[i] /= g;
        }
        int c = -1;
        for (int i = 0; i < K; ++i) if (v[i] != 0) { c = i; break; }
        if (c < 0) continue;
        rows.push_back(v);
        lead.push_back(c);
        basis.push_back(l);
    }
    return (int)basis.size() == K;
}

// N > 64 with a generated lifting: lift a basis at 0 and every other point
// at >= 1.  The hyperplane through the lifted basis is then h = 0 (a basis
// spans everything), every other point is strictly above it, so the basis is
// a cell of the regular subdivision: the walk's start cell (the degree does
// not depend on the lifting).
void seed_basis_lifting(bdeg_plan_s *p) {
    if (!p->big || p->user_lift) return;
    std::vector<int> basis;
    if (!greedy_basis(p, basis)) return;
    for (int64_t &w : p->w) if (w < 1) w = 1;
    p->basis_lo = p->basis_hi = 0;
    for (int l : basis) {
        p->w[l] = 0;
        if (l < 64) p->basis_lo |= 1ull << l; else p->basis_hi |= 1ull << (l - 64);
    }
}

bdeg_status finish_plan(bdeg_plan_s *p) {
    if (p->K > kMaxK || p->N > kMaxNWalk)
        return fail(p, BDEG_E_TOO_LARGE, "point configuration exceeds N <= 128, K <= 32 (N=" +
                                              std::to_string(p->N) + ", K=" + std::to_string(p->K) + ")");
    p->big = p->N > kMaxN;
    for (int64_t v : p->V)
        if (v >= ((int64_t)1 << 62) || v <= -((int64_t)1 << 62))
            return fail(p, BDEG_E_TOO_LARGE, "point coordinate beyond 2^62");
    for (int64_t v : p->w)
        if (v >= ((int64_t)1 << 62) || v <= -((int64_t)1 << 62))
            return fail(p, BDEG_E_TOO_LARGE, "lifting value beyond 2^62");
    // Every value the elimination stores is a minor of the lifted (K+1) x N
    // matrix (Sylvester's identity).  Hadamard: a minor of V rows only is at
    // most H_V = the product of the K largest column norms of V; expanding a
    // minor with the lift row along that row, it is at most (K+1) max|w| H_V.
    // Below 2^125 the int128-value tier (the end of the overflow chain) can
    // never overflow.
    {
        std::vector<double> lg(p->N, 0.0);
        double wmax = 1;
        for (int l = 0; l < p->N; ++l) {
            long double n2 = 0;
            for (int i = 0; i < p->K; ++i) n2 += (long double)p->V[(size_t)l * p->K + i] * p->V[(size_t)l * p->K + i];
            lg[l] = n2 > 1 ? 0.5 * std::log2((double)n2) : 0.0;
            wmax = std::max(wmax, std::fabs((double)p->w[l]));
        }
        std::sort(lg.begin(), lg.end(), [](double a, double b) { return a > b; });
        double hv = 0;
        for (int i = 0; i < std::min(p->K, p->N); ++i) hv += lg[i];
        // the same by rows (tighter when a row is small, e.g. the row of ones
        // of an affine configuration): each row restricted to its K largest
        // entries, factors below 1 counted as 1 (minors of fewer rows)
        double hr = 0;
        for (int i = 0; i < p->K; ++i) {
            std::vector<long double> sq(p->N);
            for (int l = 0; l < p->N; ++l) sq[l] = (long double)p->V[(size_t)l * p->K + i] * p->V[(size_t)l * p->K + i];
            std::sort(sq.begin(), sq.end(), [](long double a, long double b) { return a > b; });
            long double n2 = 0;
            for (int l = 0; l < std::min(p->K, p->N); ++l) n2 += sq[l];
            hr += n2 > 1 ? 0.5 * std::log2((double)n2) : 0.0;
        }
        hv = std::min(hv, hr);
        const double bound = std::max(hv, std::log2((double)(p->K + 1)) + std::log2(wmax) + hv);
        if (bound >= 124.9)
            return fail(p, BDEG_E_TOO_LARGE, "Hadamard bound of the lifted minors is 2^" + std::to_string((int)bound) +
                                                 " >= 2^125 (beyond the int128 tier)");
    }
    if (p->big) {
        // walk only: no rank space (C(N,K) may exceed 2^64), no enumeration items
        int bv = 0, bl = 0;
        sample_bits(p, bv, bl);
        p->bits_v = std::min(30, std::max(bv + 2, 8));
        p->bits_l = 61 - p->bits_v;
        p->tier = (bv <= 28 && bl <= 28) ? 0 : ((bv + 2 <= 30 && bl < p->bits_l) ? 1 : 2);
        if (p->opt.flags & BDEG_FLAG_FORCE_TIER0) p->tier = 0;
        if (p->opt.flags & BDEG_FLAG_FORCE_TIER1) p->tier = 1;
        if (p->opt.flags & BDEG_FLAG_FORCE_TIER2) p->tier = 2;
        p->total = 0;
        p->S = p->T = p->D = 0;
        p->nblocks = 0;
        seed_basis_lifting(p);
        raw_tier_bounds(p);
    } else {
        choose_tier_and_blocks(p);
    }
    // the re-run bitmaps have one bit per work item (either mode), up to 2^27
    // items (16 MB each); positions beyond that are counted in SLOT_QFULL and
    // the synchronous entry points redo the whole space in tier 2
    p->ovf_words = std::min<uint64_t>((std::max<uint64_t>(std::max(p->nblocks, p->q->nitems), 1) + 63) / 64,
                                      kMaxOvfWords);
    p->l_dirty = true;
    return BDEG_OK;
}

// rebuild V/w from the current lifting (system plans), in the plan's point
// order: fixed at planning time as the points sorted by ascending lifting
// residual (the lifting minus its least-squares linear fit; stable;
// BDEG_FLAG_NATURAL_ORDER keeps first occurrence).  High points are fixed
// first by the colex DFS, so cell-dead prefixes are found higher up.  The
// order changes which K-subsets share prefixes, never a result (reading O);
// measured on the master spaces (profiles/r2aq/r2az_order_sweep.jsonl) against
// first occurrence: W_{2,6} -15 %, W_{2,5} -23 %, W_{2,7} -13 %, W_{3,5} and
// W_{4,4} degree-only -17 % and -12 %.  Re-lifts keep the order.
void rebuild_points(bdeg_plan_s *p) {
    build_points(p->fe, p->lift.data(), !(p->opt.flags & BDEG_FLAG_NO_HOMOG_SHORTCUT), p->K, p->N, p->V,
                 p->w, p->point_of_var, p->origin_index);
    if (p->opt.flags & BDEG_FLAG_NATURAL_ORDER) return;
    if ((int)p->order.size() != p->N) {
        // sort key: the lifting minus its least-squares linear fit (normal
        // equations in double; only an order, so rounding is harmless) -- adding
        // a linear function to the lifting changes neither the subdivision nor
        // this key (the raw lifting would be ordered by the added function)
        const int K = p->K, N = p->N;
        std::vector<double> G((size_t)K * K, 0.0), r(K, 0.0), h(K, 0.0), key(N);
        for (int l = 0; l < N; ++l)
            for (int i = 0; i < K; ++i) {
                const double vi = (double)p->V[(size_t)l * K + i];
                r[i] += vi * (double)p->w[l];
                for (int j = 0; j < K; ++j) G[(size_t)i * K + j] += vi * (double)p->V[(size_t)l * K + j];
            }
        bool ok = true;                        // Gaussian elimination with partial pivoting
        for (int c = 0; c < K && ok; ++c) {
            int piv = c;
            for (int i = c + 1; i < K; ++i)
                if (std::fabs(G[(size_t)i * K + c]) > std::fabs(G[(size_t)piv * K + c])) piv = i;
            if (std::fabs(G[(size_t)piv * K + c]) < 1e-300) { ok = false; break; }
            if (piv != c) {
                for (int j = 0; j < K; ++j) std::swap(G[(size_t)c * K + j], G[(size_t)piv * K + j]);
                std::swap(r[c], r[piv]);
            }
            for (int i = c + 1; i < K; ++i) {
                const double f = G[(size_t)i * K + c] / G[(size_t)c * K + c];
                for (int j = c; j < K; ++j) G[(size_t)i * K + j] -= f * G[(size_t)c * K + j];
                r[i] -= f * r[c];
            }
        }
        for (int c = K - 1; c >= 0 && ok; --c) {
            double t = r[c];
            for (int j = c + 1; j < K; ++j) t -= G[(size_t)c * K + j] * h[j];
            h[c] = t / G[(size_t)c * K + c];
        }
        for (int l = 0; l < N; ++l) {
            double fit = 0;
            if (ok)
                for (int i = 0; i < K; ++i) fit += h[i] * (double)p->V[(size_t)l * K + i];
            key[l] = (double)p->w[l] - fit;
        }
        p->order.resize(N);
        for (int l = 0; l < N; ++l) p->order[l] = l;
        std::stable_sort(p->order.begin(), p->order.end(), [&](int a, int b) { return key[a] < key[b]; });
    }
    std::vector<int64_t> V2((size_t)p->N * p->K), w2(p->N);
    std::vector<int> pos(p->N);
    for (int t = 0; t < p->N; ++t) {
        const int l = p->order[t];
        for (int i = 0; i < p->K; ++i) V2[(size_t)t * p->K + i] = p->V[(size_t)l * p->K + i];
        w2[t] = p->w[l];
        pos[l] = t;
    }
    p->V.swap(V2);
    p->w.swap(w2);
    for (int &v : p->point_of_var)
        if (v >= 0) v = pos[v];
    if (p->origin_index >= 0) p->origin_index = pos[p->origin_index];
}

// The split-item table of a work queue on the plan's device: uploaded once
// per (device, queue) and kept for the process (queues are cached by shape).
std::map<std::pair<int, const WorkQueue *>, std::pair<std::shared_ptr<const WorkQueue>, uint64_t *>> g_dsplit;

uint64_t *device_split_table(bdeg_plan_s *p) {
    if (p->q->split.empty()) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    const auto key = std::make_pair(p->opt.device, p->q.get());
    auto it = g_dsplit.find(key);
    if (it != g_dsplit.end()) return it->second.second;
    uint64_t *d = nullptr;
    if (cudaMalloc(&d, p->q->split.size() * 8) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, p->q->split.data(), p->q->split.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    g_dsplit[key] = {p->q, d};                 // holds the queue: the pointer key stays unique
    return d;
}

void *pool_get(int d, size_t bytes, size_t *got) {
    if (d >= 0 && d < kMaxDevices) {
        std::lock_guard<std::mutex> lk(g_mu);
        auto &v = g_pool[d];
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].first >= bytes) {
                void *ptr = v[i].second;
                *got = v[i].first;
                v.erase(v.begin() + i);
                return ptr;
            }
    }
    void *ptr = nullptr;
    if (cudaMalloc(&ptr, bytes) != cudaSuccess) return nullptr;
    *got = bytes;
    return ptr;
}

void pool_put(int d, void *ptr, size_t bytes) {
    if (d < 0 || d >= kMaxDevices) { cudaFree(ptr); return; }
    std::lock_guard<std::mutex> lk(g_mu);
    auto &v = g_pool[d];
    if (v.size() < 8) v.push_back({bytes, ptr});
    else cudaFree(ptr);
}

bdeg_status ensure_device(bdeg_plan_s *p) {
    cudaError_t e;
    if (p->opt.device < 0 || p->opt.device >= kMaxDevices)
        return fail(p, BDEG_E_INVALID, "device ordinal out of range");
    if (p->dev_ready || p->opt.device >= 0) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= p->opt.device)
            return fail(p, BDEG_E_CUDA, "no CUDA device available (libbdeg has no CPU fallback)");
        // every device entry point runs on the plan's device (one process may drive several)
        if ((e = cudaSetDevice(p->opt.device)) != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(e));
    }
    if (!p->dev_ready) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= p->opt.device)
            return fail(p, BDEG_E_CUDA, "no CUDA device available (libbdeg has no CPU fallback)");

        const DevInfo &di = dev_info(p->opt.device);
        if (!di.ok) return fail(p, BDEG_E_CUDA, "cudaGetDeviceProperties failed");
        if (di.major < 10) return fail(p, BDEG_E_CUDA, "libbdeg is built for sm_100a (B200); device is older");
        const Layout L = layout(p);
        if (!p->ws) {
            size_t got = 0;
            p->ws = (char *)pool_get(p->opt.device, L.total, &got);
            if (!p->ws) return fail(p, BDEG_E_CUDA, "cudaMalloc of the workspace failed");
            p->own_ws = true;
            p->ws_bytes = got;
        } else if (p->ws_bytes < L.total) {
            return fail(p, BDEG_E_INVALID, "workspace too small");
        }
        p->d_slots = reinterpret_cast<unsigned long long *>(p->ws + L.slots);
        p->d_ctr = reinterpret_cast<unsigned long long *>(p->ws + L.ctr);
        p->d_L = reinterpret_cast<int64_t *>(p->ws + L.L);
        p->d_B = reinterpret_cast<uint64_t *>(p->ws + L.B);
        p->d_ovfq = reinterpret_cast<unsigned long long *>(p->ws + L.q);
        if ((e = cudaMemsetAsync(p->d_ovfq, 0, 2 * p->ovf_words * 8, (cudaStream_t)p->opt.stream)) != cudaSuccess)
            return fail(p, BDEG_E_CUDA, cudaGetErrorString(e));      // the replay keeps it clean after this
        p->d_split = device_split_table(p);
        p->d_gu = reinterpret_cast<uint64_t *>(p->ws + L.gu);
        p->d_gc = reinterpret_cast<uint64_t *>(p->ws + L.gc);
        cudaStream_t st = (cudaStream_t)p->opt.stream;
        if ((e = cudaMemcpyAsync(p->d_B, p->binom.data(), p->binom.size() * 8, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess)
            return fail(p, BDEG_E_CUDA, cudaGetErrorString(e));
        // the work queue (plan-constant): split items and the group tables
        if (!p->q->split.empty() && !p->d_split) return fail(p, BDEG_E_CUDA, "upload of the split-item table failed");
        if (!p->q->grp_u.empty() &&
            ((e = cudaMemcpyAsync(p->d_gu, p->q->grp_u.data(), p->q->grp_u.size() * 8, cudaMemcpyHostToDevice, st)) !=
                 cudaSuccess ||
             (e = cudaMemcpyAsync(p->d_gc, p->q->grp_cum.data(), p->q->grp_cum.size() * 8, cudaMemcpyHostToDevice, st)) !=
                 cudaSuccess))
            return fail(p, BDEG_E_CUDA, cudaGetErrorString(e));
        if ((e = cudaEventCreate(&p->ev0)) != cudaSuccess || (e = cudaEventCreate(&p->ev1)) != cudaSuccess)
            return fail(p, BDEG_E_CUDA, std::string("cudaEventCreate: ") + cudaGetErrorString(e));
        LaunchArgs a{};
        a.P.K = p->K; a.P.N = p->N; a.P.S = p->S; a.P.T = p->T;
        a.tier = p->tier;
        const int occ = std::max(enumerate_max_ctas_per_sm(a), 1);
        const int per_sm = p->opt.ctas_per_sm > 0 ? std::min(p->opt.ctas_per_sm, occ) : occ;
        p->grid = di.sms * per_sm;
        p->dev_ready = true;
    }
    if (p->l_dirty) {
        // lifted matrix, column-major (K+1) x N, padded to 16 bytes
        std::vector<int64_t> Lh((size_t)(p->K + 1) * p->N + 2, 0);
        for (int l = 0; l < p->N; ++l) {
            for (int i = 0; i < p->K; ++i) Lh[(size_t)l * (p->K + 1) + i] = p->V[(size_t)l * p->K + i];
            Lh[(size_t)l * (p->K + 1) + p->K] = p->w[l];
        }
        const size_t bytes = (((size_t)(p->K + 1) * p->N * 8 + 15) & ~(size_t)15);
        if ((e = cudaMemcpyAsync(p->d_L, Lh.data(), bytes, cudaMemcpyHostToDevice, (cudaStream_t)p->opt.stream)) !=
            cudaSuccess)
            return fail(p, BDEG_E_CUDA, cudaGetErrorString(e));
        // pageable source: make sure the copy has consumed Lh before it dies
        cudaStreamSynchronize((cudaStream_t)p->opt.stream);
        p->l_dirty = false;
    }
    return BDEG_OK;
}

// Enqueue the enumeration of ranks [b, e) (this rank's interleaved share of
// blocks) accumulating into `slots` (zeroed here).
bdeg_status enqueue_range(bdeg_plan_s *p, uint64_t b, uint64_t e, unsigned long long *slots, int rank,
                          int world, int force_tier, unsigned long long *cells_out = nullptr,
                          unsigned long long *cells_cnt = nullptr, uint64_t cells_cap = 0,
                          bool first_cell_search = false) {
    Nvtx range("bdeg enumerate (main + replays)");
    cudaStream_t st = (cudaStream_t)p->opt.stream;
    cudaError_t ce;
    if ((ce = cudaMemsetAsync(slots, 0, kNSlots * 8, st)) != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    if ((ce = cudaMemsetAsync(p->d_ctr, 0, 8 * 8, st)) != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    if (e > p->total) e = p->total;
    if (b >= e) return BDEG_OK;
    LaunchArgs a{};
    a.P.L = p->d_L;
    a.P.binom = p->d_B;
    a.P.K = p->K; a.P.N = p->N; a.P.S = p->S; a.P.T = p->T; a.P.D = p->D;
    a.rank_begin = b;
    a.rank_end = e;
    a.rank = rank;
    a.world = std::max(world, 1);
    if (b == 0 && e >= p->total) {        // the whole space: the largest-first work queue
        a.mode = 1;
        a.split = p->d_split;
        a.n_split = p->q->split.size();
        a.grp_u = p->d_gu;
        a.grp_cum = p->d_gc;
        a.n_grp = (int)p->q->grp_u.size();
        a.n_items = p->q->nitems;
    } else {                              // a rank range: contiguous base-depth items
        a.mode = 0;
        a.blk_first = block_of(p, b);
        a.blk_last = block_of(p, e - 1);
        a.n_items = a.blk_last - a.blk_first + 1;
    }
    a.n_static = a.n_items;
    a.grab = 1;
    a.slots = slots;
    a.ovf_words = std::min<uint64_t>((a.n_items + 63) / 64, p->ovf_words);
    unsigned long long *bitsA = p->d_ovfq, *bitsB = p->d_ovfq + p->ovf_words;
    a.grid = p->grid;
    a.stream = st;
    a.tier = force_tier >= 0 ? force_tier : p->tier;
    if (a.tier == 0 && p->v_safe) a.tier = 3;   // tier 0 without V-row range checks (Hadamard)
    a.bits_v = p->bits_v;
    a.degree_only = (p->opt.flags & BDEG_FLAG_DEGREE_ONLY) ? 1 : 0;
    a.dead_full = p->dead_full ? 1 : 0;
    a.cells_out = cells_out;
    a.cells_cnt = cells_cnt;
    a.cells_cap = cells_cap;
    if (first_cell_search) {            // any one cell, as fast as possible
        a.degree_only = 1;
        a.stop_on_cell = 1;
    }
    a.bits_l = p->bits_l;
    a.replay = 0;
    a.counter = p->d_ctr + 0;
    if (p->steal && world > 1 && a.mode == 1) {
        // static interleaved share of the first ~80% of the candidates, then
        // one global tail queue over all GPUs (system-scope atomics, NVLink)
        a.n_static = p->q->nstatic_steal;
        a.grab = p->q->grab;
        a.gcounter = p->steal + p->steal_parity;
        a.system_counter = 1;
        if (rank == 0) a.reset_next = p->steal + (p->steal_parity ^ 1);
        p->steal_parity ^= 1;
    }
    // overflow chain: an item that leaves its tier is marked
    // and redone by the next one — narrow (tiers 0/1/3) -> tier 2 (int64
    // values, checked int128 products) -> tier 4 (int128 values, 256-bit)
    a.mark_bits = a.tier == 2 ? bitsB : bitsA;
    int rc = launch_enumerate(a);
    if (rc) return fail(p, BDEG_E_CUDA, std::string("k_enumerate launch: ") + cudaGetErrorString((cudaError_t)rc));
    a.replay = 1;
    a.gcounter = nullptr;
    a.system_counter = 0;
    a.reset_next = nullptr;
    a.stop_on_cell = 0;
    if (a.tier != 2) {
        a.tier = 2;
        a.counter = p->d_ctr + 1;
        a.replay_bits = bitsA;
        a.mark_bits = bitsB;
        a.replay_gate = slots + SLOT_OVF_BLOCKS;   // items the narrow launch marked
        rc = launch_enumerate(a);
        if (rc) return fail(p, BDEG_E_CUDA, std::string("k_enumerate replay: ") + cudaGetErrorString((cudaError_t)rc));
    }
    a.counter = p->d_ctr + 3;
    a.replay_bits = bitsB;
    a.mark_bits = nullptr;
    a.replay_gate = slots + SLOT_WIDE;             // items the tier-2 launches marked
    rc = launch_enumerate_wide(a);
    if (rc) return fail(p, BDEG_E_CUDA, std::string("k_enumerate_wide: ") + cudaGetErrorString((cudaError_t)rc));
    return BDEG_OK;
}

void fill_front(const bdeg_plan_s *p, bdeg_result *r) {
    std::memset(r, 0, sizeof(*r));
    r->n = p->points_mode ? p->N : p->fe.n;
    r->rank = p->points_mode ? 0 : p->fe.rank;
    r->dim = p->points_mode ? p->K - 1 : p->fe.dim;
    r->K = p->K;
    r->N = p->N;
    r->tier = p->tier;
    r->homogeneous = p->points_mode ? 0 : (p->fe.homogeneous && !(p->opt.flags & BDEG_FLAG_NO_HOMOG_SHORTCUT));
    r->inner_levels = p->S;
    r->comp_lo = p->points_mode ? 1 : (uint64_t)p->fe.components;
    r->comp_hi = p->points_mode ? 0 : (uint64_t)(p->fe.components >> 64);
    r->consistent = p->points_mode ? 1 : p->fe.consistent;
    r->seed_used = p->seed_used;
    r->singular_complete = (p->opt.flags & BDEG_FLAG_DEGREE_ONLY) ? 0 : 1;
    r->dead_full = p->dead_full ? 1 : 0;
    r->relifts = p->relifts;
    r->total_candidates = p->total;
    r->plan_ms = p->plan_ms;
}

bdeg_status slots_to_result(bdeg_plan_s *p, const int64_t *h, bdeg_result *r) {
    if (h[SLOT_FATAL] > 0)
        return fail(p, BDEG_E_TOO_LARGE, "an exact elimination value exceeded the int128 tier (|v| >= 2^125)");
    u128 vol = 0;
    for (int i = 3; i >= 0; --i) vol = (vol << 32) + (u128)(uint64_t)h[SLOT_VOL0 + i];
    r->deg_lo = (uint64_t)vol;
    r->deg_hi = (int64_t)(uint64_t)(vol >> 64);
    r->cells = (uint64_t)h[SLOT_CELLS];
    r->singular = (uint64_t)h[SLOT_SINGULAR];
    r->candidates = (uint64_t)h[SLOT_CAND];
    r->ties = (uint64_t)h[SLOT_TIES];
    r->overflow_reruns = (uint64_t)h[SLOT_OVF_BLOCKS];
    r->wide_reruns = (uint64_t)h[SLOT_WIDE];
    r->updates = (uint64_t)h[SLOT_UPDATES];
    r->leaves = (uint64_t)h[SLOT_LEAVES];
    r->dead_leaves = (uint64_t)h[SLOT_DEAD];
    return BDEG_OK;
}

// one synchronous pass over [b, e) on this GPU; re-runs everything in the
// int64 tier if an overflowing item lay beyond the re-run bitmap.
bdeg_status run_sync(bdeg_plan_s *p, uint64_t b, uint64_t e, int64_t *h, double *kms) {
    cudaStream_t st = (cudaStream_t)p->opt.stream;
    bdeg_status s = ensure_device(p);
    if (s) return s;
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(p->ev0, st);
        s = enqueue_range(p, b, e, p->d_slots, 0, 1, pass == 0 ? -1 : 2);
        if (s) return s;
        cudaEventRecord(p->ev1, st);
        cudaError_t ce = cudaMemcpyAsync(h, p->d_slots, kNSlots * 8, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
        float ms = 0;
        cudaEventElapsedTime(&ms, p->ev0, p->ev1);
        *kms += ms;
        if (h[SLOT_QFULL] == 0) return BDEG_OK;
    }
    return fail(p, BDEG_E_TOO_LARGE, "values beyond int64 in more work items than the re-run bitmap holds");
}

// Device buffers of one walk (freed on scope exit).
struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    bool alloc(size_t bytes) {
        if (p) { cudaFree(p); p = nullptr; }
        return cudaMalloc(&p, bytes) == cudaSuccess;
    }
    unsigned long long *u() const { return (unsigned long long *)p; }
};

// Cells (mask, |det|) of ranks [b, e) into host memory (tier 2: no replays,
// so nothing is emitted twice).
bdeg_status cells_range(bdeg_plan_s *p, uint64_t b, uint64_t e, uint64_t *h_out, uint64_t cap, uint64_t *count,
                        bool first_cell_search = false) {
    bdeg_status s = ensure_device(p);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)p->opt.stream;
    DevBuf buf, cnt;
    if (!buf.alloc((2 * std::max<uint64_t>(cap, 1)) * 8) || !cnt.alloc(8))
        return fail(p, BDEG_E_CUDA, "cudaMalloc failed");
    cudaMemsetAsync(cnt.p, 0, 8, st);
    s = enqueue_range(p, b, e, p->d_slots, 0, 1, 2, buf.u(), cnt.u(), cap, first_cell_search);
    if (s) return s;
    uint64_t n = 0;
    int64_t h[kNSlots];
    cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h, p->d_slots, kNSlots * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    // tier 2, then tier 4 for the items whose values left int64
    if (h[SLOT_FATAL] > 0)
        return fail(p, BDEG_E_TOO_LARGE, "cell emission: an exact elimination value exceeded the int128 tier");
    // a would-be cell on a tie: the lifting is not generic, the list is not a subdivision
    if (h[SLOT_TIES] > 0)
        return fail(p, BDEG_E_DEGENERATE, "degenerate lifting: a would-be cell has a zero facet value");
    const uint64_t m = std::min(n, cap);
    if (m && h_out) {
        ce = cudaMemcpyAsync(h_out, buf.p, m * 16, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    }
    *count = n;
    return BDEG_OK;
}

uint64_t pow2_at_least(uint64_t x) {
    uint64_t c = 1;
    while (c < x) c <<= 1;
    return c;
}

// One breadth-first walk of the subdivision.  Cell masks are
// 16-byte {lo, hi} pairs.
bdeg_status walk_once(bdeg_plan_s *p, bdeg_result *r, double *kms) {
    Nvtx range("bdeg walk");
    cudaStream_t st = (cudaStream_t)p->opt.stream;
    const double t0 = now_ms();
    uint64_t start[2] = {0, 0};
    if (p->big) {
        // basis-seeded lifting: the basis is a cell by construction
        if (p->user_lift || (p->basis_lo == 0 && p->basis_hi == 0))
            return fail(p, BDEG_E_INVALID, "N > 64 needs a generated lifting (basis-seeded start cell)");
        start[0] = p->basis_lo;
        start[1] = p->basis_hi;
    } else {
        // a starting cell: the enumeration kernel over the whole rank space in
        // degree-only mode (cell-dead subtrees skipped), stopping at the first
        // cell any warp verifies (tier 2: no replays, exact)
        uint64_t pair[2 * 64];
        uint64_t n = 0;
        bdeg_status s = cells_range(p, 0, p->total, pair, 64, &n, true);
        if (s) return s;
        if (n == 0) return fail(p, BDEG_E_DEGENERATE, "no cell found (degenerate lifting)");
        start[0] = pair[0];
    }
    const double t_start = now_ms();
    const bool dbg = std::getenv("BDEG_DEBUG") != nullptr;
    const int K = p->K;
    int levels = 0;
    uint64_t cap = 1ull << 20, ncur = 1, total_cells = 1, ccap = 1 << 16, ncap = 1 << 16;
    if (const char *c0 = std::getenv("BDEG_WALK_CAP0"))   // test knob: initial hash set slots
        cap = pow2_at_least(std::max<uint64_t>(64, std::strtoull(c0, nullptr, 10)));
    DevBuf table, tags, cur, nxt, aux;
    if (!table.alloc(cap * 16) || !tags.alloc(cap) || !cur.alloc(ccap * 16) || !nxt.alloc(ncap * 16) ||
        !aux.alloc(16 * 8))
        return fail(p, BDEG_E_CUDA, "cudaMalloc failed");
    // aux: [0] next count, [1] work counter, [2..9] stats, [10..14] level volume limbs + cells
    unsigned long long *next_cnt = aux.u(), *counter = aux.u() + 1, *stats = aux.u() + 2, *lvol = aux.u() + 10;
    cudaMemsetAsync(table.p, 0, cap * 16, st);
    cudaMemsetAsync(tags.p, 0, cap, st);                 // level 0 (the start cell) has tag 0
    const uint64_t h0 = (uint64_t)(((u128)walk_hash(start[0], start[1]) * cap) >> 64);   // = device range reduction
    cudaMemcpyAsync((char *)table.p + h0 * 16, start, 16, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(cur.p, start, 16, cudaMemcpyHostToDevice, st);
    const int grid = std::max(1, dev_info(p->opt.device).sms) * 4;
    // int64 fast path of the ridge elimination: the plan's tier bounds
    // (tier 0: 2^31 / 2^31, tier 1: 2^Bv / 2^Bl); tier 2 plans go wide at once
    const int64_t limV = p->tier == 2 ? 0 : (int64_t)1 << (p->tier == 0 ? 30 : p->bits_v);
    const int64_t limL = p->tier == 2 ? 0 : (int64_t)1 << (p->tier == 0 ? 31 : p->bits_l);
    uint64_t ridges = 0, boundary = 0, fused_cells = 0, wide_cells = 0, collects = 0, narrow_redo = 0;
    // int32-storage D&C walk for tier-0 plans (values < 2^30, lifts < 2^31)
    const int narrow = (p->tier == 0 && !std::getenv("BDEG_WALK_WIDE")) ? 1 : 0;
    DevBuf ovfl;
    uint64_t ovfl_cap = 0;
    u128 fused_vol = 0;
    int fused = 0;
    double growth = K;                                   // expected next / current frontier size
    const bool tight = std::getenv("BDEG_WALK_TIGHT") != nullptr;
    if (tight) growth = 0;
    // Breadth-first window (fused D&C walk only; the separate volume pass
    // needs every cell): the table must hold levels L-1, L, L+1 while level
    // L is expanded, so older levels are dropped whenever the table is
    // rebuilt.  lsz[l] = cells of level l; live = cells in the table.
    std::vector<uint64_t> lsz{1};
    uint64_t live = 1, evictions = 0;
    int oldest = 0;                                      // oldest level possibly in the table
    // keep_from >= 0: keep only levels keep_from .. keep_from+2
    auto grow_table = [&](uint64_t ncap_t, int keep_from = -1) -> bdeg_status {
        DevBuf t2, g2;
        if (!t2.alloc(ncap_t * 16) || !g2.alloc(ncap_t))
            return fail(p, BDEG_E_TOO_LARGE, "cell walk: hash set of " + std::to_string(ncap_t) +
                                                 " slots does not fit in device memory");
        cudaMemsetAsync(t2.p, 0, ncap_t * 16, st);
        cudaMemsetAsync(g2.p, 0, ncap_t, st);
        cudaMemsetAsync(stats, 0, 8 * 8, st);
        int rc = launch_rehash(table.p, (const uint8_t *)tags.p, cap, t2.p, (uint8_t *)g2.p, ncap_t, stats + 3, st,
                               (uint8_t)(keep_from & 255), keep_from >= 0 ? 3 : 0);
        if (keep_from >= 0) {
            oldest = keep_from;
            ++evictions;
        }
        if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
        cudaStreamSynchronize(st);
        std::swap(table.p, t2.p);
        std::swap(tags.p, g2.p);
        cap = ncap_t;
        return BDEG_OK;
    };
    // the largest table (17 B per slot, a multiple of 1024 slots) that fits beside `keep` bytes
    auto mem_cap = [&](uint64_t keep) -> uint64_t {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const uint64_t avail = fr > keep + (2ull << 30) ? fr - keep - (2ull << 30) : 0;
        return std::max<uint64_t>(1024, (uint64_t)((avail / 17) & ~1023ull));
    };
    auto round_up = [](uint64_t x) -> uint64_t { return (x + 1023) & ~1023ull; };
    while (ncur > 0) {
        const double t_level = now_ms();
        const uint64_t est = std::min<uint64_t>(ncur * (uint64_t)K, (uint64_t)(ncur * growth) + (tight ? 1 : 1024));
        // hash set at load <= 1/2 for the expected growth (<= 3/4 when device
        // memory is the limit); a level that overflows it is re-run
        const int L = levels;
        const uint64_t window = (L > 0 ? lsz[L - 1] : 0) + lsz[L];
        // evict when the table is due to grow (or the level tags would wrap)
        const bool evictable = fused && L >= 2 && oldest < L - 1;
        if (evictable && (L - oldest >= 250 || (live + est) * 2 > cap)) {
            // rebuild from the frontier buffers: level L is `cur`, level L-1 is
            // still in `nxt` (the previous `cur`), so the old table is dropped
            // first and the new one can take all free memory
            cudaStreamSynchronize(st);
            table.alloc(0);
            tags.alloc(0);
            // (free memory already excludes cur and nxt; keep room for a larger nxt)
            const uint64_t lim = mem_cap(est > ncap ? round_up(est + est / 8) * 16 : 0);
            const uint64_t want = std::min(std::max<uint64_t>(round_up(3 * (window + est)), 1024), lim);
            if (want * 3 < window * 4)
                return fail(p, BDEG_E_TOO_LARGE, "cell walk: " + std::to_string(window) +
                                                     " cells of two levels exceed the hash set that fits in device memory");
            if (!table.alloc(want * 16) || !tags.alloc(want))
                return fail(p, BDEG_E_TOO_LARGE, "cell walk: cudaMalloc of the hash set failed");
            cap = want;
            cudaMemsetAsync(table.p, 0, cap * 16, st);
            cudaMemsetAsync(tags.p, 0, cap, st);
            cudaMemsetAsync(stats, 0, 8 * 8, st);
            int rc = launch_insert_list(nxt.p, lsz[L - 1], table.p, (uint8_t *)tags.p, cap, (uint8_t)((L - 1) & 255),
                                        stats + 3, st);
            if (!rc) rc = launch_insert_list(cur.p, ncur, table.p, (uint8_t *)tags.p, cap, (uint8_t)(L & 255),
                                             stats + 3, st);
            if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
            uint64_t fullc = 0;
            cudaMemcpyAsync(&fullc, stats + 3, 8, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            if (fullc) return fail(p, BDEG_E_TOO_LARGE, "cell walk: window rebuild overflowed the hash set");
            oldest = L - 1;
            ++evictions;
            live = window;
        }
        const uint64_t need = live + est;
        if (need * 2 > cap) {
            uint64_t want = round_up(3 * need);
            // old table still live (already excluded from free memory); room for a larger nxt
            const uint64_t lim = std::max(cap, mem_cap(est > ncap ? round_up(est + est / 8) * 16 : 0));
            if (want > lim) want = lim;
            if (want > cap) {
                bdeg_status s = grow_table(want);
                if (s) return s;
            }
            if (need * 4 > cap * 3)
                return fail(p, BDEG_E_TOO_LARGE, "cell walk: " + std::to_string(need) +
                                                     " cells exceed the hash set that fits in device memory");
        }
        if (est > ncap) {                          // next frontier (collected from the table if it overflows)
            ncap = round_up(est + est / 8);
            if (!nxt.alloc(ncap * 16)) return fail(p, BDEG_E_TOO_LARGE, "cudaMalloc (frontier) failed");
        }
        const unsigned tag = (unsigned)(levels + 1) & 255u;
        cudaMemsetAsync(aux.p, 0, 16 * 8, st);
        uint64_t h[16];
        for (int attempt = 0;; ++attempt) {
            const uint64_t ocap = std::min<uint64_t>(ncur, 1ull << 20);
            if (narrow && ocap > ovfl_cap) {
                ovfl_cap = pow2_at_least(ocap);
                if (!ovfl.alloc(ovfl_cap * 16)) return fail(p, BDEG_E_CUDA, "cudaMalloc (walk overflow list) failed");
            }
            int rc = launch_walk(p->d_L, K, p->N, cur.p, ncur, nxt.p, next_cnt, table.p, cap, counter, stats,
                                 grid, st, limV, limL, lvol, &fused, (uint8_t *)tags.p, tag, ncap,
                                 narrow, ovfl.p, aux.u() + 15, ovfl_cap, p->v_safe ? 1 : 0);
            if (rc) return fail(p, BDEG_E_CUDA, std::string("k_walk: ") + cudaGetErrorString((cudaError_t)rc));
            cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
            cudaError_t ce = cudaStreamSynchronize(st);
            if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
            if (narrow && h[15] > 0) {
                // cells whose values left int32: redo them with int64 storage (their
                // volumes were not counted; neighbours they inserted are exact)
                const bool listed = h[15] <= ovfl_cap;
                if (listed) cudaMemsetAsync(counter, 0, 8, st);
                else cudaMemsetAsync(counter, 0, 15 * 8, st);   // list overflow: redo the whole level wide
                cudaMemsetAsync(aux.u() + 15, 0, 8, st);
                rc = launch_walk(p->d_L, K, p->N, listed ? ovfl.p : cur.p, listed ? h[15] : ncur, nxt.p, next_cnt,
                                 table.p, cap, counter, stats, grid, st, limV, limL, lvol, &fused,
                                 (uint8_t *)tags.p, tag, ncap, 0, nullptr, nullptr, 0);
                if (rc) return fail(p, BDEG_E_CUDA, std::string("k_walk: ") + cudaGetErrorString((cudaError_t)rc));
                narrow_redo += listed ? h[15] : ncur;
                cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
                ce = cudaStreamSynchronize(st);
                if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
            }
            if (h[2 + 3] == 0) break;
            // full: keep the cells already inserted (tagged), grow, redo the level
            if (attempt > 4) return fail(p, BDEG_E_TOO_LARGE, "cell walk: hash set overflow");
            if (fused && L >= 2 && oldest < L - 1) {     // drop levels < L-1 (and grow if it helps)
                const uint64_t keep = window + h[0];
                const uint64_t lim = mem_cap(0);
                uint64_t want = std::min(std::max(cap, round_up(3 * keep)), lim);
                bdeg_status s = grow_table(want, L - 1);
                if (s) return s;
                live = keep;
            } else {
                const uint64_t want = std::min(cap * 2, std::max(cap, mem_cap(0)));
                if (want <= cap) return fail(p, BDEG_E_TOO_LARGE, "cell walk: hash set full at the device memory limit");
                bdeg_status s = grow_table(want);
                if (s) return s;
            }
            cudaMemsetAsync(counter, 0, 15 * 8, st);   // work counter, stats, level volumes
        }
        const uint64_t *sv = h + 2;
        ridges += sv[0];
        boundary += sv[5];
        wide_cells += sv[6];
        if (sv[1] > 0) return fail(p, BDEG_E_DEGENERATE, "degenerate lifting: a ridge has a tie (cell walk)");
        if (sv[2] > 0 || sv[4] > 0)
            return fail(p, BDEG_E_TOO_LARGE, "cell walk: inconsistent ridge or value overflow (level " +
                                                 std::to_string(levels) + ": " + std::to_string(sv[2]) +
                                                 " inconsistent, " + std::to_string(sv[4]) + " overflow)");
        const uint64_t nnext = h[0];
        if (nnext > ncap) {
            // frontier overflow: the level's cells are all in the table with
            // this tag; collect them into a buffer of the right size
            ncap = round_up(nnext);
            if (!nxt.alloc(ncap * 16)) return fail(p, BDEG_E_TOO_LARGE, "cudaMalloc (frontier) failed");
            cudaMemsetAsync(next_cnt, 0, 8, st);
            int rc = launch_collect(table.p, (const uint8_t *)tags.p, cap, (uint8_t)tag, nxt.p, next_cnt, st);
            if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
            uint64_t got = 0;
            cudaMemcpyAsync(&got, next_cnt, 8, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            // levels more than 255 apart share a tag: only cells of this level
            // can carry it while fewer than 256 levels exist
            if (got != nnext && levels - oldest < 255)
                return fail(p, BDEG_E_TOO_LARGE, "cell walk: frontier re-collection mismatch");
            if (got != nnext) return fail(p, BDEG_E_TOO_LARGE, "cell walk: > 255 levels with frontier overflow");
            ++collects;
        }
        if (dbg && std::getenv("BDEG_DEBUG_LEVELS"))
            fprintf(stderr, "  level %d: cells %llu -> %llu, %.2f ms (cap %llu, next cap %llu)\n", levels,
                    (unsigned long long)ncur, (unsigned long long)nnext, now_ms() - t_level,
                    (unsigned long long)cap, (unsigned long long)ncap);
        for (int i = 3; i >= 0; --i) fused_vol += (u128)h[10 + i] << (32 * i);
        fused_cells += h[14];
        // growth estimate for the next level: the ratio just seen, with slack
        growth = std::min<double>(K, 1.1 * (double)nnext / (double)ncur + 0.1);
        if (tight) growth = 0;                     // test knob: every growing level overflows
        std::swap(cur.p, nxt.p);
        std::swap(ccap, ncap);
        ncur = nnext;
        total_cells += ncur;
        live += ncur;
        lsz.push_back(ncur);
        ++levels;
    }
    if (dbg)
        fprintf(stderr, "[bdeg walk] start cell %.2f ms, %d levels, walk %.2f ms, cells %llu, cap %llu, "
                "int128 redo %llu, tier %d, frontier re-collections %llu, window evictions %llu, narrow %d "
                "(int64 redo %llu)\n", t_start - t0,
                levels, now_ms() - t_start, (unsigned long long)total_cells, (unsigned long long)cap,
                (unsigned long long)wide_cells, p->tier, (unsigned long long)collects,
                (unsigned long long)evictions, narrow, (unsigned long long)narrow_redo);
    if (fused) {   // the D&C walk summed |det| as it went
        r->deg_lo = (uint64_t)fused_vol;
        r->deg_hi = (int64_t)(uint64_t)(fused_vol >> 64);
        r->cells = fused_cells;
        r->candidates = 0;
        r->singular = 0;
        r->singular_complete = 0;
        r->leaves = ridges;
        r->dead_leaves = boundary;
        if (r->cells != total_cells) return fail(p, BDEG_E_TOO_LARGE, "cell walk: table / frontier mismatch");
        *kms += now_ms() - t0;
        return BDEG_OK;
    }
    // exact volumes, one determinant per cell
    cudaMemsetAsync(aux.p, 0, 16 * 8, st);
    int rc = launch_cellvol(p->d_L, K, p->N, table.p, cap, aux.u() + 8, aux.u(), grid, st, limV, limL);
    if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
    uint64_t h[16];
    cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    if (h[8 + 5] > 0) return fail(p, BDEG_E_TOO_LARGE, "cell volume overflow");
    u128 vol = 0;
    for (int i = 3; i >= 0; --i) vol = (vol << 32) + (u128)h[8 + i];
    r->deg_lo = (uint64_t)vol;
    r->deg_hi = (int64_t)(uint64_t)(vol >> 64);
    r->cells = h[8 + 4];
    r->candidates = 0;
    r->singular = 0;
    r->singular_complete = 0;
    r->leaves = ridges;          // ridge tests (pivots)
    r->dead_leaves = boundary;   // boundary ridges
    if (r->cells != total_cells) return fail(p, BDEG_E_TOO_LARGE, "cell walk: table / frontier mismatch");
    *kms += now_ms() - t0;
    return BDEG_OK;
}

// SURVEY §8.f3 sharded walk: the hash set split over the ranks by owner =
// hash(cell) mod world; one all-to-all of the neighbours owned elsewhere per
// level (chunked so the outgoing buffer stays bounded), per-level collective
// decisions (termination, ties, overflow) through one small all-reduce, and
// the volumes summed by the owners.  Same kernels as walk_once.
bdeg_status walk_sharded(bdeg_plan_s *p, const bdeg_comm *cm, bdeg_result *r, double *kms) {
    Nvtx range("bdeg sharded walk");
    cudaStream_t st = (cudaStream_t)p->opt.stream;
    const double t0 = now_ms();
    const int W = std::max(1, p->opt.world), R = p->opt.rank;
    const int K = p->K;
    auto comm_fail = [&](const char *what) { return fail(p, BDEG_E_COMM, std::string("sharded walk: ") + what); };
    auto allreduce = [&](int64_t *v, int n) -> bool { return cm->allreduce_sum(cm->ctx, v, n) == 0; };
    // ---- start cell: rank 0's, broadcast by a sum where the others give 0
    int64_t sv[4] = {0, 0, 0, 0};
    if (R == 0) {
        if (p->big) {
            if (p->user_lift || (p->basis_lo == 0 && p->basis_hi == 0)) sv[3] = BDEG_E_INVALID;
            else { sv[0] = (int64_t)p->basis_lo; sv[1] = (int64_t)p->basis_hi; sv[2] = 1; }
        } else {
            uint64_t pair[2 * 64];
            uint64_t n = 0;
            bdeg_status s = cells_range(p, 0, p->total, pair, 64, &n, true);
            if (s) sv[3] = s;
            else if (n > 0) { sv[0] = (int64_t)pair[0]; sv[2] = 1; }
        }
    }
    if (!allreduce(sv, 4)) return comm_fail("allreduce failed");
    if (sv[3] == BDEG_E_INVALID) return fail(p, BDEG_E_INVALID, "N > 64 needs a generated lifting (basis-seeded start cell)");
    if (sv[3] != 0) return fail(p, (bdeg_status)sv[3], "start-cell search failed on rank 0");
    if (sv[2] == 0) return fail(p, BDEG_E_DEGENERATE, "no cell found (degenerate lifting)");
    const uint64_t start[2] = {(uint64_t)sv[0], (uint64_t)sv[1]};
    // ---- buffers
    uint64_t cap = 1ull << 22;
    if (const char *c0 = std::getenv("BDEG_WALK_CAP0")) cap = std::max<uint64_t>(1024, std::strtoull(c0, nullptr, 10));
    else {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cap = std::max<uint64_t>(cap, (uint64_t)((fr * 0.4) / 17) & ~1023ull);
    }
    const uint64_t chunk_max = std::max<uint64_t>(1024, (1ull << 30) / (16ull * (uint64_t)K));   // <= 1 GB outgoing
    DevBuf table, tags, cur, nxt, aux, remote, sendb, recvb, ovfl, ocnt;
    uint64_t ccap = 1 << 16, ncap = 1 << 16, rcap = 0, scap = 0, vcap = 0, ovfl_cap = 0;
    if (!table.alloc(cap * 16) || !tags.alloc(cap) || !cur.alloc(ccap * 16) || !nxt.alloc(ncap * 16) ||
        !aux.alloc(16 * 8) || !ocnt.alloc(2 * 8 * (size_t)W))
        return fail(p, BDEG_E_TOO_LARGE, "sharded walk: cudaMalloc of the hash set failed");
    unsigned long long *next_cnt = aux.u(), *counter = aux.u() + 1, *stats = aux.u() + 2, *lvol = aux.u() + 10;
    cudaMemsetAsync(table.p, 0, cap * 16, st);
    cudaMemsetAsync(tags.p, 0, cap, st);
    uint64_t ncur = 0;
    if (walk_owner(start[0], start[1], W) == R) {
        const uint64_t h0 = (uint64_t)(((u128)walk_hash(start[0], start[1]) * cap) >> 64);
        cudaMemcpyAsync((char *)table.p + h0 * 16, start, 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(cur.p, start, 16, cudaMemcpyHostToDevice, st);
        ncur = 1;
    }
    cudaStreamSynchronize(st);
    const int grid = std::max(1, dev_info(p->opt.device).sms) * 4;
    const int64_t limV = p->tier == 2 ? 0 : (int64_t)1 << (p->tier == 0 ? 30 : p->bits_v);
    const int64_t limL = p->tier == 2 ? 0 : (int64_t)1 << (p->tier == 0 ? 31 : p->bits_l);
    const int narrow = (p->tier == 0 && !std::getenv("BDEG_WALK_WIDE")) ? 1 : 0;
    u128 vol = 0;
    uint64_t cells = 0, ridges = 0, boundary = 0, sent_total = 0, evictions = 0;
    int fused = 1, levels = 0;
    uint64_t live = ncur, prev_level = 0;   // cells in this rank's table; cells of level L-1 (kept in `nxt`)
    std::vector<uint64_t> scnt(W), rcnt(W);
    std::vector<int64_t> red(8 + W);
    for (;;) {
        const unsigned tag = (unsigned)(levels + 1) & 255u;
        // chunks of this level: the same count on every rank (max)
        std::fill(red.begin(), red.end(), 0);
        red[8 + R] = (int64_t)((ncur + chunk_max - 1) / chunk_max);
        if (!allreduce(red.data(), 8 + W)) return comm_fail("allreduce failed");
        int64_t nch = 0;
        for (int i = 0; i < W; ++i) nch = std::max(nch, red[8 + i]);
        uint64_t nnext = 0;
        int64_t flags[6] = {0, 0, 0, 0, 0, 0};   // ties, inconsistent/overflow, table full, comm, next total, -
        for (int64_t c = 0; c < nch; ++c) {
            const uint64_t b = std::min<uint64_t>(ncur, (uint64_t)c * chunk_max);
            const uint64_t e = std::min<uint64_t>(ncur, b + chunk_max);
            const uint64_t nc = e - b;
            // room for this chunk's local neighbours (<= K per cell) in the next frontier
            if (nnext + nc * (uint64_t)K > ncap) {
                const uint64_t want = (nnext + nc * (uint64_t)K + 1023) & ~1023ull;
                DevBuf t;
                if (!t.alloc(want * 16)) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: frontier allocation failed");
                if (nnext) cudaMemcpyAsync(t.p, nxt.p, nnext * 16, cudaMemcpyDeviceToDevice, st);
                cudaStreamSynchronize(st);
                std::swap(t.p, nxt.p);
                ncap = want;
            }
            // <= K neighbours per cell, twice for cells redone in int64 after the narrow kernel
            if (2 * nc * (uint64_t)K > rcap) {
                rcap = (2 * nc * (uint64_t)K + 1023) & ~1023ull;
                if (!remote.alloc(rcap * 16) || !sendb.alloc(rcap * 16))
                    return fail(p, BDEG_E_TOO_LARGE, "sharded walk: exchange buffer allocation failed");
            }
            if (narrow && nc > ovfl_cap) {
                ovfl_cap = std::max<uint64_t>(1024, nc);
                if (!ovfl.alloc(ovfl_cap * 16)) return fail(p, BDEG_E_CUDA, "cudaMalloc (walk overflow list) failed");
            }
            uint64_t nn = nnext;
            cudaMemsetAsync(aux.p, 0, 16 * 8, st);
            cudaMemcpyAsync(next_cnt, &nn, 8, cudaMemcpyHostToDevice, st);
            cudaMemsetAsync(ocnt.p, 0, 2 * 8 * (size_t)W, st);
            unsigned long long *rcnt_d = ocnt.u() + 2 * W - 1;   // remote count lives in the spare slot
            cudaMemsetAsync(rcnt_d, 0, 8, st);
            uint64_t h[16] = {0};
            if (nc > 0) {
                int rc = launch_walk(p->d_L, K, p->N, (const char *)cur.p + b * 16, nc, nxt.p, next_cnt, table.p, cap,
                                     counter, stats, grid, st, limV, limL, lvol, &fused, (uint8_t *)tags.p, tag, ncap,
                                     narrow, ovfl.p, aux.u() + 15, ovfl_cap, p->v_safe ? 1 : 0, W, R, remote.p,
                                     rcnt_d, rcap);
                if (rc) return fail(p, BDEG_E_CUDA, std::string("k_walk: ") + cudaGetErrorString((cudaError_t)rc));
                cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
                if (cudaStreamSynchronize(st) != cudaSuccess) return fail(p, BDEG_E_CUDA, "walk level failed");
                if (narrow && h[15] > 0) {   // cells whose values left int32: redo them with int64 storage
                    cudaMemsetAsync(counter, 0, 8, st);
                    cudaMemsetAsync(aux.u() + 15, 0, 8, st);
                    rc = launch_walk(p->d_L, K, p->N, ovfl.p, h[15], nxt.p, next_cnt, table.p, cap, counter, stats,
                                     grid, st, limV, limL, lvol, &fused, (uint8_t *)tags.p, tag, ncap, 0, nullptr,
                                     nullptr, 0, 0, W, R, remote.p, rcnt_d, rcap);
                    if (rc) return fail(p, BDEG_E_CUDA, std::string("k_walk: ") + cudaGetErrorString((cudaError_t)rc));
                    cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
                    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(p, BDEG_E_CUDA, "walk level failed");
                }
            }
            const uint64_t *sv2 = h + 2;
            ridges += sv2[0];
            boundary += sv2[5];
            flags[0] += (int64_t)sv2[1];
            flags[1] += (int64_t)(sv2[2] + sv2[4]);
            flags[2] += (int64_t)sv2[3];
            if (fused) {
                for (int i = 3; i >= 0; --i) vol += (u128)h[10 + i] << (32 * i);
                cells += h[14];
            }
            nnext = h[0];
            // ---- route the neighbours owned by other ranks
            uint64_t nrem = 0;
            cudaMemcpy(&nrem, rcnt_d, 8, cudaMemcpyDeviceToHost);
            if (nrem > rcap) flags[2] += 1;             // cannot happen (<= K per cell); reported as full
            nrem = std::min(nrem, rcap);
            unsigned long long *cnt_d = ocnt.u();
            cudaMemsetAsync(cnt_d, 0, 8 * (size_t)W, st);
            launch_owner_count(remote.p, nrem, W, cnt_d, st);
            std::vector<unsigned long long> hc(W);
            cudaMemcpyAsync(hc.data(), cnt_d, 8 * (size_t)W, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            std::vector<unsigned long long> off(W, 0);
            for (int i = 1; i < W; ++i) off[i] = off[i - 1] + hc[i - 1];
            cudaMemcpyAsync(cnt_d, off.data(), 8 * (size_t)W, cudaMemcpyHostToDevice, st);
            launch_owner_scatter(remote.p, nrem, W, cnt_d, sendb.p, st);
            if (cudaStreamSynchronize(st) != cudaSuccess) return fail(p, BDEG_E_CUDA, "owner partition failed");
            for (int i = 0; i < W; ++i) scnt[i] = hc[i];
            sent_total += nrem;
            if (cm->alltoall_counts(cm->ctx, scnt.data(), rcnt.data()) != 0) return comm_fail("alltoall (counts) failed");
            uint64_t nrecv = 0;
            for (int i = 0; i < W; ++i) nrecv += rcnt[i];
            if (nrecv > vcap) {
                vcap = (nrecv + 1023) & ~1023ull;
                if (!recvb.alloc(vcap * 16)) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: receive buffer allocation failed");
            }
            if (cm->alltoall_cells(cm->ctx, sendb.p, scnt.data(), recvb.p, rcnt.data()) != 0)
                return comm_fail("alltoall (cells) failed");
            if (nnext + nrecv > ncap) {
                const uint64_t want = (nnext + nrecv + 1023) & ~1023ull;
                DevBuf t;
                if (!t.alloc(want * 16)) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: frontier allocation failed");
                if (nnext) cudaMemcpyAsync(t.p, nxt.p, nnext * 16, cudaMemcpyDeviceToDevice, st);
                cudaStreamSynchronize(st);
                std::swap(t.p, nxt.p);
                ncap = want;
            }
            if (nrecv > 0) {
                cudaMemsetAsync(stats + 3, 0, 8, st);
                int rc = launch_insert_recv(recvb.p, nrecv, table.p, (uint8_t *)tags.p, cap, (uint8_t)tag, nxt.p,
                                            next_cnt, ncap, stats + 3, st);
                if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
                uint64_t fullc = 0;
                cudaMemcpyAsync(&nnext, next_cnt, 8, cudaMemcpyDeviceToHost, st);
                cudaMemcpyAsync(&fullc, stats + 3, 8, cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                flags[2] += (int64_t)fullc;
            }
        }
        // ---- collective decisions for the level
        std::fill(red.begin(), red.end(), 0);
        red[0] = flags[0];
        red[1] = flags[1];
        red[2] = flags[2];
        red[3] = (int64_t)nnext;
        red[4] = fused ? 0 : 1;
        if (!allreduce(red.data(), 8 + W)) return comm_fail("allreduce failed");
        if (red[0] > 0) return fail(p, BDEG_E_DEGENERATE, "degenerate lifting: a ridge has a tie (sharded walk)");
        if (red[1] > 0) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: inconsistent ridge or value overflow");
        if (red[2] > 0) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: hash set shard full");
        const bool any_unfused = red[4] > 0;
        std::swap(cur.p, nxt.p);
        std::swap(ccap, ncap);
        prev_level = ncur;
        ncur = nnext;
        live += nnext;
        ++levels;
        if (red[3] == 0) break;                       // no rank has a next frontier
        // BFS window: rebuild this rank's shard from levels L-1 (nxt) and L (cur)
        // when it passes half load (fused walk only: the volumes are already summed)
        if (!any_unfused && live * 2 > cap) {
            cudaMemsetAsync(table.p, 0, cap * 16, st);
            cudaMemsetAsync(tags.p, 0, cap, st);
            cudaMemsetAsync(stats + 3, 0, 8, st);
            int rc = launch_insert_list(nxt.p, prev_level, table.p, (uint8_t *)tags.p, cap,
                                        (uint8_t)((levels - 1) & 255), stats + 3, st);
            if (!rc) rc = launch_insert_list(cur.p, ncur, table.p, (uint8_t *)tags.p, cap, (uint8_t)(levels & 255),
                                             stats + 3, st);
            if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
            cudaStreamSynchronize(st);
            live = prev_level + ncur;
            ++evictions;
            if (live * 4 > cap * 3) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: two levels exceed the hash set shard");
        }
        if (levels > 100000) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: too many levels");
    }
    if (!fused) {   // exact volumes of this rank's cells (every owned cell is still in the table)
        if (evictions) return fail(p, BDEG_E_TOO_LARGE, "sharded walk: unfused walk needs the whole shard");
        cudaMemsetAsync(aux.p, 0, 16 * 8, st);
        int rc = launch_cellvol(p->d_L, K, p->N, table.p, cap, aux.u() + 8, aux.u(), grid, st, limV, limL);
        if (rc) return fail(p, BDEG_E_CUDA, cudaGetErrorString((cudaError_t)rc));
        uint64_t h[16];
        cudaMemcpyAsync(h, aux.p, 16 * 8, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return fail(p, BDEG_E_CUDA, "cell volume pass failed");
        if (h[8 + 5] > 0) return fail(p, BDEG_E_TOO_LARGE, "cell volume overflow");
        vol = 0;
        for (int i = 3; i >= 0; --i) vol = (vol << 32) + (u128)h[8 + i];
        cells = h[8 + 4];
    }
    // ---- combine: the volume as four 32-bit limbs (exact in int64 sums)
    int64_t tot[8] = {(int64_t)(uint64_t)(vol & 0xFFFFFFFFu), (int64_t)(uint64_t)((vol >> 32) & 0xFFFFFFFFu),
                      (int64_t)(uint64_t)((vol >> 64) & 0xFFFFFFFFu), (int64_t)(uint64_t)(vol >> 96),
                      (int64_t)cells, (int64_t)ridges, (int64_t)boundary, (int64_t)sent_total};
    if (!allreduce(tot, 8)) return comm_fail("allreduce failed");
    u128 v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 32) + (u128)(uint64_t)tot[i];
    r->deg_lo = (uint64_t)v;
    r->deg_hi = (int64_t)(uint64_t)(v >> 64);
    r->cells = (uint64_t)tot[4];
    r->candidates = 0;
    r->singular = 0;
    r->singular_complete = 0;
    r->leaves = (uint64_t)tot[5];
    r->dead_leaves = (uint64_t)tot[6];
    if (std::getenv("BDEG_DEBUG"))
        fprintf(stderr, "[bdeg sharded walk] rank %d/%d: %d levels, %llu owned cells, %llu sent, %llu evictions, "
                "%.2f ms\n", R, W, levels, (unsigned long long)cells, (unsigned long long)sent_total,
                (unsigned long long)evictions, now_ms() - t0);
    *kms += now_ms() - t0;
    return BDEG_OK;
}

}  // namespace

extern "C" {

void bdeg_default_options(bdeg_options *o) {
    std::memset(o, 0, sizeof(*o));
    o->seed = 1;
    o->lift_bits = 20;
    o->max_relift = 32;
    o->device = 0;
    o->rank = 0;
    o->world = 1;
    o->stream = nullptr;
    o->flags = 0;
    o->inner_levels = -1;
    o->ctas_per_sm = 0;
}

bdeg_status bdeg_plan(const bdeg_problem *prob, const bdeg_options *opt, bdeg_plan_t *out) {
    Nvtx range("bdeg plan (front end + planner)");
    if (!prob || !out) return fail(nullptr, BDEG_E_INVALID, "NULL argument");
    if (prob->n < 1 || prob->m < 0 || (prob->m > 0 && !prob->A))
        return fail(nullptr, BDEG_E_INVALID, "bad problem shape");
    const double t0 = now_ms();
    bdeg_plan_s *p = new bdeg_plan_s();
    if (opt) p->opt = *opt; else bdeg_default_options(&p->opt);
    if (p->opt.world < 1) p->opt.world = 1;
    fill_binom(p->binom);
    p->n = prob->n;
    p->m = prob->m;
    p->A.assign(prob->A, prob->A + (size_t)prob->n * prob->m);
    if (prob->b_re) p->bre.assign(prob->b_re, prob->b_re + prob->m);
    if (prob->b_im) p->bim.assign(prob->b_im, prob->b_im + prob->m);
    p->seed_used = p->opt.seed;
    if (prob->lifting) {
        p->user_lift = true;
        p->lift.assign(prob->lifting, prob->lifting + prob->n + 1);
    } else {
        gen_lifting(p->opt.seed, prob->n + 1, p->opt.lift_bits, p->lift);
    }
    std::string err;
    if (!analyze_system(p->n, p->m, p->A.data(), p->bre.empty() ? nullptr : p->bre.data(),
                        p->bim.empty() ? nullptr : p->bim.data(), !(p->opt.flags & BDEG_FLAG_NO_LLL), p->fe, err)) {
        delete p;
        return fail(nullptr, BDEG_E_TOO_LARGE, err);
    }
    if (!p->fe.consistent) {
        delete p;
        return fail(nullptr, BDEG_E_INCONSISTENT, "inconsistent system: b^{Q_0} != 1 (PAPER.md P:366-367)");
    }
    if (p->fe.dim == 0) {
        p->K = 0;
        p->N = 0;
        p->total = 0;
    } else {
        rebuild_points(p);
        bdeg_status s = finish_plan(p);
        if (s) {
            g_err = p->err;
            delete p;
            return s;
        }
    }
    p->plan_ms = now_ms() - t0;
    *out = p;
    return BDEG_OK;
}

bdeg_status bdeg_plan_points(int32_t K, int32_t N, const int64_t *V, const int64_t *lifting,
                             const bdeg_options *opt, bdeg_plan_t *out) {
    Nvtx range("bdeg plan (points)");
    if (!V || !out || K < 1 || N < K) return fail(nullptr, BDEG_E_INVALID, "bad point configuration");
    const double t0 = now_ms();
    bdeg_plan_s *p = new bdeg_plan_s();
    if (opt) p->opt = *opt; else bdeg_default_options(&p->opt);
    if (p->opt.world < 1) p->opt.world = 1;
    fill_binom(p->binom);
    p->points_mode = true;
    p->K = K;
    p->N = N;
    p->V.assign(V, V + (size_t)K * N);
    p->seed_used = p->opt.seed;
    if (lifting) {
        p->user_lift = true;
        p->lift.assign(lifting, lifting + N);
    } else {
        gen_lifting(p->opt.seed, N, p->opt.lift_bits, p->lift);
    }
    p->w = p->lift;
    bdeg_status s = finish_plan(p);
    if (s) {
        g_err = p->err;
        delete p;
        return s;
    }
    p->plan_ms = now_ms() - t0;
    *out = p;
    return BDEG_OK;
}

bdeg_status bdeg_plan_info(bdeg_plan_t p, bdeg_result *out) {
    if (!p || !out) return fail(p, BDEG_E_INVALID, "NULL argument");
    fill_front(p, out);
    return BDEG_OK;
}

bdeg_status bdeg_plan_points_get(bdeg_plan_t p, int64_t *V, int64_t *omega) {
    if (!p) return fail(p, BDEG_E_INVALID, "NULL plan");
    if (p->K == 0) return fail(p, BDEG_E_INVALID, "d = 0: the plan has no point configuration");
    if (V) std::memcpy(V, p->V.data(), p->V.size() * sizeof(int64_t));
    if (omega) std::memcpy(omega, p->w.data(), p->w.size() * sizeof(int64_t));
    return BDEG_OK;
}

size_t bdeg_workspace_bytes(bdeg_plan_t p) { return p && p->K > 0 ? layout(p).total : 0; }

bdeg_status bdeg_set_workspace(bdeg_plan_t p, void *d_ptr, size_t bytes) {
    if (!p || !d_ptr) return fail(p, BDEG_E_INVALID, "NULL argument");
    if (p->dev_ready) return fail(p, BDEG_E_INVALID, "workspace already in use");
    if (bytes < layout(p).total) return fail(p, BDEG_E_INVALID, "workspace too small");
    if (((uintptr_t)d_ptr & 255) != 0) return fail(p, BDEG_E_INVALID, "workspace must be 256-byte aligned");
    p->ws = (char *)d_ptr;
    p->ws_bytes = bytes;
    p->own_ws = false;
    return BDEG_OK;
}

bdeg_status bdeg_relift(bdeg_plan_t p, int32_t attempt) {
    if (!p) return fail(p, BDEG_E_INVALID, "NULL plan");
    if (p->user_lift) return fail(p, BDEG_E_INVALID, "the lifting was given by the caller");
    p->seed_used = derive_seed(p->opt.seed, attempt);
    const int count = p->points_mode ? p->N : p->n + 1;
    gen_lifting(p->seed_used, count, p->opt.lift_bits, p->lift);
    if (p->points_mode) p->w = p->lift;
    else rebuild_points(p);
    seed_basis_lifting(p);
    raw_tier_bounds(p);
    p->relifts = attempt;
    p->l_dirty = true;
    return BDEG_OK;
}

bdeg_status bdeg_degree(bdeg_plan_t p, bdeg_result *out) {
    if (!p || !out) return fail(p, BDEG_E_INVALID, "NULL argument");
    if (p->big) return fail(p, BDEG_E_TOO_LARGE, "N > 64: rank-space enumeration unavailable, use bdeg_degree_walk");
    const double t0 = now_ms();
    bdeg_result r;
    fill_front(p, &r);
    if (p->K == 0) {                      // d = 0: isolated points
        r.deg_lo = 1;
        r.total_ms = now_ms() - t0;
        *out = r;
        return BDEG_OK;
    }
    double kms = 0;
    for (int attempt = p->relifts;; ++attempt) {
        int64_t h[kNSlots];
        bdeg_status s = run_sync(p, 0, p->total, h, &kms);
        if (s) return s;
        fill_front(p, &r);
        s = slots_to_result(p, h, &r);
        if (s) return s;
        if (r.ties == 0) break;
        if (p->user_lift || (p->opt.flags & BDEG_FLAG_NO_RELIFT))
            return fail(p, BDEG_E_DEGENERATE, "degenerate lifting: a would-be cell has a zero facet value");
        if (attempt + 1 > p->opt.max_relift)
            return fail(p, BDEG_E_DEGENERATE, "no generic lifting found within max_relift attempts");
        bdeg_relift(p, attempt + 1);
    }
    r.kernel_ms = kms;
    r.total_ms = now_ms() - t0;
    *out = r;
    return BDEG_OK;
}

bdeg_status bdeg_degree_range(bdeg_plan_t p, uint64_t begin, uint64_t end, bdeg_result *out) {
    if (!p || !out) return fail(p, BDEG_E_INVALID, "NULL argument");
    if (p->big) return fail(p, BDEG_E_TOO_LARGE, "N > 64: rank-space enumeration unavailable, use bdeg_degree_walk");
    const double t0 = now_ms();
    bdeg_result r;
    fill_front(p, &r);
    if (p->K == 0) {
        *out = r;
        return BDEG_OK;
    }
    double kms = 0;
    int64_t h[kNSlots];
    bdeg_status s = run_sync(p, begin, end, h, &kms);
    if (s) return s;
    s = slots_to_result(p, h, &r);
    if (s) return s;
    r.kernel_ms = kms;
    r.total_ms = now_ms() - t0;
    *out = r;
    return BDEG_OK;
}

bdeg_status bdeg_degree_partial(bdeg_plan_t p, int64_t *d_slots) {
    if (!p || !d_slots) return fail(p, BDEG_E_INVALID, "NULL argument");
    if (p->big) return fail(p, BDEG_E_TOO_LARGE, "N > 64: rank-space enumeration unavailable, use bdeg_degree_walk");
    if (p->K == 0) {
        cudaError_t ce = cudaMemsetAsync(d_slots, 0, kNSlots * 8, (cudaStream_t)p->opt.stream);
        return ce == cudaSuccess ? BDEG_OK : fail(p, BDEG_E_CUDA, cudaGetErrorString(ce));
    }
    bdeg_status s = ensure_device(p);
    if (s) return s;
    return enqueue_range(p, 0, p->total, reinterpret_cast<unsigned long long *>(d_slots), p->opt.rank,
                         p->opt.world, -1);
}

bdeg_status bdeg_finalize(bdeg_plan_t p, const int64_t *h_slots, bdeg_result *out) {
    Nvtx range("bdeg finalize");
    if (!p || !h_slots || !out) return fail(p, BDEG_E_INVALID, "NULL argument");
    bdeg_result r;
    fill_front(p, &r);
    if (p->K == 0) {
        r.deg_lo = 1;
        *out = r;
        return BDEG_OK;
    }
    // more than 2^27 work items and an overflow beyond the re-run bitmap
    if (h_slots[SLOT_QFULL] > 0)
        return fail(p, BDEG_E_TOO_LARGE, "overflow re-run bitmap exhausted (> 2^27 work items); rerun with "
                                         "BDEG_FLAG_FORCE_TIER2");
    bdeg_status s = slots_to_result(p, h_slots, &r);
    if (s) return s;
    // a would-be cell with a zero facet value on any rank: the lifting is not
    // generic, the summed volume is not a degree.  Every rank must
    // re-lift with the same attempt (bdeg_relift) and recompute (multi.py).
    if (r.ties > 0)
        return fail(p, BDEG_E_DEGENERATE,
                    p->user_lift ? "degenerate user lifting: a would-be cell has a zero facet value"
                                 : "degenerate generated lifting: call bdeg_relift(attempt+1) on every rank and recompute");
    *out = r;
    return BDEG_OK;
}

uint64_t bdeg_num_items(bdeg_plan_t p) { return (p && p->K > 0) ? p->q->nitems : 0; }

bdeg_status bdeg_item_range(bdeg_plan_t p, uint64_t item, uint64_t *begin, uint64_t *end) {
    if (!p || !begin || !end) return fail(p, BDEG_E_INVALID, "NULL argument");
    if (p->K == 0 || p->big || item >= p->q->nitems) return fail(p, BDEG_E_INVALID, "item out of range");
    int d = 0;
    std::vector<int> top;
    decode_position(p, item, d, top);
    const int kd = p->K - d;
    uint64_t base = 0;
    for (int t = 0; t < d; ++t) base += C(p->binom, top[t], kd + t + 1);
    *begin = base;
    *end = base + C(p->binom, d > 0 ? top[0] : p->N, kd);
    return BDEG_OK;
}

bdeg_status bdeg_queue_info(bdeg_plan_t p, uint64_t *n_items, uint64_t *n_split, uint64_t *n_static,
                            uint64_t *grab) {
    if (!p) return fail(p, BDEG_E_INVALID, "NULL plan");
    const bool k = p->K > 0 && !p->big;
    if (n_items) *n_items = k ? p->q->nitems : 0;
    if (n_split) *n_split = k ? p->q->split.size() : 0;
    if (n_static) *n_static = k ? p->q->nstatic_steal : 0;
    if (grab) *grab = k ? p->q->grab : 0;
    return BDEG_OK;
}

bdeg_status bdeg_cells(bdeg_plan_t p, uint64_t begin, uint64_t end, uint64_t *h_out, uint64_t capacity,
                       uint64_t *count) {
    if (!p || !count) return fail(p, BDEG_E_INVALID, "NULL argument");
    *count = 0;
    if (p->big) return fail(p, BDEG_E_TOO_LARGE, "N > 64: rank-space enumeration unavailable");
    if (p->K == 0) return BDEG_OK;
    return cells_range(p, begin, end, h_out, capacity, count);
}

bdeg_status bdeg_cell_normal(bdeg_plan_t p, uint64_t mask_lo, uint64_t mask_hi, int64_t *h_num, int64_t *den) {
    if (!p || !h_num || !den) return fail(p, BDEG_E_INVALID, "NULL argument");
    const int K = p->K;
    std::vector<int> idx;
    for (int l = 0; l < p->N; ++l)
        if (l < 64 ? ((mask_lo >> l) & 1ull) : ((mask_hi >> (l - 64)) & 1ull)) idx.push_back(l);
    if ((int)idx.size() != K) return fail(p, BDEG_E_INVALID, "mask does not hold K points");
    // solve V_sigma h = w_sigma (rows v_c) fraction-free: h = h~ / D, D = det V_sigma
    // (Cramer's rule by Bareiss on the augmented matrix, exact in checked __int128)
    std::vector<std::vector<i128>> M(K, std::vector<i128>(K + 1));
    for (int r = 0; r < K; ++r) {
        for (int t = 0; t < K; ++t) M[r][t] = p->V[(size_t)idx[r] * K + t];
        M[r][K] = p->w[idx[r]];
    }
    i128 prev = 1;
    int sign = 1;
    for (int k = 0; k < K; ++k) {
        int piv = -1;
        for (int r = k; r < K; ++r) if (M[r][k] != 0) { piv = r; break; }
        if (piv < 0) return fail(p, BDEG_E_INVALID, "singular cell");
        if (piv != k) { std::swap(M[piv], M[k]); sign = -sign; }
        for (int r = 0; r < K; ++r) {
            if (r == k) continue;
            for (int t = 0; t <= K; ++t) {
                if (t == k) continue;
                i128 a, b;
                if (__builtin_mul_overflow(M[k][k], M[r][t], &a) || __builtin_mul_overflow(M[r][k], M[k][t], &b))
                    return fail(p, BDEG_E_TOO_LARGE, "normal overflow");
                M[r][t] = (a - b) / prev;       // exact (Gauss-Jordan Bareiss)
            }
            M[r][k] = 0;
        }
        prev = M[k][k];
    }
    // now M = diag(D,...,D | h~) with D = det (up to the row-swap sign)
    const i128 D = M[K - 1][K - 1];
    for (int t = 0; t < K; ++t) {
        const i128 v = M[t][K];
        if (v > INT64_MAX || v < INT64_MIN) return fail(p, BDEG_E_TOO_LARGE, "normal beyond int64");
        h_num[t] = (int64_t)v;
    }
    if (D > INT64_MAX || D < INT64_MIN) return fail(p, BDEG_E_TOO_LARGE, "determinant beyond int64");
    *den = (int64_t)D;
    (void)sign;
    return BDEG_OK;
}

bdeg_status bdeg_degree_walk(bdeg_plan_t p, bdeg_result *out) {
    if (!p || !out) return fail(p, BDEG_E_INVALID, "NULL argument");
    const double t0 = now_ms();
    bdeg_result r;
    fill_front(p, &r);
    if (p->K == 0) {
        r.deg_lo = 1;
        *out = r;
        return BDEG_OK;
    }
    bdeg_status s = ensure_device(p);
    if (s) return s;
    double kms = 0;
    for (int attempt = p->relifts;; ++attempt) {
        fill_front(p, &r);
        s = walk_once(p, &r, &kms);
        if (s != BDEG_E_DEGENERATE) break;
        if (p->user_lift || (p->opt.flags & BDEG_FLAG_NO_RELIFT)) return s;
        if (attempt + 1 > p->opt.max_relift) return s;
        bdeg_relift(p, attempt + 1);
        s = ensure_device(p);
        if (s) return s;
    }
    if (s) return s;
    r.relifts = p->relifts;
    r.seed_used = p->seed_used;
    r.kernel_ms = kms;
    r.total_ms = now_ms() - t0;
    *out = r;
    return BDEG_OK;
}

bdeg_status bdeg_degree_walk_sharded(bdeg_plan_t p, const bdeg_comm *comm, bdeg_result *out) {
    if (!p || !out || !comm || !comm->allreduce_sum || !comm->alltoall_counts || !comm->alltoall_cells)
        return fail(p, BDEG_E_INVALID, "NULL argument");
    const double t0 = now_ms();
    bdeg_result r;
    fill_front(p, &r);
    if (p->K == 0) {
        r.deg_lo = 1;
        *out = r;
        return BDEG_OK;
    }
    bdeg_status s = ensure_device(p);
    if (s) return s;
    double kms = 0;
    // ties are reduced over all ranks inside, so every rank takes the same
    // branch here and re-lifts with the same attempt
    for (int attempt = p->relifts;; ++attempt) {
        fill_front(p, &r);
        s = walk_sharded(p, comm, &r, &kms);
        if (s != BDEG_E_DEGENERATE) break;
        if (p->user_lift || (p->opt.flags & BDEG_FLAG_NO_RELIFT)) return s;
        if (attempt + 1 > p->opt.max_relift) return s;
        bdeg_relift(p, attempt + 1);
        s = ensure_device(p);
        if (s) return s;
    }
    if (s) return s;
    r.relifts = p->relifts;
    r.seed_used = p->seed_used;
    r.kernel_ms = kms;
    r.total_ms = now_ms() - t0;
    *out = r;
    return BDEG_OK;
}

bdeg_status bdeg_steal_create(int32_t device, uint8_t *out_handle) {
    if (!out_handle) return fail(nullptr, BDEG_E_INVALID, "NULL argument");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(nullptr, BDEG_E_CUDA, cudaGetErrorString(e));
    void *ptr = nullptr;
    if ((e = cudaMalloc(&ptr, 256)) != cudaSuccess) return fail(nullptr, BDEG_E_CUDA, cudaGetErrorString(e));
    if ((e = cudaMemset(ptr, 0, 256)) != cudaSuccess) return fail(nullptr, BDEG_E_CUDA, cudaGetErrorString(e));
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, ptr)) != cudaSuccess) return fail(nullptr, BDEG_E_CUDA, cudaGetErrorString(e));
    static_assert(sizeof(h) == BDEG_STEAL_HANDLE_BYTES, "IPC handle size");
    std::memcpy(out_handle, &h, sizeof(h));
    {   // the exporting process cannot IPC-open its own allocation: remember it
        std::lock_guard<std::mutex> lk(g_mu);
        g_steal_local[std::string((const char *)out_handle, sizeof(h))] = ptr;
    }
    return BDEG_OK;
}

bdeg_status bdeg_steal_attach(bdeg_plan_t p, const uint8_t *handle) {
    if (!p || !handle) return fail(p, BDEG_E_INVALID, "NULL argument");
    bdeg_status s = ensure_device(p);
    if (s) return s;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *ptr = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_steal_local.find(std::string((const char *)handle, sizeof(h)));
        if (it != g_steal_local.end()) ptr = it->second;
    }
    if (!ptr) {
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(p, BDEG_E_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    p->steal = (unsigned long long *)ptr;
    p->steal_parity = 0;
    return BDEG_OK;
}

bdeg_status bdeg_rank_modp(int32_t n, int32_t m, const int64_t *A, uint32_t prime, int32_t device, void *stream,
                           int64_t *rank) {
    if (!A || !rank || n < 1 || m < 0 || prime < 3) return fail(nullptr, BDEG_E_INVALID, "bad arguments");
    if (m == 0) { *rank = 0; return BDEG_OK; }
    const long long r = rank_modp(A, n, m, prime, device, stream);
    if (r < 0) return fail(nullptr, BDEG_E_CUDA, "GPU row reduction failed (no CUDA device?)");
    *rank = r;
    return BDEG_OK;
}

bdeg_status bdeg_dimension_modp(int32_t n, int32_t m, const int64_t *A, int32_t device, int32_t *dim) {
    if (!dim) return fail(nullptr, BDEG_E_INVALID, "NULL argument");
    const uint32_t primes[2] = {2147483647u, 2147483629u};   // 2^31 - 1, 2^31 - 19
    int64_t best = 0;
    for (uint32_t pr : primes) {
        int64_t r = 0;
        bdeg_status s = bdeg_rank_modp(n, m, A, pr, device, nullptr, &r);
        if (s) return s;
        best = std::max(best, r);
    }
    *dim = (int32_t)(n - best);
    return BDEG_OK;
}

bdeg_status bdeg_smith_gpu(int32_t n, int32_t m, const int64_t *A, int32_t device, void *stream, int64_t *rank,
                           uint64_t *comp_lo, uint64_t *comp_hi, int64_t *unit_pivots) {
    Nvtx range("bdeg smith (unit pivots)");
    if (!A || !rank || n < 1 || m < 0) return fail(nullptr, BDEG_E_INVALID, "bad arguments");
    for (size_t i = 0; i < (size_t)n * m; ++i)
        if (A[i] >= ((int64_t)1 << 61) || A[i] <= -((int64_t)1 << 61))
            return fail(nullptr, BDEG_E_TOO_LARGE, "matrix entry beyond 2^61");
    long long piv = 0;
    std::vector<int64_t> res;
    int rr = 0, rc = 0;
    if (m > 0) {
        const int e = smith_unimodular(A, n, m, device, stream, &piv, res, rr, rc);
        if (e < 0) return fail(nullptr, BDEG_E_CUDA, "GPU unimodular elimination failed (no CUDA device?)");
        if (e > 0) return fail(nullptr, BDEG_E_TOO_LARGE, "unimodular elimination: an entry grew beyond 2^61");
    }
    int rres = 0;
    u128 prod = 1;
    if (rr > 0 && rc > 0) {
        if ((double)rr * rc > 4.0e6)
            return fail(nullptr, BDEG_E_TOO_LARGE, "residual block without unit pivots is too large (" +
                                                       std::to_string(rr) + " x " + std::to_string(rc) + ")");
        std::string err;
        if (!smith_factors(rr, rc, res.data(), rres, prod, err)) return fail(nullptr, BDEG_E_TOO_LARGE, err);
    }
    *rank = piv + rres;
    if (comp_lo) *comp_lo = (uint64_t)prod;
    if (comp_hi) *comp_hi = (uint64_t)(prod >> 64);
    if (unit_pivots) *unit_pivots = piv;
    return BDEG_OK;
}

const char *bdeg_last_error(bdeg_plan_t p) { return p ? p->err.c_str() : g_err.c_str(); }

const char *bdeg_status_str(bdeg_status s) {
    switch (s) {
        case BDEG_OK: return "ok";
        case BDEG_E_INVALID: return "invalid argument";
        case BDEG_E_INCONSISTENT: return "inconsistent system";
        case BDEG_E_DEGENERATE: return "degenerate lifting";
        case BDEG_E_IO: return "io error";
        case BDEG_E_TOO_LARGE: return "too large";
        case BDEG_E_CUDA: return "cuda error";
        case BDEG_E_COMM: return "communication error";
    }
    return "unknown";
}

void bdeg_destroy(bdeg_plan_t p) {
    if (!p) return;
    // bdeg_degree_partial is asynchronous: the plan's kernels may still read
    // the workspace, which the pool may hand to the next plan
    if (p->dev_ready) cudaStreamSynchronize((cudaStream_t)p->opt.stream);
    if (p->own_ws && p->ws) pool_put(p->opt.device, p->ws, p->ws_bytes);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    delete p;
}

uint64_t bdeg_launch_count(void) { return launch_counter_add(0); }

}  // extern "C"
