// Internal declarations shared by the host front end (frontend.cpp,
// bdeg_capi.cpp) and the CUDA kernels (bdeg_kernels.cu) of libbdeg.so.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bdeg {

typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr int kMaxN = 64;    // points: the kernel maps one point to a lane slot (2 slots/lane)
constexpr int kMaxK = 32;    // subset size (K+1 rows of the lifted matrix, <= 33)
constexpr int kMaxInner = 7;   // register-resident DFS levels (template parameter S)
constexpr int kBinomRows = 65;
constexpr int kBinomCols = 34;

// ----------------------------------------------------------------- front end
struct FrontEnd {
    int n = 0, m = 0, rank = 0, dim = 0;
    u128 components = 1;
    bool consistent = true;
    bool homogeneous = false;
    std::vector<std::vector<i128>> P0;   // dim x n (rows = basis of the left kernel lattice)
};

// SNF-based analysis of x^A = b.  Returns false with
// `err` set on arithmetic overflow.
bool analyze_system(int n, int m, const int64_t *A, const double *b_re, const double *b_im,
                    bool lll, FrontEnd &fe, std::string &err);

// Invariant factors of a (small) integer matrix by the same Euclidean
// Smith form: rank and |prod d_j|.  false + err on overflow.
bool smith_factors(int n, int m, const int64_t *A, int &rank, u128 &prod, std::string &err);

// Point configuration (Prop. 4; readings Z2/Z5): distinct non-zero
// columns of P0 in first-occurrence order (min lifting on merge), then the
// origin (generic case, K = d+1, v = (1, a)), or only the columns (homogeneous
// pyramid case, K = d).  lifting: n+1 values.  V is point-major N x K.
void build_points(const FrontEnd &fe, const int64_t *lifting, bool homog_shortcut,
                  int &K, int &N, std::vector<int64_t> &V, std::vector<int64_t> &w,
                  std::vector<int> &point_of_var, int &origin_index);

// SplitMix64 (DESIGN.md input recipe; the same generator workloads/ uses).
struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
};
uint64_t derive_seed(uint64_t seed, int attempt);

// ----------------------------------------------------------------- kernels
struct DeviceProblem {
    const int64_t *L;        // (K+1) x N lifted matrix, column-major: L[l*(K+1) + i]
    const uint64_t *binom;   // kBinomRows x kBinomCols
    int K, N, S, T;          // subset size, points, register-DFS levels, smem prefix levels (K-1-S)
    int D;                   // work-item depth: items are D-tuples of the largest indices (D >= T)
};

struct LaunchArgs {
    DeviceProblem P;
    uint64_t rank_begin, rank_end;    // candidate colex ranks [begin, end)
    // Work queue (bdeg_capi.cpp build_queue): positions [0, n_items).
    //   mode 0 (rank range): position i = base-depth colex item blk_last - i
    //   mode 1 (whole space, largest-first): positions < n_split are split
    //     items (depth << 58 | colex id at that depth), the rest are grouped
    //     base-depth items (group g: smallest top index grp_u[g], first
    //     position n_split + grp_cum[g], members in colex order of the rest)
    int mode;
    uint64_t blk_first, blk_last;     // mode 0: inclusive base-depth item range covering [begin, end)
    const uint64_t *split;            // mode 1
    uint64_t n_split;
    const uint64_t *grp_u, *grp_cum;  // mode 1: n_grp groups, grp_cum[n_grp] = grouped total
    int n_grp;
    uint64_t n_items;
    uint64_t n_static;                // positions rank + i*world < n_static: static interleave
    uint64_t grab;                    // tail positions taken per global atomic
    int rank, world;
    unsigned long long *counter;      // this GPU's queue counter (zeroed before launch)
    unsigned long long *gcounter;     // cross-GPU tail counter (IPC-mapped) or null
    unsigned long long *slots;        // kNSlots accumulators
    unsigned long long *mark_bits;    // bitmap over queue positions: items this launch could not
                                      // finish in its tier (narrow -> int64 -> int128 chain)
    unsigned long long *replay_bits;  // replay launches: the positions to redo (cleared as read)
    uint64_t ovf_words;               // 64-bit words of each bitmap
    int tier;                         // 0: int32/int32, 1: int32/int64 (bounds), 2: int64/int128
    int bits_v, bits_l;               // tier-1 bounds: |V| < 2^bits_v, |lift| < 2^bits_l
    int replay;                       // 1: process the positions set in replay_bits (tier 2 or 4)
    const unsigned long long *replay_gate;   // replays: the slot counting the marked items (0 => exit at once)
    int grid, block;                  // launch shape
    int degree_only;                  // skip cell-dead subtrees
    int dead_full;                    // full mode: detect cell-dead subtrees, their leaves count singular only
    unsigned long long *cells_out;    // optional (mask, |det|) output of the cells found
    unsigned long long *cells_cnt;
    uint64_t cells_cap;
    int stop_on_cell;                 // warps stop taking items once a cell was emitted
    unsigned long long *reset_next;   // cross-GPU stealing: counter of the next step, zeroed by rank 0
    int system_counter;               // counter lives in a peer GPU (IPC): system-scope atomics
    void *stream;
};

constexpr int kNSlots = 16;
enum Slot {
    SLOT_VOL0 = 0, SLOT_VOL1, SLOT_VOL2, SLOT_VOL3,   // 32-bit limbs of the volume
    SLOT_CELLS = 4, SLOT_SINGULAR = 5, SLOT_CAND = 6, SLOT_TIES = 7,
    SLOT_OVF_BLOCKS = 8,   // int32-tier blocks queued for re-run
    SLOT_FATAL = 9,        // int64-tier overflow (value beyond int64)
    SLOT_QFULL = 10,       // (unused: the re-run bitmap has one bit per work item)
    SLOT_BLOCKS = 11, SLOT_UPDATES = 12, SLOT_LEAVES = 13,
    SLOT_DEAD = 14,        // leaves inside cell-dead subtrees (singular count only)
    SLOT_WIDE = 15         // items re-run in the int128-value tier (tier 4)
};

// Dynamic shared memory bytes for a launch of the enumeration kernel.
size_t enumerate_smem_bytes(int K, int N, int warps_per_cta);
// Launch k_enumerate (returns cudaError_t as int).
int launch_enumerate(const LaunchArgs &a);
// Tier 4 (int128 values, 256-bit exact intermediates): replay of the items
// marked in a.replay_bits by a tier-2 launch.
int launch_enumerate_wide(const LaunchArgs &a);
int kernel_warps_per_cta();
// Max resident CTAs per SM for this configuration (occupancy API).
int enumerate_max_ctas_per_sm(const LaunchArgs &a);

uint64_t launch_counter_add(uint64_t k);

// ---- cell walk, bdeg_walk.cu.  Cell masks are 128-bit
// {lo, hi} pairs (N <= 128); device buffers hold 16 bytes per mask.
constexpr int kMaxNWalk = 128;
size_t walk_smem_bytes(int K, int N);
uint64_t walk_hash(uint64_t lo, uint64_t hi);
int launch_walk(const int64_t *L, int K, int N, const void *cur, uint64_t ncur, void *next,
                unsigned long long *next_cnt, void *table, uint64_t cap, unsigned long long *counter,
                unsigned long long *stats, int grid, void *stream, int64_t limV, int64_t limL,
                unsigned long long *vol, int *fused, uint8_t *tags, unsigned tag, uint64_t next_cap,
                int narrow = 0, void *ovfl = nullptr, unsigned long long *ovfl_cnt = nullptr,
                uint64_t ovfl_cap = 0, int vsafe = 0, int world = 1, int rank = 0, void *remote = nullptr,
                unsigned long long *remote_cnt = nullptr, uint64_t remote_cap = 0);
// sharded walk: owner of a cell (= device owner_of), receive-side insert,
// partition of the remote cells by owner
inline int walk_owner(uint64_t lo, uint64_t hi, int world) {
    return (int)((uint32_t)walk_hash(lo, hi) % (uint32_t)world);
}
int launch_insert_recv(const void *list, uint64_t n, void *tab, uint8_t *tags, uint64_t cap, uint8_t tag, void *next,
                       unsigned long long *next_cnt, uint64_t next_cap, unsigned long long *full_flag, void *stream);
int launch_owner_count(const void *list, uint64_t n, int world, unsigned long long *cnt, void *stream);
int launch_owner_scatter(const void *list, uint64_t n, int world, unsigned long long *cursor, void *out,
                         void *stream);
int launch_cellvol(const int64_t *L, int K, int N, const void *table, uint64_t cap, unsigned long long *out,
                   unsigned long long *counter, int grid, void *stream, int64_t limV, int64_t limL);
int launch_rehash(const void *old, const uint8_t *old_tags, uint64_t oldcap, void *tab, uint8_t *tags, uint64_t cap,
                  unsigned long long *full_flag, void *stream, uint8_t keep0 = 0, int keep_n = 0);
int launch_insert_list(const void *list, uint64_t n, void *tab, uint8_t *tags, uint64_t cap, uint8_t tag,
                       unsigned long long *full_flag, void *stream);
int launch_collect(const void *tab, const uint8_t *tags, uint64_t cap, uint8_t tag, void *out,
                   unsigned long long *cnt, void *stream);

// ---- front end at scale, bdeg_rank.cu
long long rank_modp(const int64_t *A, int n, int m, uint32_t p, int device, void *stream);
int smith_unimodular(const int64_t *A, int n, int m, int device, void *stream, long long *pivots,
                     std::vector<int64_t> &residual, int &res_rows, int &res_cols);

}  // namespace bdeg
