// arrow_internal.h -- internal types shared by the host decomposer, plan builder and kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace arrow {

// One arrow matrix B_i of the decomposition, in positions (Eq. (1)).
// perm[p] = original vertex at position p (pi_i^{-1}); entries carry the index of the
// originating entry of A (`src`) so that values are gathered in the plan's dtype.
struct HostLevel {
    int64_t rows = 0;     // n for level 0 (A-isolated vertices appended), n_i otherwise
    int64_t n_i = 0;      // vertices with an entry in A_i
    int64_t head = 0;     // h_i = min(b, n_i)
    std::vector<int32_t> perm;      // [rows]
    std::vector<int64_t> row_ptr;   // [rows + 1]
    std::vector<int32_t> col;       // [nnz] positions, strictly increasing per row
    std::vector<uint32_t> src;      // [nnz] entry index into A's CSR arrays (decomposer output)
    std::vector<double> val;        // [nnz] values (exact copy of A's fp32/fp64 values)
    std::vector<int64_t> home_start;  // [homes + 1] (home-aware, levels >= 1): trees of home g at [hs[g], hs[g+1])
};

struct HostDecomposition {
    int64_t n = 0, b = 0;
    int band = 0;                    // step 3's band: 0 block-diagonal tiles (R3), 1 strict |p-q| <= b
    std::vector<HostLevel> levels;
    std::vector<uint32_t> residual;  // entry indices of A left when the level cap is reached
    int homes = 1;                   // G of the home-set-aware arrangement (R25); 1 = R11
    int home_levels = 0;             // levels 1..home_levels are home-aware (homes > 1)
    std::vector<int64_t> home_los;   // [homes + 1] pi_0 home ranges (homes > 1)
};

// LA-Decompose (decompose.cpp).  homes > 1: levels 1..home_levels home-set-aware (R25).  Returns 0
// on success, else sets `err`.
int la_decompose(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t b, int32_t max_levels,
                 uint64_t seed, int band, int homes, int home_levels, HostDecomposition &out, std::string &err);

// R25: tile boundaries of a G-way split of prefix costs pre[0..T] (each boundary the
// prefix nearest g/G of the total, ties to the upper one, never before the previous) -> tb[0..G]
std::vector<int64_t> split_prefix(const std::vector<int64_t> &pre, int G);
// R25: pi_0 home ranges los[0..G] from level 0's tile work plus the remainder degree of every vertex
// (rem_deg[v] = entries of row v left for levels >= 1); A-isolated positions are a last pseudo-tile
std::vector<int64_t> home_ranges(const HostLevel &L0, int64_t n, int64_t b, int G, const int32_t *rem_deg);

// LA-Decompose on the current CUDA device (gdecompose.cu): the same output as
// la_decompose, bit for bit (same rules and keys; Boruvka + Euler-tour list ranking in place of the
// sequential Kruskal / BFS / DFS).  n < 2^30, nnz < 2^31 - 1.  Checks the pattern's symmetry on the
// device (2 if it is not).  0 on success, else sets `err` (1: CUDA failure).
int la_decompose_gpu(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t b, int32_t max_levels,
                     uint64_t seed, int band, int homes, int home_levels, HostDecomposition &out,
                     std::string &err);

// Validation helpers (decompose.cpp): 0 ok, 1 bad CSR, 2 not symmetric.
int validate_csr(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col, std::string &err);
int check_symmetric(int64_t n, const int64_t *row_ptr, const int32_t *col, std::string &err);

// ------------------------------------------------------------------ device layout of one level
// Built on the host as a stream of records (key, val) in tile-window order:
//   plain record  : key = X row (the folded permutation: P_pi^T X is never materialised, S4);
//                   kAux set (distributed only) = row of the staged head block D0 = X[head_i]
//   pseudo record : kPseudo | out row -- closes the current segment.  kAux set = head-row partial of
//                   one tile window (Alg. 1 line 2, C^(0) = sum_t B^(0,t) D^(t)) added
//                   atomically (single GPU: into Y[perm_i[j]]; distributed: into C0[j]); otherwise
//                   body row p >= h_i stored (level 0) or read-modify-written (levels >= 1, S5).
// and converted into the segment layout below (layout.cpp).
constexpr uint32_t kPseudoRec = 0x80000000u;
constexpr uint32_t kFlag = 0x80000000u;
constexpr uint32_t kAuxRec = 0x40000000u;
constexpr int64_t kMaxRows = (int64_t)1 << 30;
// default home-aware levels (R25) for G homes, measured at config R: at G = 2 the
// halo already hides under level 0, so one level; from G = 4 on three levels
inline int default_home_levels(int homes) { return homes <= 2 ? 1 : 3; }
constexpr int kDefaultBatchSegs = 16;  // segments per K-A work batch of full-warp rows (measured: 16 > 32)

// metadata of one level (introspection) and its level-0 zero-row list
struct DeviceLevel {
    int64_t rows = 0, n_i = 0, head = 0, nnz = 0, head_nnz = 0, tiles = 0;
    int64_t nseg = 0, nzero = 0;
    int mode = 0;                  // 0: level 0 stores Y rows; 1: levels >= 1 read-modify-write (S5)
    int32_t *zero_rows = nullptr;  // [nzero] level 0: Y rows written as 0 (head rows first, then entry-less rows)
};

// Segment layout of one level (the K-A input).  Segments (an output row, or one window's chunk of a
// head row; never empty) in tile-window order, their (col, val) entries contiguous; work batch b is
// segments [b (bs+1), b (bs+1) + bs), starting at a multiple of 8 entries, and is followed by one
// padding segment (output kDiscard) that fills the gap to the next batch.
//   seg_out[nseg]  output row (bit 31: head-row partial, added atomically; bit 30: final write, iterate)
//   seg_end[nseg]  end offset of the segment's entries
//   ent_col[nent]  X row of each entry (bit 31, distributed: row of the head block D0)
//   ent_val[nent]  value (plan dtype)
//   gmask[nent/8]  bit t of byte g: entry 8g + t is the last entry of its segment
//   bat[2*nbatch]  (first entry, end entry) of batch b's real segments
struct SegLevel {
    int64_t nseg = 0, nent = 0, nbatch = 0;
    int bs = kDefaultBatchSegs;
    int mode = 0;
    int64_t max_x_row = (int64_t)1 << 40;  // bound on the X / D0 rows referenced (32-bit offsets below 4 GiB)
    int32_t *seg_out = nullptr;
    uint32_t *seg_end = nullptr;
    int32_t *ent_col = nullptr;
    void *ent_val = nullptr;
    uint8_t *gmask = nullptr;
    uint32_t *bat = nullptr;
};

// host form of a level's segment list before padding (layout.cpp input): seg_end relative to ent_col
struct HostSegs {
    std::vector<int32_t> seg_out;
    std::vector<uint32_t> seg_end;
    std::vector<int32_t> ent_col;
    std::vector<uint8_t> ent_val;  // plan dtype, element size es
};
// Build the end masks and batch table, and upload (cudaMalloc'ed pointers appended to `allocs`, freed by the
// owner).  Returns 0 or a cudaError_t; `err` gets a message for layout errors (offsets beyond 32 bits).
int upload_seg_level(const HostSegs &h, int es, int bs, int mode, int64_t max_x_row, std::vector<void *> &allocs,
                     SegLevel &out, std::string &err);

// Peer (NVLink) addressing of the distributed P2P transport: an encoded row is
// (rank << kPeerShift | row) into the per-rank base pointers of a PeerPtrs; kParityBit marks a row
// of the double-buffered head partial C0 (shifted by the current call's parity offset).
constexpr int kMaxPeers = 8;
constexpr int kPeerShift = 27;
constexpr uint32_t kPeerRowMask = (1u << kPeerShift) - 1u;
constexpr uint32_t kParityBit = 0x40000000u;
constexpr uint32_t kLocalRmwBit = 0x40000000u;  // K-A (dist 2): out row is a local Y row, read-modify-written
struct PeerPtrs {
    void *p[kMaxPeers];
    int act = 0;  // K-A only: activation applied when a row's final segment is flushed (iterate mode)
    // K-A level 0, single GPU: Y rows to zero (entry-less and A-isolated rows), shared out over the
    // warps' batch grabs so that their stores overlap the gathers instead of a separate K-Z pass
    const int32_t *zrows = nullptr;
    int64_t nzero = 0;
};
// single GPU: a body segment whose row receives no later contribution (arrow_spmm_iterate's
// activation is applied when it is flushed); activations: 0 identity, 1 ReLU
constexpr uint32_t kFinalBit = 0x40000000u;
constexpr uint32_t kDiscard = 0x7fffffffu;  // seg_out of a padding segment: its result is dropped
constexpr uint32_t kRowMask30 = 0x3fffffffu;
// per-call K-A options (from arrow_options; none at present)
struct SegLaunch {};
// dist: 0 single GPU, 1 distributed (head columns from D0, head partials into C0), 2 as 1 with
// body rows stored through `outs` (encoded rows, levels >= 1 of the P2P transport) or, with
// kLocalRmwBit, added into Y (rows whose home is this rank)
int launch_seg(int dtype, int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
               int num_sms, unsigned *counter, void *stream, const SegLaunch &opt, const PeerPtrs *outs = nullptr,
               int act = 0, const int32_t *zrows = nullptr, int64_t nzero = 0);
// Y[rows[i]] = act(Y[rows[i]]) (rows whose last contribution is a head-row partial)
int launch_act_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, int act, void *Y, void *stream);
// dst row enc(didx[i]) of bases = src[sidx[i]] (sidx < 0: zero); grid of `blocks` (0: sized to n)
int launch_push_rows(int dtype, const void *src, const int32_t *sidx, const int32_t *didx, int64_t n, int64_t k,
                     const PeerPtrs &bases, int blocks, void *stream);
// Y[drow[r]] += sum of row enc(src[e]) of bases (+ par_shift rows when kParityBit), e in [ptr[r], ptr[r+1])
int launch_gather_add_peers(int dtype, const PeerPtrs &bases, int64_t par_shift, const int32_t *ptr,
                            const int32_t *src, const int32_t *drow, int64_t n, int64_t k, void *Y, void *stream);
// cross-GPU barrier: thread g publishes `epoch` into slot `slot` of rank g's flag array, then waits
// until every rank has published it into this rank's array (system-scope release/acquire; traps
// after ~60 s so a lost peer cannot hang the GPU)
int launch_barrier(const PeerPtrs &flags, const unsigned *mine, int slot, unsigned epoch, int me, int G, void *stream);

// kernels.cu launchers (all on `stream`; return cudaError_t as int)
int device_sms();  // SM count of the current device (cudaDevAttrMultiProcessorCount, cached)
int launch_zero_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, void *Y, void *stream, int blocks = 0);
int launch_zero(void *Y, int64_t bytes, void *stream);
// dst[didx[i]] (= | +=) src[sidx[i]] (identity when an index list is NULL; sidx[i] < 0 writes zero)
int launch_rows(int dtype, const void *src, const int32_t *sidx, const int32_t *didx, int64_t n, int64_t k, int add,
                void *dst, void *stream);
// dst[drow[r]] += sum of src[sidx[e]] for e in [ptr[r], ptr[r+1]) (CSR of contributions, list order)
int launch_gather_add(int dtype, const void *src, const int32_t *ptr, const int32_t *sidx, const int32_t *drow,
                      int64_t n, int64_t k, void *dst, void *stream);

}  // namespace arrow
