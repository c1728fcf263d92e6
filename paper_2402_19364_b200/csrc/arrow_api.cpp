// arrow_api.cpp -- the C ABI (include/arrow.h): validation, plan build (decomposition ->
// window-ordered device segment layout), upload, and the arrow_spmm launch sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <omp.h>
#include <string>
#include <vector>

#include "../../include/arrow.h"
#include "arrow_internal.h"
#include "comm.h"
#include "plan.h"

using namespace arrow;

namespace {

thread_local std::string g_err;

arrow_status fail(arrow_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess) return fail(ARROW_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

}  // namespace

arrow_status arrow::set_error(arrow_status s, const std::string &msg) { return fail(s, msg); }

// ------------------------------------------------------------------------------------ layout
namespace {

struct BuiltLevel {
    std::vector<uint32_t> keys;    // record stream (arrow_internal.h)
    std::vector<uint8_t> vals;     // plan dtype
    std::vector<int32_t> zero_rows;
    int64_t rows = 0, n_i = 0, head = 0, nnz = 0, head_nnz = 0, tiles = 0, nseg = 0;
    int mode = 0;
};

inline void put_val(std::vector<uint8_t> &dst, int64_t at, arrow_dtype pdt, double v) {
    if (pdt == ARROW_F64) {
        std::memcpy(dst.data() + at * 8, &v, 8);
    } else {
        const float f = (float)v;
        std::memcpy(dst.data() + at * 4, &f, 4);
    }
}

// Window-ordered record stream of one arrow level (encoding: arrow_internal.h).
//   dist = 0: head columns read X directly, head-row partials add into Y[perm_i[j]];
//             level 0 zeroes head rows and entry-less rows first (zero_rows).
//   dist = 1: head columns read the staged head block D0, head partials add into C0[j].
void build_level(const HostLevel &L, int level_idx, int64_t b, int64_t window_rows, int32_t head_chunk,
                 const std::vector<int32_t> *pos0, arrow_dtype pdt, int dist, BuiltLevel &B) {
    const int64_t n_i = L.n_i, h = L.head, rows = L.rows;
    B.rows = rows;
    B.n_i = n_i;
    B.head = h;
    B.nnz = L.row_ptr[rows];
    B.head_nnz = L.row_ptr[h];
    B.tiles = (n_i + b - 1) / b;
    B.mode = level_idx == 0 ? 0 : 1;
    auto rowid = [&](int32_t v) -> uint32_t { return (uint32_t)(pos0 ? (*pos0)[v] : v); };
    auto colkey = [&](int32_t q) -> uint32_t {
        return (dist && q < h) ? (kAuxRec | (uint32_t)q) : rowid(L.perm[q]);
    };
    auto headkey = [&](int64_t j) -> uint32_t {
        return kPseudoRec | kAuxRec | (dist ? (uint32_t)j : rowid(L.perm[j]));
    };
    if (level_idx == 0) {
        if (!dist)
            for (int64_t j = 0; j < h; ++j) B.zero_rows.push_back((int32_t)rowid(L.perm[j]));
        for (int64_t p = h; p < rows; ++p)
            if (L.row_ptr[p + 1] == L.row_ptr[p]) B.zero_rows.push_back((int32_t)rowid(L.perm[p]));
    }

    const int64_t wt = std::max<int64_t>(1, window_rows / b);
    const int64_t W = wt * b;
    const int64_t NW = (n_i + W - 1) / W;
    std::vector<int64_t> wrec(NW + 1, 0), wseg(NW + 1, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < NW; ++w) {
        const int64_t lo = w * W, hi = std::min(n_i, lo + W);
        int64_t sc = 0, ec = 0;
        for (int64_t p = std::max(h, lo); p < hi; ++p) {
            const int64_t c = L.row_ptr[p + 1] - L.row_ptr[p];
            sc += c > 0 ? 1 : 0;
            ec += c;
        }
        for (int64_t j = 0; j < h; ++j) {
            const int32_t *a = L.col.data() + L.row_ptr[j], *z = L.col.data() + L.row_ptr[j + 1];
            const int64_t c = std::lower_bound(a, z, (int32_t)hi) - std::lower_bound(a, z, (int32_t)lo);
            sc += (c + head_chunk - 1) / head_chunk;
            ec += c;
        }
        wseg[w + 1] = sc;
        wrec[w + 1] = ec + sc;
    }
    for (int64_t w = 0; w < NW; ++w) { wrec[w + 1] += wrec[w]; wseg[w + 1] += wseg[w]; }
    const int64_t nrec = wrec[NW];
    B.nseg = wseg[NW];
    B.keys.resize(nrec);
    B.vals.assign(nrec * (pdt == ARROW_F64 ? 8 : 4), 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < NW; ++w) {
        const int64_t lo = w * W, hi = std::min(n_i, lo + W);
        int64_t r = wrec[w];
        auto entry = [&](int64_t e) {
            B.keys[r] = colkey(L.col[e]);
            put_val(B.vals, r, pdt, L.val[e]);
            ++r;
        };
        for (int64_t p = std::max(h, lo); p < hi; ++p) {
            if (L.row_ptr[p + 1] == L.row_ptr[p]) continue;
            for (int64_t x = L.row_ptr[p]; x < L.row_ptr[p + 1]; ++x) entry(x);
            // level 0 stores the row; levels >= 1 read-modify-write it (S5)
            B.keys[r++] = kPseudoRec | rowid(L.perm[p]);
        }
        for (int64_t j = 0; j < h; ++j) {
            const int32_t *a = L.col.data() + L.row_ptr[j], *z = L.col.data() + L.row_ptr[j + 1];
            int64_t x0 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)lo) - a);
            const int64_t x1 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)hi) - a);
            while (x0 < x1) {
                const int64_t x2 = std::min<int64_t>(x1, x0 + head_chunk);
                for (int64_t x = x0; x < x2; ++x) entry(x);
                B.keys[r++] = headkey(j);
                x0 = x2;
            }
        }
    }
}

// Residual CSR level (ARROW_RESIDUAL_CSR): every row with leftover entries is one RMW segment.
void build_residual(const arrow_decomposition_s &D, const std::vector<int32_t> *pos0, arrow_dtype pdt,
                    BuiltLevel &B) {
    auto rowid = [&](int32_t v) -> uint32_t { return (uint32_t)(pos0 ? (*pos0)[v] : v); };
    const size_t m = D.res_u.size();
    B.mode = 1;
    B.nnz = (int64_t)m;
    const size_t es = pdt == ARROW_F64 ? 8 : 4;
    B.vals.reserve((m + m / 2 + 1) * es);
    for (size_t t = 0; t < m; ++t) {
        B.keys.push_back(rowid(D.res_v[t]));
        B.vals.resize(B.keys.size() * es);
        put_val(B.vals, (int64_t)B.keys.size() - 1, pdt, D.res_a[t]);
        if (t + 1 == m || D.res_u[t + 1] != D.res_u[t]) {
            B.keys.push_back(kPseudoRec | rowid(D.res_u[t]));
            B.vals.resize(B.keys.size() * es, 0);
            ++B.nseg;
        }
    }
    B.rows = B.nseg;
    B.n_i = B.nseg;
}

arrow_status validate_args(const arrow_csr *A, int64_t b, int32_t levels) {
    if (!A) return fail(ARROW_E_INVALID_ARG, "A is NULL");
    if (b < 2) return fail(ARROW_E_INVALID_ARG, "arrow width b must be >= 2 (PAPER.md P:807)");
    if (levels < 0) return fail(ARROW_E_INVALID_ARG, "levels must be >= 0");
    if (A->n < 0 || A->nnz < 0) return fail(ARROW_E_INVALID_ARG, "negative n or nnz");
    if (A->dtype != ARROW_F32 && A->dtype != ARROW_F64) return fail(ARROW_E_INVALID_ARG, "bad dtype");
    if (!A->row_ptr) return fail(ARROW_E_INVALID_ARG, "row_ptr is NULL");
    if (A->nnz > 0 && (!A->col_idx || !A->values)) return fail(ARROW_E_INVALID_ARG, "col_idx/values NULL");
    if (A->n >= ((int64_t)1 << 31) - 1) return fail(ARROW_E_UNSUPPORTED, "n must be < 2^31 - 1 (int32 indices)");
    if (A->nnz >= ((int64_t)1 << 32) - 1) return fail(ARROW_E_UNSUPPORTED, "nnz must be < 2^32 - 1");
    return ARROW_OK;
}

}  // namespace

// ------------------------------------------------------------------------------------ ABI

extern "C" {

const char *arrow_status_string(arrow_status s) {
    switch (s) {
        case ARROW_OK: return "ARROW_OK";
        case ARROW_E_INVALID_ARG: return "ARROW_E_INVALID_ARG";
        case ARROW_E_BAD_CSR: return "ARROW_E_BAD_CSR";
        case ARROW_E_NOT_SYMMETRIC: return "ARROW_E_NOT_SYMMETRIC";
        case ARROW_E_LEVELS: return "ARROW_E_LEVELS";
        case ARROW_E_CUDA: return "ARROW_E_CUDA";
        case ARROW_E_NCCL: return "ARROW_E_NCCL";
        case ARROW_E_NOMEM: return "ARROW_E_NOMEM";
        case ARROW_E_STATE: return "ARROW_E_STATE";
        case ARROW_E_UNSUPPORTED: return "ARROW_E_UNSUPPORTED";
    }
    return "ARROW_E_UNKNOWN";
}

const char *arrow_last_error(void) { return g_err.c_str(); }
int32_t arrow_abi_version(void) { return ARROW_ABI_VERSION; }

arrow_status arrow_options_default(arrow_options *opt) {
    if (!opt) return fail(ARROW_E_INVALID_ARG, "opt is NULL");
    std::memset(opt, 0, sizeof(*opt));
    opt->compute = ARROW_DTYPE_DEFAULT;
    opt->seed = 4;
    opt->order = ARROW_ORDER_ORIGINAL;
    opt->residual = ARROW_RESIDUAL_ERROR;
    opt->window_rows = 0;
    opt->head_chunk = 0;
    return ARROW_OK;
}

arrow_status arrow_plan_create(const arrow_csr *A, int64_t b, int32_t levels, arrow_plan *out) {
    return arrow_plan_create_ex(A, b, levels, nullptr, nullptr, out);
}

static arrow_status decompose_impl(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, bool keep_residual,
                                   int32_t band, int32_t homes, int32_t home_levels, bool on_gpu,
                                   std::unique_ptr<arrow_decomposition_s> &D) {
    const auto t0 = std::chrono::steady_clock::now();
    arrow_status st = validate_args(A, b, levels);
    if (st != ARROW_OK) return st;
    if (band != ARROW_BAND_BLOCK && band != ARROW_BAND_STRICT) return fail(ARROW_E_INVALID_ARG, "bad band");
    if (homes < 1 || homes > 8) return fail(ARROW_E_INVALID_ARG, "homes must be in [1, 8]");
    if (home_levels < 0) return fail(ARROW_E_INVALID_ARG, "home_levels must be >= 0 (0 = default)");
    if (homes > 1 && home_levels == 0) home_levels = default_home_levels(homes);
    std::string err;
    const int64_t n = A->n;
    if (validate_csr(n, A->nnz, A->row_ptr, A->col_idx, err)) return fail(ARROW_E_BAD_CSR, err);
    // the GPU decomposer checks the symmetry itself (on the device)
    if (!on_gpu && check_symmetric(n, A->row_ptr, A->col_idx, err)) return fail(ARROW_E_NOT_SYMMETRIC, err);
    const auto t1 = std::chrono::steady_clock::now();
    try {
        D.reset(new arrow_decomposition_s());
        D->n = n;
        D->b = b;
        D->seed = seed;
        D->band = band;
        HostDecomposition H;
        if (on_gpu) {
            if (n >= ((int64_t)1 << 30) || A->nnz >= ((int64_t)1 << 31) - 1)  // CUB item counts (2 n arcs) are int
                return fail(ARROW_E_INVALID_ARG, "GPU decomposer: n or nnz beyond 32-bit indices");
            const int ge = la_decompose_gpu(n, A->row_ptr, A->col_idx, b, levels, seed, band, homes, home_levels, H, err);
            if (ge) return fail(ge == 2 ? ARROW_E_NOT_SYMMETRIC : ARROW_E_CUDA, err);
        } else if (la_decompose(n, A->row_ptr, A->col_idx, b, levels, seed, band, homes, home_levels, H, err)) {
            return fail(ARROW_E_INVALID_ARG, err);
        }
        const auto t2 = std::chrono::steady_clock::now();
        if (std::getenv("ARROW_DECOMPOSE_TRACE"))
            fprintf(stderr, "[arrow decompose] %s: checks %.1f ms, LA-Decompose %.1f ms\n", on_gpu ? "gpu" : "host",
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
        if (!H.residual.empty() && !keep_residual)
            return fail(ARROW_E_LEVELS, "levels cap " + std::to_string(levels) + " reached with " +
                                            std::to_string(H.residual.size()) + " entries left");
        auto value = [&](uint32_t e) -> double {
            return A->dtype == ARROW_F64 ? ((const double *)A->values)[e] : (double)((const float *)A->values)[e];
        };
        for (auto &L : H.levels) {
            L.val.resize(L.src.size());
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < (int64_t)L.src.size(); ++t) L.val[t] = value(L.src[t]);
            L.src.clear();
            L.src.shrink_to_fit();
        }
        std::vector<uint32_t> r(H.residual);
        std::sort(r.begin(), r.end());  // CSR order: rows then columns ascending
        int64_t row = 0;
        for (uint32_t e : r) {
            while (A->row_ptr[row + 1] <= (int64_t)e) ++row;
            D->res_u.push_back((int32_t)row);
            D->res_v.push_back(A->col_idx[e]);
            D->res_a.push_back(value(e));
        }
        for (int64_t v = 0; v < n; ++v) D->isolated += (A->row_ptr[v + 1] == A->row_ptr[v]) ? 1 : 0;
        D->levels = std::move(H.levels);
        D->homes = H.homes;
        D->home_levels = H.home_levels;
        D->home_los = std::move(H.home_los);
    } catch (const std::bad_alloc &) {
        D.reset();
        return fail(ARROW_E_NOMEM, "host allocation failed during decomposition");
    }
    D->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return ARROW_OK;
}

// Structural checks of a decomposition before a plan is built from it (a loaded file is only
// checksummed): every perm_i injective into [0, n), sizes ordered n_i <= rows_i <= n and
// head_i <= n_i, CSR offsets from 0 nondecreasing to nnz_i, positions in [0, rows_i), residual
// entries in [0, n).  Returns 0 if valid, else 1 with `err` set.
static int validate_decomposition(const arrow_decomposition_s &D, std::string &err) {
    const int64_t n = D.n;
    std::vector<int32_t> seen((size_t)std::max<int64_t>(n, 0), -1);
    for (size_t i = 0; i < D.levels.size(); ++i) {
        const HostLevel &L = D.levels[i];
        const std::string at = "level " + std::to_string(i) + ": ";
        if (L.rows < 0 || L.rows > n || L.n_i < 0 || L.n_i > L.rows || L.head < 0 || L.head > L.n_i) {
            err = at + "sizes out of range";
            return 1;
        }
        if ((int64_t)L.perm.size() != L.rows || (int64_t)L.row_ptr.size() != L.rows + 1 || L.row_ptr[0] != 0) {
            err = at + "array sizes";
            return 1;
        }
        for (int64_t p = 0; p < L.rows; ++p) {
            const int32_t v = L.perm[p];
            if (v < 0 || v >= n || seen[v] == (int32_t)i) {
                err = at + "perm is not injective into [0, n)";
                return 1;
            }
            seen[v] = (int32_t)i;
            if (L.row_ptr[p + 1] < L.row_ptr[p]) {
                err = at + "row_ptr decreases";
                return 1;
            }
        }
        if (L.row_ptr[L.rows] != (int64_t)L.col.size() || L.col.size() != L.val.size()) {
            err = at + "row_ptr[rows] != nnz";
            return 1;
        }
        for (int32_t q : L.col)
            if (q < 0 || q >= L.rows) {
                err = at + "column position out of range";
                return 1;
            }
    }
    if (D.res_u.size() != D.res_v.size() || D.res_u.size() != D.res_a.size()) {
        err = "residual array sizes";
        return 1;
    }
    if (D.homes < 1 || D.homes > 8) {
        err = "homes out of range";
        return 1;
    }
    auto ranges_ok = [&](const std::vector<int64_t> &r, int64_t lo, int64_t hi) {
        if ((int)r.size() != D.homes + 1 || r[0] != lo || r[D.homes] != hi) return false;
        for (int g = 0; g < D.homes; ++g)
            if (r[g] > r[g + 1]) return false;
        return true;
    };
    if (D.homes > 1) {
        if (!D.levels.empty() && !ranges_ok(D.home_los, 0, n)) {
            err = "home ranges";
            return 1;
        }
        if (D.home_levels < 1) {
            err = "home_levels";
            return 1;
        }
        for (size_t i = 1; i < D.levels.size(); ++i)
            if ((int64_t)i <= D.home_levels ? !ranges_ok(D.levels[i].home_start, D.levels[i].head, D.levels[i].n_i)
                                            : !D.levels[i].home_start.empty()) {
                err = "level " + std::to_string(i) + ": home starts";
                return 1;
            }
    }
    for (size_t t = 0; t < D.res_u.size(); ++t)
        if (D.res_u[t] < 0 || D.res_u[t] >= n || D.res_v[t] < 0 || D.res_v[t] >= n) {
            err = "residual entry out of range";
            return 1;
        }
    return 0;
}

// Single-GPU schedule, level by level (default): K-A level 0 stores every Y row it owns, then one
// K-A launch per level >= 1 adds its rows into Y (read-modify-write, in level order) -- Alg. 2's
// reverse aggregation with the permutations folded into the output rows (S4, S5).
static arrow_status build_single_gpu(arrow_plan P, std::vector<BuiltLevel> &built, int bs) {
    const size_t es = P->esize();
    const size_t nlv = built.size();
    {
        const BuiltLevel &B = built[0];
        const int64_t zb = align_up(std::max<int64_t>((int64_t)B.zero_rows.size() * 4, 1), 256);
        const int64_t total = zb + align_up((int64_t)(nlv + 1) * 4, 256);
        cudaError_t e = cudaMalloc(&P->arena, (size_t)total);
        if (e != cudaSuccess) return fail(ARROW_E_CUDA, std::string("cudaMalloc(plan arena): ") + cudaGetErrorString(e));
        P->arena_bytes = total;
        for (size_t li = 0; li < nlv; ++li) {
            DeviceLevel L = P->meta[li];
            L.zero_rows = reinterpret_cast<int32_t *>(P->arena);
            L.nzero = li == 0 ? (int64_t)B.zero_rows.size() : 0;
            P->levels.push_back(L);
        }
        CUDA_TRY(cudaMemcpy(P->arena, B.zero_rows.data(), B.zero_rows.size() * 4, cudaMemcpyHostToDevice));
        P->counters = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(P->arena) + zb);
    }
    // the last launch writing each Y row: 2 * level + (1 if as a head-row partial); a body segment in
    // its row's last launch is final (kFinalBit: arrow_spmm_iterate applies the activation when it is
    // flushed); rows last written by head partials get a post pass
    // (deterministic mode: every head partial is added by the one K-C pass after the last level)
    std::vector<int32_t> last((size_t)P->n, -1);
    for (size_t li = 0; li < nlv; ++li)
        for (const uint32_t key : built[li].keys)
            if (key & kPseudoRec) {
                const int32_t w = (key & kAuxRec) ? (int32_t)(P->det ? 2 * nlv + 1 : 2 * li + 1) : (int32_t)(2 * li);
                int32_t &l = last[key & (kAuxRec - 1)];
                l = std::max(l, w);
            }
    std::vector<int32_t> post_rows;
    for (int64_t r = 0; r < P->n; ++r)
        if (last[r] >= 0 && (last[r] & 1)) post_rows.push_back((int32_t)r);
    // deterministic head partials (ARROW_FLAG_DETERMINISTIC): chunk c of head row j of level i is
    // stored into its own slot (level i's slots follow level i-1's); after the last level one K-C pass
    // adds every row's slots into Y in a fixed order (by level, then chunk) -- addition order is all
    // determinism needs, so the partials of all levels are combined once instead of per level
    int64_t slot_base = 0;
    struct HeadSlots { int32_t row; int64_t a, b; };
    std::vector<HeadSlots> hslots;
    for (size_t li = 0; li < nlv; ++li) {
        BuiltLevel &B = built[li];
        HostSegs hs;
        hs.ent_val.reserve(B.vals.size());
        std::vector<int64_t> nchunk, hstart;
        std::vector<int32_t> hrows;
        std::vector<int32_t> hidx;  // row -> head index of this level
        if (P->det) {
            hidx.assign((size_t)P->n, -1);
            for (const uint32_t key : B.keys)
                if ((key & kPseudoRec) && (key & kAuxRec)) {
                    const uint32_t row = key & (kAuxRec - 1);
                    if (hidx[row] < 0) {
                        hidx[row] = (int32_t)hrows.size();
                        hrows.push_back((int32_t)row);
                        nchunk.push_back(0);
                    }
                    ++nchunk[hidx[row]];
                }
            hstart.assign(hrows.size() + 1, slot_base);
            for (size_t j = 0; j < hrows.size(); ++j) hstart[j + 1] = hstart[j] + nchunk[j];
            std::fill(nchunk.begin(), nchunk.end(), 0);
            for (size_t j = 0; j < hrows.size(); ++j) hslots.push_back(HeadSlots{hrows[j], hstart[j], hstart[j + 1]});
            slot_base = hstart.back();
            if (slot_base >= ((int64_t)1 << 31)) return fail(ARROW_E_UNSUPPORTED, "too many head-row chunks");
        }
        for (size_t r = 0; r < B.keys.size(); ++r) {
            const uint32_t key = B.keys[r];
            if (key & kPseudoRec) {
                const uint32_t row = key & (kAuxRec - 1);
                const bool fin = !(key & kAuxRec) && last[row] == (int32_t)(2 * li);
                if (P->det && (key & kAuxRec)) {
                    const int32_t j = hidx[row];
                    hs.seg_out.push_back((int32_t)(kFlag | (uint32_t)(hstart[j] + nchunk[j]++)));
                } else {
                    hs.seg_out.push_back((int32_t)(((key & kAuxRec) ? kFlag : 0u) | (fin ? kFinalBit : 0u) | row));
                }
                hs.seg_end.push_back((uint32_t)hs.ent_col.size());
            } else {
                hs.ent_col.push_back((int32_t)(key & (kAuxRec - 1)));
                hs.ent_val.insert(hs.ent_val.end(), B.vals.begin() + r * es, B.vals.begin() + (r + 1) * es);
            }
        }
        std::vector<uint32_t>().swap(B.keys);
        std::vector<uint8_t>().swap(B.vals);
        SegLevel S;
        std::string err;
        const int e = upload_seg_level(hs, (int)es, bs, li == 0 ? 0 : 1, P->n, P->seg_allocs, S, err);
        if (e) return fail(e == -1 ? ARROW_E_UNSUPPORTED : ARROW_E_CUDA, err);
        P->seg.push_back(S);
    }
    if (P->det && !hslots.empty()) {  // K-C: slots -> groups of kDetGroup -> head rows, in a fixed order
        std::stable_sort(hslots.begin(), hslots.end(), [](const HeadSlots &x, const HeadSlots &y) { return x.row < y.row; });
        std::vector<int32_t> gptr(1, 0), gsrc, gdst, ptr(1, 0), src, rows;
        gsrc.reserve((size_t)slot_base);
        for (size_t t = 0; t < hslots.size();) {
            const int32_t row = hslots[t].row;
            int32_t in_group = 0;
            for (; t < hslots.size() && hslots[t].row == row; ++t)
                for (int64_t sl = hslots[t].a; sl < hslots[t].b; ++sl) {
                    if (in_group == 0) {
                        src.push_back((int32_t)gdst.size());
                        gdst.push_back((int32_t)gdst.size());
                        gptr.push_back(gptr.back());
                    }
                    gsrc.push_back((int32_t)sl);
                    ++gptr.back();
                    in_group = (in_group + 1) % kDetGroup;
                }
            rows.push_back(row);
            ptr.push_back((int32_t)src.size());
        }
        DetLevel &K = P->det_kc;
        K.nh = (int64_t)rows.size();
        K.ng = (int64_t)gdst.size();
        P->det_slots = slot_base;
        P->det_groups = K.ng;
        auto up = [&](const std::vector<int32_t> &v) -> int32_t * {
            void *d = nullptr;
            if (cudaMalloc(&d, std::max<size_t>(v.size() * 4, 16)) != cudaSuccess) return nullptr;
            P->seg_allocs.push_back(d);
            if (!v.empty() && cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
            return (int32_t *)d;
        };
        K.ptr = up(ptr);
        K.src = up(src);
        K.rows = up(rows);
        K.gptr = up(gptr);
        K.gsrc = up(gsrc);
        K.gdst = up(gdst);
        if (!K.ptr || !K.src || !K.rows || !K.gptr || !K.gsrc || !K.gdst)
            return fail(ARROW_E_CUDA, "upload of the head-combine lists failed");
    }
    P->n_post = (int64_t)post_rows.size();
    if (P->n_post) {
        CUDA_TRY(cudaMalloc(&P->post_rows, post_rows.size() * 4));
        CUDA_TRY(cudaMemcpy(P->post_rows, post_rows.data(), post_rows.size() * 4, cudaMemcpyHostToDevice));
    }
    return ARROW_OK;
}

static arrow_status plan_from(const arrow_decomposition_s &D, const arrow_options *opt_in, arrow_dtype default_dt,
                              arrow_comm comm, arrow_plan *out) {
    const auto t0 = std::chrono::steady_clock::now();
    arrow_options opt;
    arrow_options_default(&opt);
    if (opt_in) opt = *opt_in;
    if ((int)opt.compute != -1 && opt.compute != ARROW_F32 && opt.compute != ARROW_F64)
        return fail(ARROW_E_INVALID_ARG, "bad options.compute");
    const arrow_dtype pdt = (opt.compute == ARROW_F32 || opt.compute == ARROW_F64) ? opt.compute : default_dt;
    if (opt.order != ARROW_ORDER_ORIGINAL && opt.order != ARROW_ORDER_PERMUTED)
        return fail(ARROW_E_INVALID_ARG, "bad options.order");
    if (opt.window_rows < 0 || opt.head_chunk < 0 || opt.batch_segments < 0)
        return fail(ARROW_E_INVALID_ARG, "negative window/chunk/batch");
    if (opt.batch_segments != 0 && opt.batch_segments != kDefaultBatchSegs)
        return fail(ARROW_E_INVALID_ARG, "options.batch_segments must be 0 or 16");
    if ((opt.flags & ~ARROW_FLAGS_ALL) != 0) return fail(ARROW_E_INVALID_ARG, "unknown options.flags bits");
    if (opt.transport < ARROW_TRANSPORT_AUTO || opt.transport > ARROW_TRANSPORT_NCCL)
        return fail(ARROW_E_INVALID_ARG, "bad options.transport");
    const int64_t window_rows = opt.window_rows > 0 ? opt.window_rows : kDefaultWindowRows;
    // deterministic head partials: one slot per chunk; longer chunks (fewer slots for K-C to add) but
    // not one chunk per (head row, window), which made a hub's whole window one warp's serial work
    // (config R level 0: 10.7 vs 1.6 ms)
    const bool det = (opt.flags & ARROW_FLAG_DETERMINISTIC) && !comm;
    const int32_t head_chunk = opt.head_chunk > 0 ? opt.head_chunk : det ? kDetHeadChunk : kDefaultHeadChunk;
    const int bs = opt.batch_segments > 0 ? opt.batch_segments : kDefaultBatchSegs;
    const int order = comm ? ARROW_ORDER_PERMUTED : opt.order;
    const int64_t n = D.n, b = D.b;
    if (n >= kMaxRows) return fail(ARROW_E_UNSUPPORTED, "n must be < 2^30 (30-bit row keys)");
    if (std::string e; validate_decomposition(D, e)) return fail(ARROW_E_INVALID_ARG, "invalid decomposition: " + e);

    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::unique_ptr<arrow_plan_s> P;
    std::vector<BuiltLevel> built;
    std::vector<int32_t> pos0;
    const std::vector<int32_t> *pos0p = nullptr;
    try {
        P.reset(new arrow_plan_s());
        P->device = dev;
        CUDA_TRY(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, dev));
        P->dtype = pdt;
        P->order = order;
        P->n = n;
        P->b = b;
        P->isolated = D.isolated;
        P->use_graphs = (opt.flags & ARROW_FLAG_NO_GRAPHS) == 0;
        P->det = (opt.flags & ARROW_FLAG_DETERMINISTIC) != 0 && !comm;
        P->transport = opt.transport;
        P->nnz = (int64_t)D.res_u.size();
        for (auto &L : D.levels) P->nnz += L.row_ptr[L.rows];
        if (order == ARROW_ORDER_PERMUTED && !D.levels.empty()) {
            pos0.assign(n, 0);
            for (int64_t p = 0; p < n; ++p) pos0[D.levels[0].perm[p]] = (int32_t)p;
            pos0p = &pos0;
        }
        built.resize(D.levels.size() + (D.res_u.empty() ? 0 : 1));
        // default window: level 0 (store-only, gather-bound) runs faster with a larger window, the
        // read-modify-write levels with 16,384 rows (profiles/r02/win/)
        for (size_t i = 0; i < D.levels.size(); ++i)
            build_level(D.levels[i], (int)i, b,
                        (i == 0 && opt.window_rows == 0) ? std::max(window_rows, kDefaultLevel0WindowRows) : window_rows,
                        head_chunk, pos0p, pdt, comm ? 1 : 0, built[i]);
        if (!D.res_u.empty()) build_residual(D, pos0p, pdt, built.back());
        P->residual_nnz = (int64_t)D.res_u.size();
        P->arrow_levels = (int32_t)D.levels.size();
        P->host_levels.resize(D.levels.size());
        P->host_level_vals.resize(D.levels.size());
        for (size_t i = 0; i < D.levels.size(); ++i) {
            const HostLevel &L = D.levels[i];
            HostLevel &C = P->host_levels[i];
            C.rows = L.rows; C.n_i = L.n_i; C.head = L.head;
            C.perm = L.perm; C.row_ptr = L.row_ptr; C.col = L.col;
            auto &hv = P->host_level_vals[i];
            hv.resize(L.val.size() * P->esize());
            for (size_t t = 0; t < L.val.size(); ++t) put_val(hv, (int64_t)t, pdt, L.val[t]);
        }
    } catch (const std::bad_alloc &) {
        return fail(ARROW_E_NOMEM, "host allocation failed during layout build");
    }

    // algorithmic bytes model
    {
        const int64_t s = (int64_t)P->esize();
        for (size_t i = 0; i < built.size(); ++i) {
            const BuiltLevel &B = built[i];
            P->bytes_alg_fixed += B.nnz * (s + 4) + (B.rows + 1) * 8 + B.rows * 4;
            P->bytes_alg_rows += B.n_i + (i == 0 ? 0 : 2 * B.n_i);
            P->sum_rows += (i < (size_t)P->arrow_levels) ? B.n_i : 0;
            P->max_head = std::max(P->max_head, B.head);
        }
        P->bytes_alg_rows += n;  // level-0 store of every Y row
    }

    // per-level metadata (introspection; single GPU: also the launch list)
    for (const BuiltLevel &B : built) {
        DeviceLevel L;
        L.rows = B.rows; L.n_i = B.n_i; L.head = B.head; L.nnz = B.nnz; L.head_nnz = B.head_nnz;
        L.tiles = B.tiles; L.nseg = B.nseg; L.mode = B.mode;
        L.nzero = (int64_t)B.zero_rows.size();
        P->meta.push_back(L);
    }

    if (!comm && !built.empty()) {
        arrow_status st = build_single_gpu(P.get(), built, bs);
        if (st != ARROW_OK) return st;
    }
    P->local_begin = 0;
    P->local_end = n;
    if (comm) {
        P->comm = comm;
        // level 0 keeps 16,384-row windows here: a rank's level-0 range is 1/G of the rows, and 65,536
        // measured +1 % at G = 4 (profiles/r02/win_dist/)
        arrow_status cs = dist_build(P.get(), D, comm, window_rows, window_rows, head_chunk, bs);
        if (cs != ARROW_OK) return cs;
    }
    P->create_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = P.release();
    return ARROW_OK;
}

arrow_status arrow_plan_create_ex(const arrow_csr *A, int64_t b, int32_t levels, const arrow_options *opt_in,
                                  arrow_comm comm, arrow_plan *out) {
    g_err.clear();
    if (!out) return fail(ARROW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    arrow_options opt;
    arrow_options_default(&opt);
    if (opt_in) opt = *opt_in;
    if (opt.residual != ARROW_RESIDUAL_ERROR && opt.residual != ARROW_RESIDUAL_CSR)
        return fail(ARROW_E_INVALID_ARG, "bad options.residual");
    std::unique_ptr<arrow_decomposition_s> D;
    if (opt.flags & ~ARROW_FLAGS_ALL) return fail(ARROW_E_INVALID_ARG, "bad options.flags");
    int32_t homes = 1;
    if ((opt.flags & ARROW_FLAG_HOME_AWARE) && comm) homes = comm->nranks;
    arrow_status st = decompose_impl(A, b, levels, opt.seed, opt.residual == ARROW_RESIDUAL_CSR, opt.band, homes,
                                     opt.home_levels, (opt.flags & ARROW_FLAG_GPU_DECOMPOSE) != 0, D);
    if (st != ARROW_OK) return st;
    st = plan_from(*D, &opt, A->dtype, comm, out);
    if (st == ARROW_OK) (*out)->create_seconds += D->seconds;
    return st;
}

arrow_status arrow_plan_create_from(arrow_decomposition d, const arrow_options *opt, arrow_comm comm, arrow_plan *out) {
    g_err.clear();
    if (!out) return fail(ARROW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!d) return fail(ARROW_E_INVALID_ARG, "decomposition is NULL");
    return plan_from(*d, opt, ARROW_F64, comm, out);
}

arrow_status arrow_decompose(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                             arrow_decomposition *out) {
    return arrow_decompose_ex(A, b, levels, seed, keep_residual, ARROW_BAND_BLOCK, out);
}

arrow_status arrow_decompose_ex(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                int32_t band, arrow_decomposition *out) {
    g_err.clear();
    if (!out) return fail(ARROW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    std::unique_ptr<arrow_decomposition_s> D;
    arrow_status st = decompose_impl(A, b, levels, seed, keep_residual != 0, band, 1, 0, false, D);
    if (st != ARROW_OK) return st;
    *out = D.release();
    return ARROW_OK;
}

arrow_status arrow_decompose_gpu(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                 int32_t band, arrow_decomposition *out) {
    g_err.clear();
    if (!out) return fail(ARROW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    std::unique_ptr<arrow_decomposition_s> D;
    arrow_status st = decompose_impl(A, b, levels, seed, keep_residual != 0, band, 1, 0, true, D);
    if (st != ARROW_OK) return st;
    *out = D.release();
    return ARROW_OK;
}

arrow_status arrow_decompose_homes(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                   int32_t band, int32_t homes, int32_t home_levels, int32_t device,
                                   arrow_decomposition *out) {
    g_err.clear();
    if (!out) return fail(ARROW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (device != 0 && device != 1) return fail(ARROW_E_INVALID_ARG, "device must be 0 (host) or 1 (CUDA)");
    std::unique_ptr<arrow_decomposition_s> D;
    arrow_status st = decompose_impl(A, b, levels, seed, keep_residual != 0, band, homes, home_levels, device == 1, D);
    if (st != ARROW_OK) return st;
    *out = D.release();
    return ARROW_OK;
}

arrow_status arrow_decomposition_homes(arrow_decomposition d, int32_t level, int32_t *homes, int32_t *home_levels,
                                       int64_t *ranges) {
    if (!d) return fail(ARROW_E_INVALID_ARG, "decomposition is NULL");
    if (level < -1 || level >= (int32_t)d->levels.size()) return fail(ARROW_E_INVALID_ARG, "level out of range");
    if (homes) *homes = d->homes;
    if (home_levels) *home_levels = d->home_levels;
    if (ranges && d->homes > 1) {
        const std::vector<int64_t> &r = level == -1 ? d->home_los : d->levels[level].home_start;
        if (r.size() != (size_t)d->homes + 1)
            return fail(ARROW_E_INVALID_ARG, "level " + std::to_string(level) + " is not home-aware (levels 1.." +
                                                 std::to_string(d->home_levels) + " are; -1: pi_0 ranges)");
        std::memcpy(ranges, r.data(), r.size() * 8);
    }
    return ARROW_OK;
}

arrow_status arrow_decomposition_destroy(arrow_decomposition d) {
    delete d;
    return ARROW_OK;
}

arrow_status arrow_decomposition_info(arrow_decomposition d, int64_t *n, int64_t *b, int32_t *levels,
                                      int64_t *residual_nnz) {
    if (!d) return fail(ARROW_E_INVALID_ARG, "decomposition is NULL");
    if (n) *n = d->n;
    if (b) *b = d->b;
    if (levels) *levels = (int32_t)d->levels.size();
    if (residual_nnz) *residual_nnz = (int64_t)d->res_u.size();
    return ARROW_OK;
}

arrow_status arrow_decomposition_level_info(arrow_decomposition d, int32_t level, arrow_level_info_t *info) {
    if (!d || !info) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    if (level < 0 || level >= (int32_t)d->levels.size()) return fail(ARROW_E_INVALID_ARG, "level out of range");
    const HostLevel &L = d->levels[level];
    std::memset(info, 0, sizeof(*info));
    info->rows = L.rows;
    info->n_i = L.n_i;
    info->head = L.head;
    info->nnz = L.row_ptr[L.rows];
    info->head_nnz = L.row_ptr[L.head];
    info->tiles = (L.n_i + d->b - 1) / d->b;
    return ARROW_OK;
}

arrow_status arrow_decomposition_export_level(arrow_decomposition d, int32_t level, int32_t *perm, int64_t *row_ptr,
                                              int32_t *col, double *val) {
    if (!d) return fail(ARROW_E_INVALID_ARG, "decomposition is NULL");
    if (level < 0 || level >= (int32_t)d->levels.size()) return fail(ARROW_E_INVALID_ARG, "level out of range");
    const HostLevel &L = d->levels[level];
    if (perm) std::memcpy(perm, L.perm.data(), L.perm.size() * 4);
    if (row_ptr) std::memcpy(row_ptr, L.row_ptr.data(), L.row_ptr.size() * 8);
    if (col) std::memcpy(col, L.col.data(), L.col.size() * 4);
    if (val) std::memcpy(val, L.val.data(), L.val.size() * 8);
    return ARROW_OK;
}

arrow_status arrow_decomposition_export_residual(arrow_decomposition d, int32_t *u, int32_t *v, double *val) {
    if (!d) return fail(ARROW_E_INVALID_ARG, "decomposition is NULL");
    if (u) std::memcpy(u, d->res_u.data(), d->res_u.size() * 4);
    if (v) std::memcpy(v, d->res_v.data(), d->res_v.size() * 4);
    if (val) std::memcpy(val, d->res_a.data(), d->res_a.size() * 8);
    return ARROW_OK;
}

namespace {
struct Fnv {
    uint64_t h = 1469598103934665603ULL;
    void add(const void *p, size_t n) {
        const uint8_t *b = (const uint8_t *)p;
        for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ULL; }
    }
};
const char kMagic[8] = {'A', 'R', 'W', 'D', 'E', 'C', '0', '3'};   // 03: header + band + homes
const char kMagic2[8] = {'A', 'R', 'W', 'D', 'E', 'C', '0', '2'};  // 02: header + band
const char kMagic1[8] = {'A', 'R', 'W', 'D', 'E', 'C', '0', '1'};  // 01: block band only
}  // namespace

arrow_status arrow_decomposition_save(arrow_decomposition d, const char *path) {
    if (!d || !path) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    FILE *f = std::fopen(path, "wb");
    if (!f) return fail(ARROW_E_INVALID_ARG, std::string("cannot open ") + path);
    Fnv fnv;
    bool ok = true;
    auto w = [&](const void *p, size_t n) {
        if (n == 0) return;
        fnv.add(p, n);
        ok = ok && std::fwrite(p, 1, n, f) == n;
    };
    w(kMagic, 8);
    const int64_t hdr[9] = {d->n, d->b, (int64_t)d->seed, (int64_t)d->levels.size(), (int64_t)d->res_u.size(), d->isolated,
                            (int64_t)d->band, (int64_t)d->homes, (int64_t)d->home_levels};
    w(hdr, sizeof(hdr));
    const bool homes = d->homes > 1 && !d->levels.empty();
    if (homes) w(d->home_los.data(), d->home_los.size() * 8);
    for (size_t i = 0; i < d->levels.size(); ++i) {
        const HostLevel &L = d->levels[i];
        const int64_t lh[4] = {L.rows, L.n_i, L.head, L.row_ptr[L.rows]};
        w(lh, sizeof(lh));
        w(L.perm.data(), L.perm.size() * 4);
        w(L.row_ptr.data(), L.row_ptr.size() * 8);
        w(L.col.data(), L.col.size() * 4);
        w(L.val.data(), L.val.size() * 8);
        if (homes && i > 0 && (int64_t)i <= d->home_levels) w(L.home_start.data(), L.home_start.size() * 8);
    }
    w(d->res_u.data(), d->res_u.size() * 4);
    w(d->res_v.data(), d->res_v.size() * 4);
    w(d->res_a.data(), d->res_a.size() * 8);
    const uint64_t sum = fnv.h;
    ok = ok && std::fwrite(&sum, 1, 8, f) == 8;
    ok = (std::fclose(f) == 0) && ok;
    return ok ? ARROW_OK : fail(ARROW_E_INVALID_ARG, std::string("write failed: ") + path);
}

arrow_status arrow_decomposition_load(const char *path, arrow_decomposition *out) {
    if (!path || !out) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    *out = nullptr;
    FILE *f = std::fopen(path, "rb");
    if (!f) return fail(ARROW_E_INVALID_ARG, std::string("cannot open ") + path);
    Fnv fnv;
    bool ok = true;
    auto r = [&](void *p, size_t n) {
        if (n == 0 || !ok) return;
        ok = std::fread(p, 1, n, f) == n;
        if (ok) fnv.add(p, n);
    };
    std::unique_ptr<arrow_decomposition_s> D;
    try {
        D.reset(new arrow_decomposition_s());
        char magic[8];
        r(magic, 8);
        const int ver = !ok ? 0 : std::memcmp(magic, kMagic1, 8) == 0 ? 1 : std::memcmp(magic, kMagic2, 8) == 0 ? 2
                                      : std::memcmp(magic, kMagic, 8) == 0 ? 3 : 0;
        if (!ver) { std::fclose(f); return fail(ARROW_E_INVALID_ARG, "not an arrow decomposition file"); }
        int64_t hdr[9] = {0, 0, 0, 0, 0, 0, 0, 1, 0};
        r(hdr, (ver == 1 ? 6 : ver == 2 ? 7 : 9) * sizeof(int64_t));
        if (!ok || hdr[0] < 0 || hdr[1] < 2 || hdr[3] < 0 || hdr[4] < 0 || hdr[6] < 0 || hdr[6] > 1 || hdr[7] < 1 ||
            hdr[7] > 8 || hdr[8] < 0 || (hdr[7] > 1) != (hdr[8] > 0)) { std::fclose(f); return fail(ARROW_E_INVALID_ARG, "corrupt header"); }
        D->n = hdr[0]; D->b = hdr[1]; D->seed = (uint64_t)hdr[2]; D->isolated = hdr[5]; D->band = (int32_t)hdr[6];
        D->homes = (int32_t)hdr[7];
        D->home_levels = (int32_t)std::min<int64_t>(hdr[8], 1 << 30);
        D->levels.resize(hdr[3]);
        const bool homes = D->homes > 1 && !D->levels.empty();
        if (homes) {
            D->home_los.resize(D->homes + 1);
            r(D->home_los.data(), D->home_los.size() * 8);
        }
        for (HostLevel &L : D->levels) {
            int64_t lh[4];
            r(lh, sizeof(lh));
            if (!ok || lh[0] < 0 || lh[0] > D->n || lh[3] < 0) { std::fclose(f); return fail(ARROW_E_INVALID_ARG, "corrupt level header"); }
            L.rows = lh[0]; L.n_i = lh[1]; L.head = lh[2];
            L.perm.resize(L.rows); L.row_ptr.resize(L.rows + 1); L.col.resize(lh[3]); L.val.resize(lh[3]);
            r(L.perm.data(), L.perm.size() * 4);
            r(L.row_ptr.data(), L.row_ptr.size() * 8);
            r(L.col.data(), L.col.size() * 4);
            r(L.val.data(), L.val.size() * 8);
            const int64_t li = &L - &D->levels[0];
            if (homes && li > 0 && li <= D->home_levels) {
                L.home_start.resize(D->homes + 1);
                r(L.home_start.data(), L.home_start.size() * 8);
            }
        }
        D->res_u.resize(hdr[4]); D->res_v.resize(hdr[4]); D->res_a.resize(hdr[4]);
        r(D->res_u.data(), D->res_u.size() * 4);
        r(D->res_v.data(), D->res_v.size() * 4);
        r(D->res_a.data(), D->res_a.size() * 8);
    } catch (const std::bad_alloc &) {
        std::fclose(f);
        return fail(ARROW_E_NOMEM, "host allocation failed while loading");
    }
    const uint64_t expect = fnv.h;
    uint64_t sum = 0;
    const bool got = std::fread(&sum, 1, 8, f) == 8;
    std::fclose(f);
    if (!ok || !got || sum != expect) return fail(ARROW_E_INVALID_ARG, "truncated file or checksum mismatch");
    *out = D.release();
    return ARROW_OK;
}

arrow_status arrow_plan_destroy(arrow_plan plan) {
    if (!plan) return ARROW_OK;
    int cur = 0;
    cudaGetDevice(&cur);
    const int dev = plan->device;
    if (cur != dev) cudaSetDevice(dev);
    if (plan->stream) cudaStreamSynchronize(plan->stream);
    else cudaDeviceSynchronize();
    delete plan;
    if (cur != dev) cudaSetDevice(cur);
    return ARROW_OK;
}

arrow_status arrow_plan_set_stream(arrow_plan plan, void *stream) {
    if (!plan) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    plan->stream = reinterpret_cast<cudaStream_t>(stream);
    return ARROW_OK;
}

// k-dependent workspace on one GPU: the head-partial slots of the deterministic mode (det_slots x k)
static arrow_status ensure_ws(arrow_plan P, int64_t k) {
    if (k <= P->ws_k || P->dist || !P->det || P->det_slots == 0) return ARROW_OK;
    if (P->ws) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { P->poisoned = true; return fail(ARROW_E_CUDA, cudaGetErrorString(e)); }
        cudaFree(P->ws);
        P->ws = nullptr;
        P->ws_k = 0;
    }
    cudaError_t e = cudaMalloc(&P->ws, (size_t)((P->det_slots + P->det_groups) * k * (int64_t)P->esize()));
    if (e != cudaSuccess) return fail(ARROW_E_CUDA, std::string("cudaMalloc(head-partial slots): ") + cudaGetErrorString(e));
    P->ws_k = k;
    return ARROW_OK;
}

arrow_status arrow_plan_reserve(arrow_plan plan, int64_t k_max) {
    if (!plan) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (k_max < 0) return fail(ARROW_E_INVALID_ARG, "k_max < 0");
    int cur = 0;
    CUDA_TRY(cudaGetDevice(&cur));
    if (cur != plan->device) return fail(ARROW_E_STATE, "plan used from another device");
    return ensure_ws(plan, k_max);
}

namespace {
inline void prof_begin(arrow_plan P, cudaStream_t st, cudaEvent_t &a) {
    if (!P->profiling) return;
    cudaEventCreate(&a);
    cudaEventRecord(a, st);
}
inline void prof_end(arrow_plan P, cudaStream_t st, int kid, cudaEvent_t a) {
    if (!P->profiling) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, st);
    P->prof.push_back(ProfRec{kid, P->prof_pos++, a, b});
}
}  // namespace

static arrow_status enqueue_rmw(arrow_plan P, const void *X, void *Y, int64_t k, cudaStream_t st, int act) {
    const int dt = P->dtype == ARROW_F64 ? 1 : 0;
    CUDA_TRY(cudaMemsetAsync(P->counters, 0, P->levels.size() * sizeof(unsigned), st));
    for (size_t i = 0; i < P->levels.size(); ++i) {
        const DeviceLevel &L = P->levels[i];
        cudaEvent_t a = nullptr;
        int e = 0;
        // level 0's head rows start at zero (its head-row slices add into them); its entry-less rows
        // are zeroed inside K-A level 0, a share per batch grab
        const int64_t nh = i == 0 ? std::min<int64_t>(L.head, L.nzero) : 0;
        if (nh > 0) {
            prof_begin(P, st, a);
            e = launch_zero_rows(dt, L.zero_rows, nh, k, Y, st);
            prof_end(P, st, ARROW_K_HEAD_STAGE, a);
            if (e) { P->poisoned = true; return fail(ARROW_E_CUDA, std::string("K-Z: ") + cudaGetErrorString((cudaError_t)e)); }
        }
        prof_begin(P, st, a);
        e = launch_seg(dt, 0, P->seg[i], X, nullptr, Y, P->det ? P->ws : nullptr, k, P->num_sms, P->counters + i, st,
                       P->launch, nullptr, act, i == 0 ? L.zero_rows + nh : nullptr, i == 0 ? L.nzero - nh : 0);
        prof_end(P, st, ARROW_K_SEGMENTS, a);
        if (e) { P->poisoned = true; return fail(ARROW_E_CUDA, std::string("K-A: ") + cudaGetErrorString((cudaError_t)e)); }
    }
    if (P->det && P->det_kc.nh > 0) {  // S3, K-C: Y[head] += its chunk partials of every level, in order
        const DetLevel &K = P->det_kc;
        cudaEvent_t a = nullptr;
        prof_begin(P, st, a);
        char *groups = reinterpret_cast<char *>(P->ws) + (size_t)(P->det_slots * k * (int64_t)P->esize());
        int e = (int)cudaMemsetAsync(groups, 0, (size_t)(K.ng * k * (int64_t)P->esize()), st);
        if (!e) e = launch_gather_add(dt, P->ws, K.gptr, K.gsrc, K.gdst, K.ng, k, groups, st);
        if (!e) e = launch_gather_add(dt, groups, K.ptr, K.src, K.rows, K.nh, k, Y, st);
        prof_end(P, st, ARROW_K_HEAD_EPI, a);
        if (e) { P->poisoned = true; return fail(ARROW_E_CUDA, std::string("K-C: ") + cudaGetErrorString((cudaError_t)e)); }
    }
    if (act && P->n_post) {  // iterate mode: rows last written by head-row partials
        const int e = launch_act_rows(dt, P->post_rows, P->n_post, k, act, Y, st);
        if (e) { P->poisoned = true; return fail(ARROW_E_CUDA, std::string("activation pass: ") + cudaGetErrorString((cudaError_t)e)); }
    }
    return ARROW_OK;
}

static arrow_status enqueue_single(arrow_plan P, const void *X, void *Y, int64_t k, cudaStream_t st, int act = 0) {
    if (P->profiling) P->prof_acc.calls += 1;
    P->prof_pos = 0;
    return enqueue_rmw(P, X, Y, k, st, act);
}

arrow_status arrow_spmm_ex(arrow_plan P, const void *X, void *Y, int64_t k, void *stream) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (P->poisoned) return fail(ARROW_E_STATE, "plan poisoned by an earlier CUDA error");
    if (k < 0) return fail(ARROW_E_INVALID_ARG, "k < 0");
    if (k == 0 || P->n == 0) return ARROW_OK;
    const int64_t rows = P->local_end - P->local_begin;
    // a rank of a distributed plan may own no rows but must still take part in the collectives
    if ((!X || !Y) && !(P->dist && rows == 0)) return fail(ARROW_E_INVALID_ARG, "X or Y is NULL");
    int cur = 0;
    CUDA_TRY(cudaGetDevice(&cur));
    if (cur != P->device) return fail(ARROW_E_STATE, "plan used from another device");
    if (k * (int64_t)P->esize() >= ((int64_t)1 << 32)) return fail(ARROW_E_UNSUPPORTED, "row of X exceeds 4 GiB");
    const int64_t bytes = rows * k * (int64_t)P->esize();
    const char *xa = (const char *)X, *ya = (const char *)Y;
    if (rows > 0 && xa < ya + bytes && ya < xa + bytes) return fail(ARROW_E_INVALID_ARG, "X and Y overlap");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (P->dist) return dist_spmm(P, X, Y, k, st);
    if (P->levels.empty()) {
        int e = launch_zero(Y, bytes, st);
        if (e) return fail(ARROW_E_CUDA, cudaGetErrorString((cudaError_t)e));
        return ARROW_OK;
    }
    // Single GPU: the whole call (memset, K-Z, one K-A launch per level) is captured once into a CUDA
    // graph per (X, Y, k, stream) and replayed.  Not while profiling (per-kernel events), on the
    // legacy stream, or when the caller is itself capturing `st` (its graph then receives the
    // kernels directly).
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (st != nullptr) CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    if (P->det && P->ws_k < k) {
        if (cap != cudaStreamCaptureStatusNone)
            return fail(ARROW_E_STATE, "workspace for this k not reserved before stream capture (arrow_plan_reserve)");
        arrow_status ws = ensure_ws(P, k);
        if (ws != ARROW_OK) return ws;
    }
    if (P->use_graphs && !P->profiling && !P->no_graph && st != nullptr && cap == cudaStreamCaptureStatusNone) {
        if (P->gexec && P->g_x == X && P->g_y == Y && P->g_k == k && P->g_stream == st) {
            CUDA_TRY(cudaGraphLaunch(P->gexec, st));
            return ARROW_OK;
        }
        if (P->gexec) {
            cudaGraphExecDestroy(P->gexec);
            P->gexec = nullptr;
        }
        CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        arrow_status s = enqueue_single(P, X, Y, k, st);
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (s != ARROW_OK) {
            if (graph) cudaGraphDestroy(graph);
            return s;
        }
        if (ce != cudaSuccess) return fail(ARROW_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        ce = cudaGraphInstantiate(&P->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) {
            P->gexec = nullptr;
            return fail(ARROW_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
        }
        P->g_x = X;
        P->g_y = Y;
        P->g_k = k;
        P->g_stream = st;
        CUDA_TRY(cudaGraphLaunch(P->gexec, st));
        return ARROW_OK;
    }
    return enqueue_single(P, X, Y, k, st);
}

arrow_status arrow_spmm(arrow_plan plan, const void *X, void *Y, int64_t k) {
    if (!plan) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    return arrow_spmm_ex(plan, X, Y, k, plan->stream);
}

arrow_status arrow_spmm_iterate(arrow_plan P, void *X, void *Y, int64_t k, int32_t iters, int32_t activation,
                                void *stream, int32_t *result_in_y) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (P->poisoned) return fail(ARROW_E_STATE, "plan poisoned by an earlier CUDA error");
    if (iters < 1) return fail(ARROW_E_INVALID_ARG, "iters < 1");
    if (activation < ARROW_ACT_NONE || activation > ARROW_ACT_RELU) return fail(ARROW_E_INVALID_ARG, "unknown activation");
    if (P->dist) return fail(ARROW_E_UNSUPPORTED, "arrow_spmm_iterate: distributed plans are not supported");
    if (P->seg.empty() && !P->levels.empty())
        return fail(ARROW_E_UNSUPPORTED, "arrow_spmm_iterate needs the segment-descriptor layout (default)");
    if (k < 0) return fail(ARROW_E_INVALID_ARG, "k < 0");
    if (result_in_y) *result_in_y = (iters & 1) ? 1 : 0;
    if (k == 0 || P->n == 0) return ARROW_OK;
    if (!X || !Y) return fail(ARROW_E_INVALID_ARG, "X or Y is NULL");
    const int64_t bytes = P->n * k * (int64_t)P->esize();
    const char *xa = (const char *)X, *ya = (const char *)Y;
    if (xa < ya + bytes && ya < xa + bytes) return fail(ARROW_E_INVALID_ARG, "X and Y overlap");
    int cur = 0;
    CUDA_TRY(cudaGetDevice(&cur));
    if (cur != P->device) return fail(ARROW_E_STATE, "plan used from another device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    arrow_status ws = ensure_ws(P, k);
    if (ws != ARROW_OK) return ws;
    for (int32_t t = 0; t < iters; ++t) {  // X_{t+1} = act(A X_t), ping-pong between X and Y
        const void *src = (t & 1) ? Y : X;
        void *dst = (t & 1) ? X : Y;
        if (P->levels.empty()) {
            CUDA_TRY(cudaMemsetAsync(dst, 0, (size_t)bytes, st));
            continue;
        }
        arrow_status s = enqueue_single(P, src, dst, k, st, activation);
        if (s != ARROW_OK) return s;
    }
    return ARROW_OK;
}

arrow_status arrow_spmm_host(arrow_plan P, const void *Xh, void *Yh, int64_t k, void *stream) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (k < 0) return fail(ARROW_E_INVALID_ARG, "k < 0");
    if (k == 0 || P->n == 0) return ARROW_OK;
    if (!Xh || !Yh) return fail(ARROW_E_INVALID_ARG, "X or Y is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t rows = P->local_end - P->local_begin;
    const int64_t bytes = rows * k * (int64_t)P->esize();
    if (k > P->host_k) {
        if (P->host_x) { cudaFree(P->host_x); P->host_x = nullptr; }
        if (P->host_y) { cudaFree(P->host_y); P->host_y = nullptr; }
        P->host_k = 0;
        CUDA_TRY(cudaMalloc(&P->host_x, (size_t)std::max<int64_t>(bytes, 1)));
        CUDA_TRY(cudaMalloc(&P->host_y, (size_t)std::max<int64_t>(bytes, 1)));
        P->host_k = k;
    }
    CUDA_TRY(cudaMemcpyAsync(P->host_x, Xh, (size_t)bytes, cudaMemcpyHostToDevice, st));
    arrow_status s = arrow_spmm_ex(P, P->host_x, P->host_y, k, stream);
    if (s != ARROW_OK) return s;
    CUDA_TRY(cudaMemcpyAsync(Yh, P->host_y, (size_t)bytes, cudaMemcpyDeviceToHost, st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { P->poisoned = true; return fail(ARROW_E_CUDA, cudaGetErrorString(e)); }
    return ARROW_OK;
}

arrow_status arrow_spmm_host_batch(arrow_plan P, const void *const *Xh, void *const *Yh, int64_t count, int64_t k,
                                   void *stream) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (count < 0) return fail(ARROW_E_INVALID_ARG, "count < 0");
    if (k < 0) return fail(ARROW_E_INVALID_ARG, "k < 0");
    if (count == 0 || k == 0 || P->n == 0) return ARROW_OK;
    if (!Xh || !Yh) return fail(ARROW_E_INVALID_ARG, "X or Y list is NULL");
    for (int64_t c = 0; c < count; ++c)
        if (!Xh[c] || !Yh[c]) return fail(ARROW_E_INVALID_ARG, "X or Y is NULL");
    if (P->poisoned) return fail(ARROW_E_STATE, "plan poisoned by an earlier CUDA error");
    if (count == 1) {
        for (int64_t c = 0; c < count; ++c) {
            const arrow_status s = arrow_spmm_host(P, Xh[c], Yh[c], k, stream);
            if (s != ARROW_OK) return s;
        }
        return ARROW_OK;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t rows = P->local_end - P->local_begin;
    const size_t bytes = (size_t)(rows * k * (int64_t)P->esize());
    if (k > P->hb_k) {
        CUDA_TRY(cudaDeviceSynchronize());
        for (int i = 0; i < 2; ++i) {
            if (P->hb_x[i]) { cudaFree(P->hb_x[i]); P->hb_x[i] = nullptr; }
            if (P->hb_y[i]) { cudaFree(P->hb_y[i]); P->hb_y[i] = nullptr; }
        }
        P->hb_k = 0;
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaMalloc(&P->hb_x[i], std::max<size_t>(bytes, 1)));
            CUDA_TRY(cudaMalloc(&P->hb_y[i], std::max<size_t>(bytes, 1)));
        }
        P->hb_k = k;
    }
    if (!P->hb_h2d) {
        CUDA_TRY(cudaStreamCreateWithFlags(&P->hb_h2d, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&P->hb_d2h, cudaStreamNonBlocking));
        for (cudaEvent_t &e : P->hb_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaEvent_t *ex = P->hb_ev, *ec = P->hb_ev + 2, *ey = P->hb_ev + 4, e_start = P->hb_ev[6];
    // everything already queued on `stream` comes first
    CUDA_TRY(cudaEventRecord(e_start, st));
    CUDA_TRY(cudaStreamWaitEvent(P->hb_h2d, e_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(P->hb_d2h, e_start, 0));
    // the slots alternate; a graph keyed by (X, Y) would be re-captured every item
    struct NoGraph { arrow_plan p; ~NoGraph() { p->no_graph = false; } } guard{P};
    P->no_graph = true;
    arrow_status status = ARROW_OK;
    for (int64_t c = 0; c < count && status == ARROW_OK; ++c) {
        const int s = (int)(c & 1);
        if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(P->hb_h2d, ec[s], 0));  // kernels of c-2 done reading slot s
        CUDA_TRY(cudaMemcpyAsync(P->hb_x[s], Xh[c], bytes, cudaMemcpyHostToDevice, P->hb_h2d));
        CUDA_TRY(cudaEventRecord(ex[s], P->hb_h2d));
        CUDA_TRY(cudaStreamWaitEvent(st, ex[s], 0));
        if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(st, ey[s], 0));          // Y of c-2 copied out of slot s
        status = arrow_spmm_ex(P, P->hb_x[s], P->hb_y[s], k, stream);
        if (status != ARROW_OK) break;
        CUDA_TRY(cudaEventRecord(ec[s], st));
        CUDA_TRY(cudaStreamWaitEvent(P->hb_d2h, ec[s], 0));
        CUDA_TRY(cudaMemcpyAsync(Yh[c], P->hb_y[s], bytes, cudaMemcpyDeviceToHost, P->hb_d2h));
        CUDA_TRY(cudaEventRecord(ey[s], P->hb_d2h));
    }
    // join both copy streams back into `stream`, then wait for everything
    CUDA_TRY(cudaEventRecord(e_start, P->hb_d2h));
    CUDA_TRY(cudaStreamWaitEvent(st, e_start, 0));
    CUDA_TRY(cudaEventRecord(e_start, P->hb_h2d));
    CUDA_TRY(cudaStreamWaitEvent(st, e_start, 0));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { P->poisoned = true; return fail(ARROW_E_CUDA, cudaGetErrorString(e)); }
    return status;
}

arrow_status arrow_plan_info(arrow_plan P, arrow_plan_info_t *info) {
    if (!P || !info) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    std::memset(info, 0, sizeof(*info));
    info->n = P->n;
    info->nnz = P->nnz;
    info->b = P->b;
    info->levels = P->arrow_levels;
    info->dtype = P->dtype;
    info->order = P->order;
    info->distributed = P->comm ? 1 : 0;
    info->residual_nnz = P->residual_nnz;
    info->sum_rows = P->sum_rows;
    info->isolated = P->isolated;
    info->create_seconds = P->create_seconds;
    info->bytes_alg_fixed = P->bytes_alg_fixed;
    info->bytes_alg_rows = P->bytes_alg_rows;
    info->device_bytes = P->arena_bytes;
    return ARROW_OK;
}

arrow_status arrow_plan_level_info(arrow_plan P, int32_t level, arrow_level_info_t *info) {
    if (!P || !info) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    if (level < 0 || level >= (int32_t)P->meta.size()) return fail(ARROW_E_INVALID_ARG, "level out of range");
    std::memset(info, 0, sizeof(*info));
    const DeviceLevel &L = P->meta[level];
    info->rows = L.rows;
    info->n_i = L.n_i;
    info->head = L.head;
    info->nnz = L.nnz;
    info->head_nnz = L.head_nnz;
    info->tiles = L.tiles;
    info->segments = L.nseg;
    return ARROW_OK;
}

arrow_status arrow_plan_export_level(arrow_plan P, int32_t level, int32_t *perm, int64_t *row_ptr, int32_t *col,
                                     void *val) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    if (level < 0 || level >= P->arrow_levels) return fail(ARROW_E_INVALID_ARG, "level out of range");
    const HostLevel &L = P->host_levels[level];
    if (perm) std::memcpy(perm, L.perm.data(), L.perm.size() * 4);
    if (row_ptr) std::memcpy(row_ptr, L.row_ptr.data(), L.row_ptr.size() * 8);
    if (col) std::memcpy(col, L.col.data(), L.col.size() * 4);
    if (val) std::memcpy(val, P->host_level_vals[level].data(), P->host_level_vals[level].size());
    return ARROW_OK;
}

arrow_status arrow_plan_local_rows(arrow_plan P, int64_t *begin, int64_t *end) {
    if (!P || !begin || !end) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    *begin = P->local_begin;
    *end = P->local_end;
    return ARROW_OK;
}

arrow_status arrow_plan_set_profiling(arrow_plan P, int32_t on) {
    if (!P) return fail(ARROW_E_INVALID_ARG, "plan is NULL");
    for (auto &r : P->prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    P->prof.clear();
    P->prof_acc = arrow_kernel_times_t{};
    P->profiling = on != 0;
    return ARROW_OK;
}

arrow_status arrow_plan_kernel_times(arrow_plan P, arrow_kernel_times_t *out) {
    if (!P || !out) return fail(ARROW_E_INVALID_ARG, "NULL argument");
    for (auto &r : P->prof) {
        CUDA_TRY(cudaEventSynchronize(r.b));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
        P->prof_acc.ms[r.kid] += ms;
        P->prof_acc.launches[r.kid] += 1;
        if (r.pos < 16) P->prof_acc.launch_ms[r.pos] += ms;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    P->prof.clear();
    *out = P->prof_acc;
    return ARROW_OK;
}

}  // extern "C"
