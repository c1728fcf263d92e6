// plan.h -- internal definitions of the plan and decomposition objects (shared by arrow_api.cpp
// and dist.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/arrow.h"
#include "arrow_internal.h"

namespace arrow {

arrow_status set_error(arrow_status s, const std::string &msg);  // thread-local detail (arrow_last_error)

constexpr int64_t kDefaultWindowRows = 16384;
constexpr int64_t kDefaultLevel0WindowRows = 65536;  // default window of level 0 (profiles/r02/win)
constexpr int32_t kDefaultHeadChunk = 32;  // measured best at config R (k = 8, 32, 128): sweep in DESIGN.md §7

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct ProfRec {
    int kid, pos;
    cudaEvent_t a, b;
};

// deterministic mode's K-C, two fixed-order passes over the head partials of every level: (1) group g
// = the sum of up to kDetGroup consecutive slots of one head row (slots by level, then chunk);
// (2) Y[rows[r]] += the groups of head row r, in order
struct DetLevel {
    int64_t nh = 0, ng = 0;
    int32_t *gptr = nullptr, *gsrc = nullptr, *gdst = nullptr;  // pass 1: group -> its slots
    int32_t *ptr = nullptr, *src = nullptr, *rows = nullptr;     // pass 2: head row -> its groups
};
constexpr int kDetGroup = 32;
constexpr int kDetHeadChunk = 128;  // deterministic mode's default head chunk (entries per slot)

struct DistState;  // dist.cpp
void dist_free(DistState *d);

}  // namespace arrow

using arrow::DeviceLevel;
using arrow::HostLevel;
using arrow::ProfRec;
using arrow::SegLevel;

struct arrow_plan_s {
    int device = 0;
    int num_sms = 148;
    arrow_dtype dtype = ARROW_F32;
    int order = ARROW_ORDER_ORIGINAL;
    int64_t n = 0, nnz = 0, b = 0;
    int64_t isolated = 0;
    int64_t residual_nnz = 0;
    int64_t max_head = 0;
    double create_seconds = 0;
    std::vector<DeviceLevel> levels;  // device launch list: level 0, then levels >= 1 (+ residual), possibly merged
    std::vector<DeviceLevel> meta;    // per arrow level (+ residual) metadata for introspection
    int32_t arrow_levels = 0;
    // host copy of the canonical levels for export
    std::vector<HostLevel> host_levels;
    std::vector<std::vector<uint8_t>> host_level_vals;  // per level, plan dtype
    // device memory
    void *arena = nullptr;
    int64_t arena_bytes = 0;
    std::vector<SegLevel> seg;     // K-A segment layout per launch level
    int32_t *post_rows = nullptr;  // rows last written by a head-row partial (iterate's activation pass)
    int64_t n_post = 0;
    std::vector<void *> seg_allocs;
    arrow::SegLaunch launch;       // per-call K-A options (options.flags)
    bool use_graphs = true;        // single GPU: replay the call as one CUDA graph (options.flags)
    int32_t transport = 0;         // ARROW_TRANSPORT_* (distributed plans)
    unsigned *counters = nullptr;  // per-level work counters of K-A (zeroed at the start of each call)
    void *ws = nullptr;            // single GPU, deterministic mode: head-partial slots (det_slots x ws_k)
    int64_t ws_k = 0;
    bool det = false;              // options.flags & ARROW_FLAG_DETERMINISTIC
    int64_t det_slots = 0, det_groups = 0;  // rows of the slot and group regions of ws
    arrow::DetLevel det_kc;  // deterministic mode: the one K-C pass over every level's head partials
    void *host_x = nullptr, *host_y = nullptr;  // device staging for arrow_spmm_host
    int64_t host_k = 0;
    // arrow_spmm_host_batch: two device slots, two copy streams, per-slot events
    void *hb_x[2] = {nullptr, nullptr}, *hb_y[2] = {nullptr, nullptr};
    int64_t hb_k = 0;
    cudaStream_t hb_h2d = nullptr, hb_d2h = nullptr;
    cudaEvent_t hb_ev[7] = {};  // x[2], c[2], y[2], start/done
    bool no_graph = false;
    cudaStream_t stream = nullptr;
    // CUDA graph of the single-GPU call, keyed by (X, Y, k, stream)
    cudaGraphExec_t gexec = nullptr;
    const void *g_x = nullptr;
    void *g_y = nullptr;
    int64_t g_k = 0;
    cudaStream_t g_stream = nullptr;
    bool poisoned = false;
    // profiling
    bool profiling = false;
    std::vector<ProfRec> prof;
    arrow_kernel_times_t prof_acc{};
    int prof_pos = 0;
    // distributed
    arrow_comm comm = nullptr;
    int64_t local_begin = 0, local_end = 0;
    int64_t bytes_alg_fixed = 0, bytes_alg_rows = 0, sum_rows = 0;

    arrow::DistState *dist = nullptr;

    ~arrow_plan_s() {
        if (dist) arrow::dist_free(dist);
        for (void *q : seg_allocs) cudaFree(q);
        for (auto &r : prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
        if (arena) cudaFree(arena);
        if (ws) cudaFree(ws);
        if (host_x) cudaFree(host_x);
        if (host_y) cudaFree(host_y);
        for (int i = 0; i < 2; ++i) { if (hb_x[i]) cudaFree(hb_x[i]); if (hb_y[i]) cudaFree(hb_y[i]); }
        for (cudaEvent_t e : hb_ev) if (e) cudaEventDestroy(e);
        if (hb_h2d) cudaStreamDestroy(hb_h2d);
        if (hb_d2h) cudaStreamDestroy(hb_d2h);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (post_rows) cudaFree(post_rows);
    }
    size_t esize() const { return dtype == ARROW_F64 ? 8 : 4; }
};

// Host decomposition object: canonical levels (values as fp64) + residual triples.
struct arrow_decomposition_s {
    int64_t n = 0, b = 0;
    uint64_t seed = 4;
    int32_t band = 0;                    // ARROW_BAND_* of step 3
    int32_t homes = 1;                   // home-set-aware arrangement for this many ranks (R25); 1 = off
    int32_t home_levels = 0;             // levels 1..home_levels home-aware (homes > 1)
    std::vector<int64_t> home_los;       // [homes + 1] pi_0 home ranges (homes > 1)
    int64_t isolated = 0;
    std::vector<HostLevel> levels;
    std::vector<int32_t> res_u, res_v;  // residual entries, original ids, CSR order
    std::vector<double> res_a;
    double seconds = 0;
};

