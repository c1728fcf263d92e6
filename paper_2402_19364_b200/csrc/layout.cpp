// layout.cpp -- the K-A segment layout of one level (arrow_internal.h SegLevel): pads every batch of
// `bs` segments to start at a multiple of 8 entries, builds the per-8-entry end masks and the batch
// table, and uploads.  Shared by the single-GPU plan builder (arrow_api.cpp) and the distributed
// one (dist.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "arrow_internal.h"

namespace arrow {

int upload_seg_level(const HostSegs &h, int es, int bs, int mode, std::vector<void *> &allocs, SegLevel &out,
                     std::string &err) {
    const int64_t nseg = (int64_t)h.seg_out.size();
    if ((int64_t)h.seg_end.size() != nseg || h.ent_val.size() != h.ent_col.size() * (size_t)es || bs < 1 || bs > 32 ||
        (bs & (bs - 1)) != 0) {
        err = "internal: inconsistent segment lists";
        return (int)cudaErrorInvalidValue;
    }
    const int64_t nbatch = (nseg + bs - 1) / bs;
    // padded offsets: batch b starts at the next multiple of 8 after batch b-1 ends
    std::vector<uint32_t> bat((size_t)(2 * nbatch));
    std::vector<uint32_t> se(h.seg_end.size());
    int64_t pos = 0;
    for (int64_t b = 0; b < nbatch; ++b) {
        const int64_t s0 = b * bs, s1 = std::min<int64_t>(nseg, s0 + bs);
        const int64_t u0 = s0 == 0 ? 0 : h.seg_end[s0 - 1], u1 = h.seg_end[s1 - 1];
        const int64_t p0 = (pos + 7) & ~(int64_t)7;
        const int64_t shift = p0 - u0;
        for (int64_t s = s0; s < s1; ++s) {
            const int64_t beg = s == 0 ? 0 : h.seg_end[s - 1];
            if ((int64_t)h.seg_end[s] <= beg) {
                err = "internal: empty segment";
                return (int)cudaErrorInvalidValue;
            }
            se[s] = (uint32_t)(h.seg_end[s] + shift);
        }
        pos = p0 + (u1 - u0);
        if (pos >= ((int64_t)1 << 32) - 16) {
            err = "level exceeds 2^32 padded entries";
            return -1;
        }
        bat[2 * b] = (uint32_t)p0;
        bat[2 * b + 1] = (uint32_t)pos;
    }
    const int64_t nent = ((pos + 7) & ~(int64_t)7) + 8;  // + one group of slack for the broadcast loads
    std::vector<int32_t> col((size_t)nent, 0);
    std::vector<uint8_t> val((size_t)(nent * es), 0);
    std::vector<uint8_t> gmask((size_t)(nent / 8), 0);
    for (int64_t b = 0; b < nbatch; ++b) {
        const int64_t s0 = b * bs, s1 = std::min<int64_t>(nseg, s0 + bs);
        const int64_t u0 = s0 == 0 ? 0 : h.seg_end[s0 - 1], u1 = h.seg_end[s1 - 1];
        const int64_t p0 = bat[2 * b];
        std::memcpy(col.data() + p0, h.ent_col.data() + u0, (size_t)(u1 - u0) * 4);
        std::memcpy(val.data() + p0 * es, h.ent_val.data() + u0 * es, (size_t)((u1 - u0) * es));
        for (int64_t s = s0; s < s1; ++s) {
            const uint32_t last = se[s] - 1u;
            gmask[last >> 3] |= (uint8_t)(1u << (last & 7u));
        }
    }
    // L2 prefetch plan: the rows a batch gathers for the first time in its level (X rows, and the
    // rows of the second source -- bit 31) are requested by the batch `ahead` batches earlier, i.e.
    // by a warp of the front that is that many batches ahead of the one that will read them.
    std::vector<uint32_t> pf_rng;
    std::vector<int32_t> pf_rows;
    if (h.pf_ahead > 0 && nbatch > h.pf_ahead) {
        int32_t maxx = 0, maxs = 0;
        for (const int32_t c : h.ent_col) {
            if (c < 0) maxs = std::max(maxs, (int32_t)(c & 0x7fffffff));
            else maxx = std::max(maxx, c);
        }
        std::vector<uint8_t> seenx((size_t)maxx + 1, 0), seens((size_t)maxs + 1, 0);
        std::vector<int64_t> off((size_t)nbatch + 1, 0);
        size_t lvl = 0;
        for (int64_t b = 0; b < nbatch; ++b) {
            const int64_t s0 = b * bs, s1 = std::min<int64_t>(nseg, s0 + bs);
            for (int64_t s = s0; s < s1; ++s) {
                if (lvl < h.level_seg.size() && s == h.level_seg[lvl]) {  // a new level: new first references
                    std::fill(seenx.begin(), seenx.end(), 0);
                    ++lvl;
                }
                for (int64_t e = (s == 0 ? 0 : h.seg_end[s - 1]); e < (int64_t)h.seg_end[s]; ++e) {
                    const int32_t c = h.ent_col[e];
                    uint8_t &f = c < 0 ? seens[(size_t)(c & 0x7fffffff)] : seenx[(size_t)c];
                    if (!f) {
                        f = 1;
                        pf_rows.push_back(c);
                    }
                }
            }
            off[b + 1] = (int64_t)pf_rows.size();
        }
        pf_rng.assign((size_t)(2 * nbatch), 0);
        for (int64_t b = 0; b + h.pf_ahead < nbatch; ++b) {
            pf_rng[2 * b] = (uint32_t)off[b + h.pf_ahead];
            pf_rng[2 * b + 1] = (uint32_t)off[b + h.pf_ahead + 1];
        }
    }
    auto up = [&](const void *src, size_t bytes) -> void * {
        void *d = nullptr;
        if (cudaMalloc(&d, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
        allocs.push_back(d);
        if (bytes && cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
        return d;
    };
    out = SegLevel{};
    out.nseg = nseg;
    out.nent = nent;
    out.nbatch = nbatch;
    out.bs = bs;
    out.mode = mode;
    out.seg_out = (int32_t *)up(h.seg_out.data(), h.seg_out.size() * 4);
    out.seg_end = (uint32_t *)up(se.data(), se.size() * 4);
    out.ent_col = (int32_t *)up(col.data(), col.size() * 4);
    out.ent_val = up(val.data(), val.size());
    out.gmask = (uint8_t *)up(gmask.data(), gmask.size());
    out.bat = (uint32_t *)up(bat.data(), bat.size() * 4);
    if (!pf_rows.empty()) {
        out.pf_rows = (int32_t *)up(pf_rows.data(), pf_rows.size() * 4);
        out.pf_rng = (uint32_t *)up(pf_rng.data(), pf_rng.size() * 4);
        if (!out.pf_rows || !out.pf_rng) {
            err = "upload of the prefetch plan failed";
            return (int)cudaErrorMemoryAllocation;
        }
    }
    if (!out.seg_out || !out.seg_end || !out.ent_col || !out.ent_val || !out.gmask || !out.bat) {
        const cudaError_t e = cudaGetLastError();
        err = std::string("upload of the segment layout failed: ") + cudaGetErrorString(e);
        return e != cudaSuccess ? (int)e : (int)cudaErrorMemoryAllocation;
    }
    return 0;
}

}  // namespace arrow
