// layout.cpp -- the K-A segment layout of one level (arrow_internal.h SegLevel): the per-8-entry end
// masks and the batch table of the segment list, uploaded with it.  Shared by the single-GPU plan builder (arrow_api.cpp) and the distributed
// one (dist.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "arrow_internal.h"

namespace arrow {

int upload_seg_level(const HostSegs &h, int es, int bs, int mode, int64_t max_x_row, std::vector<void *> &allocs,
                     SegLevel &out, std::string &err) {
    const int64_t nseg = (int64_t)h.seg_out.size();
    if ((int64_t)h.seg_end.size() != nseg || h.ent_val.size() != h.ent_col.size() * (size_t)es || bs < 1 || bs > 32 ||
        (bs & (bs - 1)) != 0) {
        err = "internal: inconsistent segment lists";
        return (int)cudaErrorInvalidValue;
    }
    // Work batch b = segments [b (bs + 1), b (bs + 1) + bs) of the list, starting at a multiple of 8
    // entries; segment b (bs + 1) + bs is a padding segment (1 to 8 value-0 entries re-reading the
    // previous column, output kDiscard) that fills the gap to the next batch.  Kernels that walk the
    // segment list in order process padding segments and drop their result; the full-warp kernel
    // reads only the batches' real entries, and a batch's segments sit at a fixed stride.
    const int64_t nbatch = (nseg + bs - 1) / bs;
    std::vector<int32_t> so, col;
    std::vector<uint32_t> se;
    std::vector<uint8_t> val;
    std::vector<uint32_t> bat((size_t)(2 * nbatch));
    so.reserve((size_t)(nseg + nbatch));
    se.reserve((size_t)(nseg + nbatch));
    col.reserve(h.ent_col.size() + (size_t)nbatch * 8 + 16);
    val.reserve((h.ent_col.size() + (size_t)nbatch * 8 + 16) * es);
    int64_t pos = 0;
    for (int64_t b = 0; b < nbatch; ++b) {
        const int64_t s0 = b * bs, s1 = std::min<int64_t>(nseg, s0 + bs);
        bat[2 * b] = (uint32_t)pos;
        for (int64_t sg = s0; sg < s1; ++sg) {
            const int64_t u0 = sg == 0 ? 0 : h.seg_end[sg - 1], u1 = h.seg_end[sg];
            if (u1 <= u0) {
                err = "internal: empty segment";
                return (int)cudaErrorInvalidValue;
            }
            col.insert(col.end(), h.ent_col.begin() + u0, h.ent_col.begin() + u1);
            val.insert(val.end(), h.ent_val.begin() + u0 * es, h.ent_val.begin() + u1 * es);
            pos += u1 - u0;
            so.push_back(h.seg_out[sg]);
            se.push_back((uint32_t)pos);
        }
        bat[2 * b + 1] = (uint32_t)pos;
        if (b + 1 < nbatch) {  // the padding segment (the last batch has none)
            const int64_t pad = 8 - (pos & 7);
            const int32_t c = col.back();
            for (int64_t t = 0; t < pad; ++t) {
                col.push_back(c);
                val.insert(val.end(), (size_t)es, (uint8_t)0);
            }
            pos += pad;
            so.push_back((int32_t)kDiscard);
            se.push_back((uint32_t)pos);
        }
        if (pos >= ((int64_t)1 << 32) - 16) {
            err = "level exceeds 2^32 entries";
            return -1;
        }
    }
    // entries padded at the end to whole groups of 8 (+ one group of slack for the broadcast loads)
    const int64_t nent = ((pos + 7) & ~(int64_t)7) + 8;
    col.resize((size_t)nent, col.empty() ? 0 : col.back());
    val.resize((size_t)(nent * es), 0);
    std::vector<uint8_t> gmask((size_t)(nent / 8), 0);
    for (const uint32_t e : se) gmask[(e - 1u) >> 3] |= (uint8_t)(1u << ((e - 1u) & 7u));
    auto up = [&](const void *src, size_t bytes) -> void * {
        void *d = nullptr;
        if (cudaMalloc(&d, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
        allocs.push_back(d);
        if (bytes && cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
        return d;
    };
    out = SegLevel{};
    out.nseg = (int64_t)so.size();
    out.nent = nent;
    out.nbatch = nbatch;
    out.bs = bs;
    out.mode = mode;
    out.max_x_row = max_x_row;
    out.seg_out = (int32_t *)up(so.data(), so.size() * 4);
    out.seg_end = (uint32_t *)up(se.data(), se.size() * 4);
    out.ent_col = (int32_t *)up(col.data(), col.size() * 4);
    out.ent_val = up(val.data(), val.size());
    out.gmask = (uint8_t *)up(gmask.data(), gmask.size());
    out.bat = (uint32_t *)up(bat.data(), bat.size() * 4);
    if (!out.seg_out || !out.seg_end || !out.ent_col || !out.ent_val || !out.gmask || !out.bat) {
        const cudaError_t e = cudaGetLastError();
        err = std::string("upload of the segment layout failed: ") + cudaGetErrorString(e);
        return e != cudaSuccess ? (int)e : (int)cudaErrorMemoryAllocation;
    }
    return 0;
}

}  // namespace arrow
