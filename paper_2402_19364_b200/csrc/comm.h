// comm.h -- distributed mode (NCCL over NVLink/NVSwitch), one process per GPU.
#pragma once
#include <cuda_runtime.h>

#include "../../include/arrow.h"

struct arrow_comm_s {
    void *comm = nullptr;  // ncclComm_t
    int nranks = 1, rank = 0;
};

struct arrow_decomposition_s;

namespace arrow {
arrow_status comm_status(int nccl_result, const char *what);
// Build this rank's part of a distributed plan (dist.cpp).
// window_rows0: the tile window of level 0 (window_rows: levels >= 1)
arrow_status dist_build(arrow_plan plan, const arrow_decomposition_s &D, arrow_comm comm, int64_t window_rows,
                        int64_t window_rows0, int32_t head_chunk, int bs);
arrow_status dist_spmm(arrow_plan plan, const void *X, void *Y, int64_t k, cudaStream_t st);
}  // namespace arrow
