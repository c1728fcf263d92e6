// comm.h -- distributed mode (NCCL over NVLink/NVSwitch), one process per GPU.
#pragma once
#include <cuda_runtime.h>

#include "../../include/arrow.h"

arrow_status comm_attach(arrow_plan plan, arrow_comm comm);
void comm_detach(arrow_plan plan);
arrow_status comm_spmm(arrow_plan plan, const void *X, void *Y, int64_t k, cudaStream_t st);
