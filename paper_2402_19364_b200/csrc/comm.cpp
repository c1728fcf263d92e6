// comm.cpp -- distributed mode (placeholder until the NCCL layer lands).
#include "comm.h"

struct arrow_comm_s {
    int nranks = 1, rank = 0;
};

arrow_status comm_attach(arrow_plan, arrow_comm) { return ARROW_E_UNSUPPORTED; }
void comm_detach(arrow_plan) {}
arrow_status comm_spmm(arrow_plan, const void *, void *, int64_t, cudaStream_t) { return ARROW_E_UNSUPPORTED; }

extern "C" {
arrow_status arrow_comm_unique_id(uint8_t id[128]) { (void)id; return ARROW_E_UNSUPPORTED; }
arrow_status arrow_comm_create(int32_t, int32_t, const uint8_t[128], arrow_comm *out) {
    if (out) *out = nullptr;
    return ARROW_E_UNSUPPORTED;
}
arrow_status arrow_comm_destroy(arrow_comm comm) { delete comm; return ARROW_OK; }
}
