// comm.cpp -- NCCL communicator of the distributed mode (one process per GPU, NVLink/NVSwitch).
#include "comm.h"

#include <nccl.h>

#include <cstring>
#include <string>

#include "plan.h"

arrow_status arrow::comm_status(int nccl_result, const char *what) {
    if (nccl_result == ncclSuccess) return ARROW_OK;
    return set_error(ARROW_E_NCCL, std::string(what) + ": " + ncclGetErrorString((ncclResult_t)nccl_result));
}

extern "C" {

arrow_status arrow_comm_unique_id(uint8_t id[128]) {
    if (!id) return arrow::set_error(ARROW_E_INVALID_ARG, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    arrow_status s = arrow::comm_status(ncclGetUniqueId(&u), "ncclGetUniqueId");
    if (s != ARROW_OK) return s;
    std::memcpy(id, &u, 128);
    return ARROW_OK;
}

arrow_status arrow_comm_create(int32_t nranks, int32_t rank, const uint8_t id[128], arrow_comm *out) {
    if (!out || !id) return arrow::set_error(ARROW_E_INVALID_ARG, "NULL argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return arrow::set_error(ARROW_E_INVALID_ARG, "bad nranks/rank");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t c;
    arrow_status s = arrow::comm_status(ncclCommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
    if (s != ARROW_OK) return s;
    auto *cm = new arrow_comm_s();
    cm->comm = c;
    cm->nranks = nranks;
    cm->rank = rank;
    *out = cm;
    return ARROW_OK;
}

arrow_status arrow_comm_destroy(arrow_comm comm) {
    if (!comm) return ARROW_OK;
    if (comm->comm) ncclCommDestroy((ncclComm_t)comm->comm);
    delete comm;
    return ARROW_OK;
}

}  // extern "C"
