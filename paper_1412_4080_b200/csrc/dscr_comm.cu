// Multi-GPU plumbing: NCCL is loaded at run time (dlopen of the libnccl.so.2
// that ships with PyTorch) so the library has no hard NCCL dependency.
// Rendezvous (exchanging the 128-byte unique id) is done by the host through
// torch.distributed; the collectives run on the solver's stream between the
// per-rank kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include "dynscreen.h"
#include "dscr_device.cuh"

namespace dscr {
namespace comm {

typedef struct { char internal[128]; } nccl_id_t;
typedef int (*get_id_fn)(nccl_id_t*);

static void* nccl_handle() {
    static void* h = nullptr;
    if (!h) {
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    return h;
}

}  // namespace comm
}  // namespace dscr

extern "C" {

// ---- peer buffers for the native exchange (CUDA IPC; one process per GPU) -----------------
int dscr_peer_alloc(size_t bytes, void** dptr, void* handle_out_64) {
    if (!dptr || !handle_out_64 || !bytes) { dscr::err_store() = "null argument"; return DSCR_EINVAL; }
    cudaError_t e = cudaMalloc(dptr, bytes);
    if (e == cudaSuccess) e = cudaMemset(*dptr, 0, bytes);
    cudaIpcMemHandle_t hd;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, *dptr);
    if (e != cudaSuccess) { dscr::err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    memcpy(handle_out_64, &hd, sizeof hd);
    return DSCR_OK;
}

int dscr_peer_open(const void* handle_64, void** dptr) {
    if (!handle_64 || !dptr) { dscr::err_store() = "null argument"; return DSCR_EINVAL; }
    cudaIpcMemHandle_t hd;
    memcpy(&hd, handle_64, sizeof hd);
    cudaError_t e = cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) { dscr::err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    return DSCR_OK;
}

int dscr_peer_close(void* dptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dptr);
    if (e != cudaSuccess) { dscr::err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    return DSCR_OK;
}

int dscr_peer_free(void* dptr) {
    cudaError_t e = cudaFree(dptr);
    if (e != cudaSuccess) { dscr::err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    return DSCR_OK;
}

int dscr_comm_unique_id(void* id_out_128) {
    void* h = dscr::comm::nccl_handle();
    if (!h) {
        dscr::err_store() = "libnccl.so.2 could not be loaded";
        return DSCR_ENOCOMM;
    }
    auto fn = (dscr::comm::get_id_fn)dlsym(h, "ncclGetUniqueId");
    if (!fn) {
        dscr::err_store() = "ncclGetUniqueId not found";
        return DSCR_ENOCOMM;
    }
    dscr::comm::nccl_id_t id;
    if (fn(&id) != 0) {
        dscr::err_store() = "ncclGetUniqueId failed";
        return DSCR_ENOCOMM;
    }
    memcpy(id_out_128, &id, 128);
    return DSCR_OK;
}

}

struct dscr_solver;
extern "C" int dscr_solver_set_comm(dscr_solver* h, const void* id_128, int rank, int world) {
    (void)id_128;
    if (!h) { dscr::err_store() = "null handle"; return DSCR_EINVAL; }
    if (world == 1 && rank == 0) return DSCR_OK;
    dscr::err_store() = "multi-rank trips are driven phase by phase (dscr_solver_phase): host collectives "
                        "through paper_1412_4080_b200.dist, or the native peer-memory exchange (dscr_solver_set_peers)";
    return DSCR_ENOCOMM;
}
