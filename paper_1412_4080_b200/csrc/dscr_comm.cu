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
    dscr::err_store() = "multi-rank iteration path is driven by paper_1412_4080_b200.dist (torch.distributed NCCL)";
    return DSCR_ENOCOMM;
}
