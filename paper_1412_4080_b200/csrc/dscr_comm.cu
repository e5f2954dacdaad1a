// Multi-GPU plumbing for the native exchange: peer buffers shared between the
// one-process-per-GPU ranks through CUDA IPC.  The host all-gathers the 64-byte
// handles through torch.distributed; NCCL collectives (the default exchange) are
// issued by the host through torch.distributed on the solver's stream.
#include <cuda_runtime.h>
#include <string.h>

#include "dynscreen.h"
#include "dscr_device.cuh"

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

}
