// CUDA IPC plumbing for runtime.PeerTransport: the two parties' processes map
// each other's message buffers, so the evaluation kernel of one party reads the
// other party's masked message straight out of the peer's HBM (NVLink / NVSwitch
// peer loads across GPUs; the same device when both processes share one GPU).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

extern "C" {

int fss_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// Exported buffers are whole cudaMalloc allocations: an IPC handle names the
// allocation BASE, so a sub-allocation of a caching allocator would map at the
// wrong address in the peer.
int fss_ipc_alloc(uint64_t nbytes, void** dev_ptr) {
    const cudaError_t err = cudaMalloc(dev_ptr, nbytes);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_ipc_free(void* dev_ptr) {
    const cudaError_t err = cudaFree(dev_ptr);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_memcpy_d2d(void* dst, const void* src, uint64_t nbytes, void* stream) {
    if (!nbytes) return FSS_OK;
    const cudaError_t err =
        cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_ipc_get_handle(const void* dev_ptr, uint8_t* handle) {
    cudaIpcMemHandle_t h;
    const cudaError_t err = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    memcpy(handle, &h, sizeof(h));
    return FSS_OK;
}

int fss_ipc_open_handle(const uint8_t* handle, void** dev_ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const cudaError_t err = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_ipc_close_handle(void* dev_ptr) {
    const cudaError_t err = cudaIpcCloseMemHandle(dev_ptr);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

}  // extern "C"
