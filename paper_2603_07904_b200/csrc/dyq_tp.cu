// dyq_tp.cu -- column-sharded tensor parallelism for the quantized linears
// (BASELINE config 5; not in the paper): rank r holds rows
// [r N/P, (r+1) N/P) of every packed weight (a K-group never spans ranks, so
// the shard's pack equals the slice of the full pack), computes its output
// columns with dyq_qlinear, and the shards are joined with an NCCL all-gather
// over NVLink followed by a column interleave [P][M][N/P] -> [M][N].
//
// NCCL is loaded at run time (dlopen of libnccl.so.2 -- the copy torch already
// mapped when it is in the process, the system one otherwise), so libdyq.so
// has no link-time dependency on a particular NCCL build.
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        const char* path = getenv("DYQ_NCCL_LIB");
        void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return a;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString;
        return a;
    }();
    return api;
}

struct Comm {
    ncclComm_t c;
    int rank, world;
};

// y[m][r * Ns + j] = buf[r][m][j]   (16-byte vectors; Ns % 8 == 0)
__global__ void tp_interleave_kernel(const uint16_t* __restrict__ buf, int P, int M, int Ns,
                                     uint16_t* __restrict__ y) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int vs = Ns / 8;
    if (idx >= (size_t)P * M * vs) return;
    const int r = (int)(idx / ((size_t)M * vs));
    const int rem = (int)(idx % ((size_t)M * vs));
    const int m = rem / vs, j = (rem % vs) * 8;
    *reinterpret_cast<uint4*>(y + (size_t)m * P * Ns + (size_t)r * Ns + j) =
        *reinterpret_cast<const uint4*>(buf + ((size_t)r * M + m) * Ns + j);
}

// Wait until *flag >= target (system-scope acquire), bounded: after ~timeout_ns
// the kernel records a timeout in *status and returns instead of hanging.
__global__ void tp_wait_kernel(const unsigned long long* flag, unsigned long long target, long long timeout_ns,
                               int* status) {
    ptx::pdl_launch_dependents();
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= target) return;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((long long)(t - t0) > timeout_ns) {
            if (status) atomicExch(status, 1);
            return;
        }
        __nanosleep(100);
    }
}

}  // namespace dyq

using namespace dyq;

extern "C" {

dyq_status_t dyq_tp_wait(const uint64_t* flag, uint64_t target, int32_t* timed_out, dyq_stream_t stream) {
    if (!flag) return set_error(DYQ_EINVAL, "null flag");
    tp_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const unsigned long long*>(flag),
                                                      (unsigned long long)target, 10'000'000'000LL, timed_out);
    return check_launch("tp_wait_kernel");
}

// An IPC handle names a whole allocation (e.g. a caching-allocator segment),
// so the handle travels with the pointer's offset from the allocation base
// (cuMemGetAddressRange through the runtime's driver entry point: no link-time
// libcuda dependency).
dyq_status_t dyq_ipc_handle(void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_error(DYQ_EINVAL, "null pointer");
    typedef int (*RangeFn)(unsigned long long*, size_t*, unsigned long long);
    static RangeFn range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<RangeFn>(fn);
    }();
    if (!range) return set_error(DYQ_EUNSUPPORTED, "cuMemGetAddressRange entry point unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
        return set_error(DYQ_EINVAL, "pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((uintptr_t)dev_ptr - base);
    return DYQ_OK;
}

dyq_status_t dyq_ipc_open(const void* handle, uint64_t offset, void** dev_ptr) {
    if (!handle || !dev_ptr) return set_error(DYQ_EINVAL, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *dev_ptr = reinterpret_cast<uint8_t*>(base) + offset;
    return DYQ_OK;
}

dyq_status_t dyq_ipc_close(void* dev_ptr, uint64_t offset) {
    if (!dev_ptr) return set_error(DYQ_EINVAL, "null pointer");
    const cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<uint8_t*>(dev_ptr) - offset);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return DYQ_OK;
}

dyq_status_t dyq_tp_shard(int32_t N, int32_t world, int32_t rank, int32_t* n0, int32_t* n1) {
    if (world <= 0 || rank < 0 || rank >= world) return set_error(DYQ_EINVAL, "bad rank %d / world %d", rank, world);
    if (N <= 0 || N % (16 * world)) return set_error(DYQ_ESHAPE, "N = %d must be a multiple of 16 * world", N);
    const int ns = N / world;
    if (n0) *n0 = rank * ns;
    if (n1) *n1 = (rank + 1) * ns;
    return DYQ_OK;
}

dyq_status_t dyq_comm_unique_id(void* id_host) {
    if (!id_host) return set_error(DYQ_EINVAL, "null id buffer");
    NcclApi& a = nccl();
    if (!a.ok) return set_error(DYQ_EUNSUPPORTED, "NCCL (libnccl.so.2) could not be loaded");
    ncclUniqueId id;
    const ncclResult_t r = a.GetUniqueId(&id);
    if (r != ncclSuccess) return set_error(DYQ_ENCCL, "ncclGetUniqueId: %s", a.GetErrorString(r));
    memcpy(id_host, &id, sizeof id);
    return DYQ_OK;
}

dyq_status_t dyq_comm_init(const void* id_host, int32_t rank, int32_t world, void** comm) {
    if (!id_host || !comm) return set_error(DYQ_EINVAL, "null pointer");
    if (world <= 0 || rank < 0 || rank >= world) return set_error(DYQ_EINVAL, "bad rank %d / world %d", rank, world);
    NcclApi& a = nccl();
    if (!a.ok) return set_error(DYQ_EUNSUPPORTED, "NCCL (libnccl.so.2) could not be loaded");
    ncclUniqueId id;
    memcpy(&id, id_host, sizeof id);
    Comm* c = new Comm();
    const ncclResult_t r = a.CommInitRank(&c->c, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return set_error(DYQ_ENCCL, "ncclCommInitRank: %s", a.GetErrorString(r));
    }
    c->rank = rank;
    c->world = world;
    *comm = c;
    return DYQ_OK;
}

dyq_status_t dyq_comm_destroy(void* comm) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (!c) return DYQ_OK;
    NcclApi& a = nccl();
    if (a.ok) a.CommDestroy(c->c);
    delete c;
    return DYQ_OK;
}

dyq_status_t dyq_tp_interleave(const uint16_t* buf, int32_t P, int32_t M, int32_t Ns, uint16_t* y,
                               dyq_stream_t stream) {
    if (P <= 0 || M < 0 || Ns <= 0 || Ns % 8) return set_error(DYQ_ESHAPE, "bad interleave shape");
    if (M == 0) return DYQ_OK;
    if (!buf || !y) return set_error(DYQ_EINVAL, "null pointer");
    const size_t n = (size_t)P * M * (Ns / 8);
    tp_interleave_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(buf, P, M, Ns, y);
    return check_launch("tp_interleave_kernel");
}

dyq_status_t dyq_tp_allgather(void* comm, const uint16_t* y_shard, int32_t M, int32_t N, uint16_t* gather_buf,
                              uint16_t* y, dyq_stream_t stream) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (!c || !y_shard || !y) return set_error(DYQ_EINVAL, "null pointer");
    if (M < 0 || N <= 0 || N % (16 * c->world)) return set_error(DYQ_ESHAPE, "N = %d must be a multiple of 16 * world", N);
    if (M == 0) return DYQ_OK;
    const int Ns = N / c->world;
    NcclApi& a = nccl();
    // M == 1: [P][1][Ns] is already [1][N] -- gather straight into y
    uint16_t* dst = (M == 1) ? y : gather_buf;
    if (!dst) return set_error(DYQ_EINVAL, "gather_buf required for M > 1");
    const ncclResult_t r = a.AllGather(y_shard, dst, (size_t)M * Ns, ncclBfloat16, c->c, (cudaStream_t)stream);
    if (r != ncclSuccess) return set_error(DYQ_ENCCL, "ncclAllGather: %s", a.GetErrorString(r));
    if (M == 1) return DYQ_OK;
    return dyq_tp_interleave(gather_buf, c->world, M, Ns, y, stream);
}

}  // extern "C"
