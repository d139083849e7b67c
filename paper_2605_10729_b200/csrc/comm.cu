// In-process NCCL communicators for the reference's thread-rank model.
//
// The reference runs its SPMD ranks as threads of one process and reduces with
// a fixed-order tree over numpy arrays (/root/reference/pkg/src/pifsim/comm.py:
// 329-339 _tree_sum, 391-408 allreduce_sum, 483-528 spawn_spmd).  Here each
// rank thread drives one GPU and the per-step allreduce of [raw rho_hat | diag]
// (strategies.py:162-164 + :106) is one ncclAllReduce over NVLink/NVSwitch on
// that rank's stream.  The communicators of all ranks come from one
// ncclCommInitAll call (single process).
//
// libnccl is opened at run time (dlopen of the soname libnccl.so.2): when torch
// has already loaded its bundled NCCL the same instance is reused, so the
// process never carries two NCCL versions.  Only the four entry points below are
// needed; their C ABI is stable across NCCL 2.x.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <new>
#include <string>

#include "pif_internal.cuh"

struct pif_comm_s {
    ncclComm_t comm = nullptr;
    int device = 0;
    int rank = 0, size = 1;
};

namespace {

struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*init_all)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*version)(int *) = nullptr;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;
std::string g_nccl_err;

void open_nccl() {
    // prefer an already loaded NCCL (torch's), then the soname on the search path
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char *e = dlerror();
        g_nccl_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
        return;
    }
    g_nccl.handle = h;
    g_nccl.init_all = reinterpret_cast<decltype(g_nccl.init_all)>(dlsym(h, "ncclCommInitAll"));
    g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(dlsym(h, "ncclAllReduce"));
    g_nccl.destroy = reinterpret_cast<decltype(g_nccl.destroy)>(dlsym(h, "ncclCommDestroy"));
    g_nccl.error_string =
        reinterpret_cast<decltype(g_nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
    g_nccl.version = reinterpret_cast<decltype(g_nccl.version)>(dlsym(h, "ncclGetVersion"));
    if (!g_nccl.init_all || !g_nccl.all_reduce || !g_nccl.destroy || !g_nccl.error_string) {
        g_nccl_err = "libnccl.so.2 lacks ncclCommInitAll/ncclAllReduce/ncclCommDestroy";
        g_nccl.handle = nullptr;
    }
}

bool nccl_ready() {
    std::call_once(g_nccl_once, open_nccl);
    if (!g_nccl.handle) {
        pif::set_error(g_nccl_err);
        return false;
    }
    return true;
}

int fail_nccl(ncclResult_t r, const char *where) {
    pif::set_error(std::string(where) + ": " + g_nccl.error_string(r));
    return PIF_ERR_CUDA;
}

}  // namespace

extern "C" {

int pif_nccl_version(int *version) {
    if (!version) {
        pif::set_error("null version");
        return PIF_ERR_VALUE;
    }
    if (!nccl_ready()) return PIF_ERR_CUDA;
    *version = 0;
    if (g_nccl.version) g_nccl.version(version);
    return PIF_OK;
}

int pif_comm_init_all(int ndev, const int *devices, pif_comm_t *comms_out) {
    if (ndev < 1 || !devices || !comms_out) {
        pif::set_error("pif_comm_init_all: need ndev >= 1, devices and comms_out");
        return PIF_ERR_VALUE;
    }
    for (int i = 0; i < ndev; ++i) {
        comms_out[i] = nullptr;
        for (int j = 0; j < i; ++j)
            if (devices[i] == devices[j]) {
                pif::set_error("pif_comm_init_all: NCCL needs one device per rank");
                return PIF_ERR_VALUE;
            }
    }
    if (!nccl_ready()) return PIF_ERR_CUDA;
    ncclComm_t *raw = new (std::nothrow) ncclComm_t[ndev];
    if (!raw) {
        pif::set_error("out of host memory");
        return PIF_ERR_VALUE;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    ncclResult_t r = g_nccl.init_all(raw, ndev, devices);
    if (prev >= 0) cudaSetDevice(prev);
    if (r != ncclSuccess) {
        delete[] raw;
        return fail_nccl(r, "ncclCommInitAll");
    }
    for (int i = 0; i < ndev; ++i) {
        pif_comm_s *c = new (std::nothrow) pif_comm_s;
        if (!c) {
            for (int j = 0; j < ndev; ++j) {
                if (j < i) delete comms_out[j];
                g_nccl.destroy(raw[j]);
                comms_out[j] = nullptr;
            }
            delete[] raw;
            pif::set_error("out of host memory");
            return PIF_ERR_VALUE;
        }
        c->comm = raw[i];
        c->device = devices[i];
        c->rank = i;
        c->size = ndev;
        comms_out[i] = c;
    }
    delete[] raw;
    return PIF_OK;
}

int pif_allreduce_f64(pif_comm_t comm, double *buf, int64_t count, void *stream) {
    if (!comm) {
        pif::set_error("null communicator");
        return PIF_ERR_VALUE;
    }
    if (count < 0 || (count > 0 && !buf)) {
        pif::set_error("invalid allreduce buffer");
        return PIF_ERR_VALUE;
    }
    if (count == 0) return PIF_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != comm->device) cudaSetDevice(comm->device);
    ncclResult_t r = g_nccl.all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, comm->comm,
                                       reinterpret_cast<cudaStream_t>(stream));
    if (prev >= 0 && prev != comm->device) cudaSetDevice(prev);
    if (r != ncclSuccess) return fail_nccl(r, "ncclAllReduce");
    return PIF_OK;
}

int pif_comm_destroy(pif_comm_t comm) {
    if (!comm) return PIF_OK;
    if (g_nccl.handle && comm->comm) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(comm->device);
        g_nccl.destroy(comm->comm);
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete comm;
    return PIF_OK;
}

}  // extern "C"
