// comm.cpp — the one collective of the sharded layer: assembling the
// head-sharded output with an in-place NCCL all-gather over NVLink/NVSwitch.
//
// KV heads shard across the GPUs of a node with no exchange on the data path; rank r
// computes Q heads [r*Hq/N, (r+1)*Hq/N) and, with VSP_O_HEAD_MAJOR, K3 writes them straight
// into their final slab of a head-major O [Hq, n, 128] (the reference's per-head n x d
// matrices, attention.hpp:150). That slab is exactly rank r's all-gather send buffer, so the
// assembly is ONE in-place ncclAllGather: no permute, no staging copy. LSE [Hq, n] is
// head-major already and rides along in a second all-gather of the same group call.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2 — torch's copy when torch already
// loaded it, else the system one), so libvsp_gpu.so itself has no hard NCCL dependency and a
// single-GPU caller never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/vsp_gpu.h"
#include "vsp_error.h"

struct vsp_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
};

namespace {

using vsp_detail::set_err;

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) {
            n.load_error = std::string("vsp: cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](const char* s) { return dlsym(n.h, s); };
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
        n.broadcast = reinterpret_cast<decltype(n.broadcast)>(sym("ncclBroadcast"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
        if (!n.get_unique_id || !n.init_rank || !n.destroy || !n.all_gather || !n.broadcast || !n.group_start ||
            !n.group_end || !n.error_string)
            n.load_error = "vsp: NCCL library lacks a required symbol";
    });
    return n;
}

int nccl_err(ncclResult_t r, const char* where) {
    return set_err(VSP_ENCCL, std::string(where) + ": " + nccl().error_string(r));
}

}  // namespace

extern "C" {

size_t vsp_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

int vsp_comm_unique_id(uint8_t* id) {
    if (!id) return set_err(VSP_EINVAL, "vsp_comm_unique_id: null id");
    Nccl& n = nccl();
    if (!n.load_error.empty()) return set_err(VSP_ENCCL, n.load_error);
    ncclUniqueId u;
    ncclResult_t r = n.get_unique_id(&u);
    if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
    return VSP_OK;
}

int vsp_comm_init(vsp_comm** out, int world, int rank, const uint8_t* id, int device) {
    if (!out || !id) return set_err(VSP_EINVAL, "vsp_comm_init: null argument");
    if (world < 1 || rank < 0 || rank >= world) return set_err(VSP_EINVAL, "vsp_comm_init: bad rank/world");
    Nccl& n = nccl();
    if (!n.load_error.empty()) return set_err(VSP_ENCCL, n.load_error);
    if (cudaSetDevice(device) != cudaSuccess) return set_err(VSP_ECUDA, "vsp_comm_init: cannot select device");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    auto* c = new vsp_comm;
    c->world = world;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = n.init_rank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_err(r, "ncclCommInitRank");
    }
    *out = c;
    return VSP_OK;
}

int vsp_comm_destroy(vsp_comm* c) {
    if (!c) return VSP_OK;
    ncclResult_t r = c->comm ? nccl().destroy(c->comm) : ncclSuccess;
    delete c;
    return r == ncclSuccess ? VSP_OK : nccl_err(r, "ncclCommDestroy");
}

int vsp_allgather_heads(vsp_comm* c, void* o_full, float* lse_full, int n, int hq, int d, void* stream) {
    if (!c) return set_err(VSP_EINVAL, "vsp_allgather_heads: null communicator");
    if (!o_full || n < 1 || hq < 1 || d < 1) return set_err(VSP_EINVAL, "vsp_allgather_heads: bad arguments");
    if (hq % c->world) return set_err(VSP_EINVAL, "vsp_allgather_heads: Q heads do not split across ranks");
    if (cudaSetDevice(c->device) != cudaSuccess) return set_err(VSP_ECUDA, "vsp_allgather_heads: cannot select device");
    Nccl& nc = nccl();
    const size_t per = static_cast<size_t>(hq / c->world);
    const size_t o_count = per * n * d;        // bf16 elements of one rank's slab
    const size_t l_count = per * n;            // fp32 LSE entries of one rank's slab
    auto* o = static_cast<uint16_t*>(o_full);  // bf16 storage
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ncclResult_t r = nc.group_start();
    if (r == ncclSuccess) r = nc.all_gather(o + c->rank * o_count, o, o_count, ncclBfloat16, c->comm, st);
    if (r == ncclSuccess && lse_full)
        r = nc.all_gather(lse_full + c->rank * l_count, lse_full, l_count, ncclFloat32, c->comm, st);
    const ncclResult_t r2 = nc.group_end();
    if (r != ncclSuccess) return nccl_err(r, "ncclAllGather");
    if (r2 != ncclSuccess) return nccl_err(r2, "ncclGroupEnd");
    return VSP_OK;
}

// Assembly of a unit split (balanced / spread): unit u = (owner rank, KV head g, query blocks
// [lo, hi)) was attended by its owner, which wrote O rows [128 lo, min(128 hi, n)) of the
// group's Q heads into its head-major o_full (and lse_full). Each such region is contiguous
// per Q head, so the assembly is one in-place ncclBroadcast per (unit, Q head) from its
// owner, all inside one NCCL group (one launch per peer set, transfers overlapped).
int vsp_assemble_units(vsp_comm* c, void* o_full, float* lse_full, int n, int hq, int hkv, int d,
                       const int32_t* units, int count, void* stream) {
    if (!c) return set_err(VSP_EINVAL, "vsp_assemble_units: null communicator");
    if (!o_full || n < 1 || hq < 1 || hkv < 1 || hq % hkv || d < 1 || count < 0 || (count && !units))
        return set_err(VSP_EINVAL, "vsp_assemble_units: bad arguments");
    const int grp = hq / hkv, nqb = (n + 127) / 128;
    for (int u = 0; u < count; ++u) {
        const int32_t* x = units + 4 * u;
        if (x[0] < 0 || x[0] >= c->world || x[1] < 0 || x[1] >= hkv || x[2] < 0 || x[2] >= x[3] || x[3] > nqb)
            return set_err(VSP_EINVAL, "vsp_assemble_units: unit " + std::to_string(u) + " out of range");
    }
    if (cudaSetDevice(c->device) != cudaSuccess) return set_err(VSP_ECUDA, "vsp_assemble_units: cannot select device");
    Nccl& nc = nccl();
    auto* o = static_cast<uint16_t*>(o_full);  // bf16 storage
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ncclResult_t r = nc.group_start();
    for (int u = 0; u < count && r == ncclSuccess; ++u) {
        const int32_t* x = units + 4 * u;
        const size_t r0 = static_cast<size_t>(x[2]) * 128, r1 = std::min(static_cast<size_t>(x[3]) * 128,
                                                                         static_cast<size_t>(n));
        for (int h = x[1] * grp; h < (x[1] + 1) * grp && r == ncclSuccess; ++h) {
            uint16_t* ob = o + (static_cast<size_t>(h) * n + r0) * d;
            r = nc.broadcast(ob, ob, (r1 - r0) * d, ncclBfloat16, x[0], c->comm, st);
            if (r == ncclSuccess && lse_full) {
                float* lb = lse_full + static_cast<size_t>(h) * n + r0;
                r = nc.broadcast(lb, lb, r1 - r0, ncclFloat32, x[0], c->comm, st);
            }
        }
    }
    const ncclResult_t r2 = nc.group_end();
    if (r != ncclSuccess) return nccl_err(r, "ncclBroadcast");
    if (r2 != ncclSuccess) return nccl_err(r2, "ncclGroupEnd");
    return VSP_OK;
}

}  // extern "C"
