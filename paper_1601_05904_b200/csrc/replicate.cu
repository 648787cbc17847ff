// replicate.cu — data replication for the single-process multi-device
// pipeline ("ncclCommInitAll over the devices, one
// ncclBroadcast of the data arrays").
//
// The data set (x, y, z: 24 B per point) is copied host -> device ONCE, to
// the first listed device, and broadcast from there to every other distinct
// device over NVLink by NCCL (one grouped ncclBroadcast per array, one
// communicator per device from ncclCommInitAll, cached per device set).
// Shards that share a device share its replica (read-only).  NCCL is
// resolved at run time (dlopen "libnccl.so.2" — the one the process already
// mapped, e.g. torch's, or the system's), so the library has no link-time
// NCCL dependency; if it cannot be loaded the replicas are filled by CUDA
// peer copies (cudaMemcpyPeerAsync) instead — still device to device,
// recorded in the replication kind.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "replicate.cuh"

namespace aidwb {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.why = e ? e : "dlopen libnccl.so.2 failed";
            return a;
        }
        a.init_all = reinterpret_cast<decltype(a.init_all)>(dlsym(h, "ncclCommInitAll"));
        a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.init_all && a.broadcast && a.group_start && a.group_end;
        if (!a.ok) a.why = "libnccl.so.2 lacks ncclCommInitAll / ncclBroadcast";
        return a;
    }();
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* e = nccl().error_string ? nccl().error_string(r) : "?";
        throw Failure(AIDW_ERR_CUDA, std::string(what) + ": " + e);
    }
}

// One communicator per device of a device set, created once (ncclCommInitAll
// costs ~100 ms) and kept for the life of the process.
std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

std::atomic<long long> g_broadcasts{0};
std::atomic<int> g_last_kind{kReplicateNone};

}  // namespace

long long nccl_broadcast_count() { return g_broadcasts.load(); }
int last_replication_kind() { return g_last_kind.load(); }

int nccl_version() {
    int v = 0;
    if (nccl().ok && nccl().get_version) nccl().get_version(&v);
    return v;
}

Replicas::~Replicas() {
    for (size_t i = 0; i < devs.size(); ++i) {
        if (cudaSetDevice(devs[i]) != cudaSuccess) continue;
        if (streams[i]) cudaStreamSynchronize(streams[i]);
        for (double* p : {x[i], y[i], z[i]})
            if (p) cudaFree(p);
        if (streams[i]) cudaStreamDestroy(streams[i]);
    }
    cudaGetLastError();
}

int Replicas::slot_of(int dev) const {
    for (size_t i = 0; i < devs.size(); ++i)
        if (devs[i] == dev) return static_cast<int>(i);
    return -1;
}

void replicate_data(const std::vector<int>& devices, const double* hx, const double* hy,
                    const double* hz, size_t m, Replicas& out) {
    struct KeepDevice {  // the caller's current device survives the call
        int dev = 0;
        KeepDevice() { cudaGetDevice(&dev); }
        ~KeepDevice() { cudaSetDevice(dev); }
    } keep;
    std::vector<int> u;  // distinct devices, first-appearance order
    for (int d : devices)
        if (std::find(u.begin(), u.end(), d) == u.end()) u.push_back(d);
    const size_t D = u.size();
    out.devs = u;
    out.m = m;
    out.x.assign(D, nullptr);
    out.y.assign(D, nullptr);
    out.z.assign(D, nullptr);
    out.streams.assign(D, nullptr);
    const size_t bytes = m * sizeof(double);
    for (size_t i = 0; i < D; ++i) {
        CK(cudaSetDevice(u[i]));
        CK(cudaStreamCreateWithFlags(&out.streams[i], cudaStreamNonBlocking));
        CK(cudaMalloc(reinterpret_cast<void**>(&out.x[i]), std::max<size_t>(bytes, 8)));
        CK(cudaMalloc(reinterpret_cast<void**>(&out.y[i]), std::max<size_t>(bytes, 8)));
        if (hz) CK(cudaMalloc(reinterpret_cast<void**>(&out.z[i]), std::max<size_t>(bytes, 8)));
    }
    // one host -> device copy, to the root device
    CK(cudaSetDevice(u[0]));
    if (m) {
        CK(cudaMemcpyAsync(out.x[0], hx, bytes, cudaMemcpyHostToDevice, out.streams[0]));
        CK(cudaMemcpyAsync(out.y[0], hy, bytes, cudaMemcpyHostToDevice, out.streams[0]));
        if (hz) CK(cudaMemcpyAsync(out.z[0], hz, bytes, cudaMemcpyHostToDevice, out.streams[0]));
    }
    CK(cudaStreamSynchronize(out.streams[0]));
    NcclApi& api = nccl();
    if (api.ok && m) {
        std::lock_guard<std::mutex> lk(g_comm_mu);
        auto it = g_comms.find(u);
        if (it == g_comms.end()) {
            std::vector<ncclComm_t> comms(D, nullptr);
            nck(api.init_all(comms.data(), static_cast<int>(D), u.data()), "ncclCommInitAll");
            it = g_comms.emplace(u, std::move(comms)).first;
        }
        const std::vector<ncclComm_t>& comms = it->second;
        nck(api.group_start(), "ncclGroupStart");
        for (size_t i = 0; i < D; ++i) {
            CK(cudaSetDevice(u[i]));
            for (int a = 0; a < (hz ? 3 : 2); ++a) {
                double* buf = a == 0 ? out.x[i] : a == 1 ? out.y[i] : out.z[i];
                const double* src = a == 0 ? out.x[0] : a == 1 ? out.y[0] : out.z[0];
                // root rank 0 sends its buffer in place; every rank receives
                nck(api.broadcast(i == 0 ? src : buf, buf, m, ncclFloat64, 0, comms[i],
                                  out.streams[i]),
                    "ncclBroadcast");
            }
        }
        nck(api.group_end(), "ncclGroupEnd");
        g_broadcasts.fetch_add(1);
        out.kind = kReplicateNccl;
    } else if (m) {
        for (size_t i = 1; i < D; ++i) {
            CK(cudaSetDevice(u[i]));
            CK(cudaMemcpyPeerAsync(out.x[i], u[i], out.x[0], u[0], bytes, out.streams[i]));
            CK(cudaMemcpyPeerAsync(out.y[i], u[i], out.y[0], u[0], bytes, out.streams[i]));
            if (hz) CK(cudaMemcpyPeerAsync(out.z[i], u[i], out.z[0], u[0], bytes, out.streams[i]));
        }
        out.kind = kReplicatePeer;
    }
    for (size_t i = 0; i < D; ++i) {
        CK(cudaSetDevice(u[i]));
        CK(cudaStreamSynchronize(out.streams[i]));
    }
    g_last_kind.store(out.kind);
}

}  // namespace aidwb
