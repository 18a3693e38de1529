// comm.cu — allgather transports for node-range sharding (comm.cuh) and the
// dhgp_comm_* C-ABI.  NCCL is resolved from libnccl.so.2 at run time (the
// copy the host process already loaded — torch's — when there is one), so
// libdhgp.so has no link-time NCCL dependency.
#include <dlfcn.h>

#include <mutex>

#include "comm.cuh"

namespace dhgp {

namespace {
struct NcclUniqueId {
    char internal[128];
};
struct NcclApi {
    bool loaded = false;
    std::string error;
    int (*GetUniqueId)(NcclUniqueId *) = nullptr;
    int (*CommInitRank)(void **, int, NcclUniqueId, int) = nullptr;
    int (*AllGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
    int (*CommDestroy)(void *) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
};
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (torch's)
        const char *env = getenv("DHGP_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        api.GetUniqueId = (int (*)(NcclUniqueId *))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (int (*)(void **, int, NcclUniqueId, int))dlsym(h, "ncclCommInitRank");
        api.AllGather = (int (*)(const void *, void *, size_t, int, void *, cudaStream_t))dlsym(h, "ncclAllGather");
        api.CommDestroy = (int (*)(void *))dlsym(h, "ncclCommDestroy");
        api.GetErrorString = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy) {
            api.error = "libnccl.so.2 lacks the NCCL 2.x entry points";
            return;
        }
        api.loaded = true;
    });
    if (!api.loaded) throw Error{DHGP_ERR_CUDA, api.error};
    return api;
}

void nccl_check(int r, const char *what) {
    if (r != 0) {
        const char *m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw Error{DHGP_ERR_CUDA, std::string(what) + ": " + m};
    }
}
}  // namespace

Shard shard_of(const Comm *cm, int64_t n) {
    Shard s;
    s.lo = 0;
    s.hi = n;
    s.chunk = n;
    if (!cm || (cm->world <= 1 && !cm->exercise) || n < cm->min_units || n <= 0) return s;
    s.on = true;
    s.chunk = cdiv(n, cm->world);
    s.lo = std::min<int64_t>(n, (int64_t)cm->rank * s.chunk);
    s.hi = std::min<int64_t>(n, s.lo + s.chunk);
    return s;
}

int64_t shard_capacity(const Comm *cm, int64_t n) {
    if (!cm) return n;
    return std::max<int64_t>(n, cdiv(n, cm->world) * cm->world);
}

void allgather(Ctx &c, Comm *cm, void *buf, size_t elem, int64_t chunk) {
    if (!cm || (cm->world <= 1 && !cm->exercise) || chunk <= 0) return;
    const size_t part = (size_t)chunk * elem;
    cm->calls++;
    cm->bytes += (double)part * (cm->world - 1);
    if (cm->kind == DHGP_COMM_NCCL) {
        char *b = (char *)buf;
        nccl_check(nccl().AllGather(b + (size_t)cm->rank * part, b, part, kNcclUint8, cm->nccl, c.stream),
                   "ncclAllGather");
        return;
    }
    // host mode: stage this rank's part, exchange on the host, copy back
    const size_t total = part * cm->world;
    if (cm->pinned_cap < total) {
        if (cm->pinned) cudaFreeHost(cm->pinned);
        cm->pinned = nullptr;
        cm->pinned_cap = 0;
        DHGP_CUDA(cudaMallocHost(&cm->pinned, total));
        cm->pinned_cap = total;
    }
    char *h = (char *)cm->pinned;
    DHGP_CUDA(cudaMemcpyAsync(h + (size_t)cm->rank * part, (char *)buf + (size_t)cm->rank * part, part,
                              cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (cm->fn(cm->user, h, (int64_t)part) != 0) throw Error{DHGP_ERR_CUDA, "host allgather callback failed"};
    DHGP_CUDA(cudaMemcpyAsync(buf, h, total, cudaMemcpyHostToDevice, c.stream));
}

namespace {
template <class T, bool MAX>
__global__ void k_reduce_ranks(int64_t n, int world, const T *parts, T *out) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T v = parts[i];
        for (int r = 1; r < world; r++) {
            const T x = parts[(int64_t)r * n + i];
            v = MAX ? (x > v ? x : v) : (T)(v + x);
        }
        out[i] = v;
    }
}
template <class T, bool MAX>
void allreduce(Ctx &c, Comm *cm, T *buf, int64_t n) {
    if (!comm_active(cm) || n <= 0) return;
    T *parts = c.alloc<T>((int64_t)cm->world * n);
    c.d2d(parts + (int64_t)cm->rank * n, buf, n);
    allgather(c, cm, parts, sizeof(T), n);
    pdl_launch(k_reduce_ranks<T, MAX>, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4096)), 256, 0,
               c.stream, n, cm->world, (const T *)parts, buf);
    DHGP_LAUNCHED(c);
    c.free(parts);
}
}  // namespace

void allreduce_max_u64(Ctx &c, Comm *cm, unsigned long long *buf, int64_t n) {
    allreduce<unsigned long long, true>(c, cm, buf, n);
}
void allreduce_sum_i64(Ctx &c, Comm *cm, long long *buf, int64_t n) { allreduce<long long, false>(c, cm, buf, n); }
void allreduce_sum_i32(Ctx &c, Comm *cm, int32_t *buf, int64_t n) { allreduce<int32_t, false>(c, cm, buf, n); }

}  // namespace dhgp

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace dhgp;

struct dhgp_comm {
    Comm c;
};

extern "C" {

int dhgp_comm_nccl_unique_id(uint8_t *id_out) {
    try {
        NcclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        memcpy(id_out, id.internal, sizeof id.internal);
        return DHGP_OK;
    } catch (const Error &e) {
        set_error(e.code, e.msg);
        return e.code;
    }
}

int dhgp_comm_init_nccl(int32_t world, int32_t rank, const uint8_t *id, int32_t device, dhgp_comm **out) {
    try {
        if (world < 1 || rank < 0 || rank >= world || !id || !out) throw Error{DHGP_ERR_ARG, "bad communicator arguments"};
        DHGP_CUDA(cudaSetDevice(device));
        NcclUniqueId uid;
        memcpy(uid.internal, id, sizeof uid.internal);
        dhgp_comm *cm = new dhgp_comm();
        cm->c.world = world;
        cm->c.rank = rank;
        cm->c.device = device;
        cm->c.kind = DHGP_COMM_NCCL;
        const char *ex = getenv("DHGP_COMM_EXERCISE");
        cm->c.exercise = ex && ex[0] == '1';
        int r = nccl().CommInitRank(&cm->c.nccl, world, uid, rank);
        if (r != 0) {
            delete cm;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = cm;
        return DHGP_OK;
    } catch (const Error &e) {
        set_error(e.code, e.msg);
        return e.code;
    }
}

int dhgp_comm_init_host(int32_t world, int32_t rank, dhgp_allgather_fn fn, void *user, dhgp_comm **out) {
    if (world < 1 || rank < 0 || rank >= world || !fn || !out) {
        set_error(DHGP_ERR_ARG, "bad communicator arguments");
        return DHGP_ERR_ARG;
    }
    dhgp_comm *cm = new dhgp_comm();
    cm->c.world = world;
    cm->c.rank = rank;
    cm->c.kind = DHGP_COMM_HOST;
    const char *ex = getenv("DHGP_COMM_EXERCISE");
    cm->c.exercise = ex && ex[0] == '1';
    cm->c.fn = fn;
    cm->c.user = user;
    *out = cm;
    return DHGP_OK;
}

int dhgp_comm_set_min_units(dhgp_comm *cm, int64_t min_units) {
    if (!cm || min_units < 0) {
        set_error(DHGP_ERR_ARG, "bad communicator arguments");
        return DHGP_ERR_ARG;
    }
    cm->c.min_units = min_units;
    return DHGP_OK;
}

int dhgp_comm_stats(const dhgp_comm *cm, int64_t *allgathers, double *bytes) {
    if (!cm) return DHGP_ERR_ARG;
    if (allgathers) *allgathers = cm->c.calls;
    if (bytes) *bytes = cm->c.bytes;
    return DHGP_OK;
}

int dhgp_shard_range(int32_t world, int32_t rank, int64_t min_units, int64_t n, int64_t *lo, int64_t *hi,
                     int64_t *chunk) {
    Comm cm;
    cm.world = world;
    cm.rank = rank;
    cm.min_units = min_units;
    const Shard s = shard_of(&cm, n);
    if (lo) *lo = s.lo;
    if (hi) *hi = s.hi;
    if (chunk) *chunk = s.chunk;
    return s.on ? 1 : 0;
}

void dhgp_comm_destroy(dhgp_comm *cm) {
    if (!cm) return;
    if (cm->c.kind == DHGP_COMM_NCCL && cm->c.nccl) {
        try {
            nccl().CommDestroy(cm->c.nccl);
        } catch (...) {
        }
    }
    if (cm->c.pinned) cudaFreeHost(cm->c.pinned);
    delete cm;
}

}  // extern "C"

Comm *comm_of(dhgp_comm *cm) { return cm ? &cm->c : nullptr; }
