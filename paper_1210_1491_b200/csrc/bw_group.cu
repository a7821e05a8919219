// bw_group.cu — the DtN path and the config-5 pipeline over several GPUs of one
// process: one bw_ctx per device, an NCCL communicator over them.
//
// The reference parallelises estimate_u_batch over worker threads with a
// static block partition and guarantees results independent of the worker
// count (wos.hpp:19,43-44; parallel.hpp:14-40). Here the unit of work is a
// boundary point: point b runs on device b mod n (strided: cavity and face
// points interleave, so the shards cost the same), keeps its global stream ids,
// and every device runs the single-device path on its shard from its own host
// thread (the per-device calls are independent and synchronous). The only
// exchange is the pipeline's all-gather of the 72-byte panel records before the
// potential sum (ncclAllGather over NVLink; ncclCommInitAll). Per-point and
// per-target results are bitwise identical for any device count: a point's
// Neumann value depends on its own streams and its class tables only, and every
// device sums the panels in the same (global) order.
#include <dlfcn.h>
#include <nccl.h> // types only: NCCL is loaded at run time (nccl_api below)

#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bw_internal.h"

using bw::cuda_check;

struct bw_group {
    int n = 0;
    std::vector<int> dev;
    std::vector<bw_ctx*> ctx;
    std::vector<ncclComm_t> comm; // empty when a device id repeats (no NCCL)
    std::string err;
};

namespace {

// NCCL entry points, resolved with dlopen when the first multi-device group is
// created. Not linked: a process that loads this library before torch would
// otherwise bind the soname libnccl.so.2 to the system NCCL and break torch's
// newer one (and the reverse). An NCCL already in the process (torch's) is
// reused; else BW_NCCL_LIBRARY, else libnccl.so.2 from the loader path.
struct NcclApi {
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("BW_NCCL_LIBRARY");
            if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        api.comm_init_all = (decltype(api.comm_init_all))dlsym(h, "ncclCommInitAll");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
        api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.comm_init_all && api.comm_destroy && api.all_gather && api.group_start &&
                 api.group_end && api.error_string;
    });
    return api;
}

bw_status gfail(bw_group* g, bw_status st, const std::string& msg) {
    g->err = msg;
    return st;
}

// Worst status of the per-device calls in the reference's exception order: hard
// errors first, then the soft ones whose outputs are still written.
bw_status combine(bw_group* g, const std::vector<bw_status>& st) {
    bw_status soft = BW_OK;
    for (int i = 0; i < g->n; ++i) {
        if (st[i] == BW_OK) continue;
        if (st[i] == BW_ERR_RELIABILITY || st[i] == BW_ERR_SOLVER) {
            if (soft == BW_OK) {
                soft = st[i];
                g->err = std::string("device ") + std::to_string(g->dev[i]) + ": " +
                         bw_last_error(g->ctx[i]);
            }
            continue;
        }
        g->err = std::string("device ") + std::to_string(g->dev[i]) + ": " + bw_last_error(g->ctx[i]);
        return st[i];
    }
    return soft;
}

template <class F>
std::vector<bw_status> on_each(bw_group* g, F f) {
    std::vector<bw_status> st((size_t)g->n, BW_OK);
    if (g->n == 1) {
        st[0] = f(0);
        return st;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < g->n; ++i) th.emplace_back([&, i] { st[(size_t)i] = f(i); });
    for (auto& t : th) t.join();
    return st;
}

int64_t shard_count(int64_t n, int i, int g) { return n > i ? (n - i + g - 1) / g : 0; }

// Host-side strided shard of a boundary-point batch.
struct Shard {
    std::vector<bw_patch> patches;
    std::vector<int64_t> ids;
    std::vector<double> dudn, err, area, u;
    std::vector<int32_t> status;
};

void make_shards(int g, const bw_patch* patches, const int64_t* bp_ids, int64_t n_bp,
                 const double* area, const double* u_bp, std::vector<Shard>& sh) {
    sh.assign((size_t)g, Shard{});
    for (int i = 0; i < g; ++i) {
        const int64_t m = shard_count(n_bp, i, g);
        Shard& s = sh[(size_t)i];
        s.patches.resize((size_t)m);
        s.ids.resize((size_t)m);
        s.dudn.resize((size_t)m);
        s.err.resize((size_t)m);
        s.status.resize((size_t)m);
        if (area) s.area.resize((size_t)m);
        if (u_bp) s.u.resize((size_t)m);
        for (int64_t k = 0; k < m; ++k) {
            const int64_t b = i + k * g;
            s.patches[(size_t)k] = patches[b];
            s.ids[(size_t)k] = bp_ids ? bp_ids[b] : b;
            if (area) s.area[(size_t)k] = area[b];
            if (u_bp) s.u[(size_t)k] = u_bp[b];
        }
    }
}

void unshard(int g, int64_t n_bp, const std::vector<Shard>& sh, double* dudn, double* err,
             int32_t* status) {
    for (int i = 0; i < g; ++i)
        for (int64_t k = 0; k < (int64_t)sh[(size_t)i].ids.size(); ++k) {
            const int64_t b = i + k * g;
            if (b >= n_bp) break;
            dudn[b] = sh[(size_t)i].dudn[(size_t)k];
            err[b] = sh[(size_t)i].err[(size_t)k];
            status[b] = sh[(size_t)i].status[(size_t)k];
        }
}

// Panel records {p, n, area, u, dudn} of a device's shard (field_eval.hpp:12-18;
// normal and dudn INTO the solution domain: dudn_in = -dudn_outward), written
// to slot k of the send buffer; slots past the shard stay zero.
__global__ void panel_records_kernel(const bw_patch* __restrict__ p, const double* __restrict__ area,
                                     const double* __restrict__ u, const double* __restrict__ dudn,
                                     int64_t m, double* __restrict__ rec) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        double* r = rec + 9 * k;
        r[0] = p[k].o[0];
        r[1] = p[k].o[1];
        r[2] = p[k].o[2];
        r[3] = p[k].axis[0];
        r[4] = p[k].axis[1];
        r[5] = p[k].axis[2];
        r[6] = area[k];
        r[7] = u[k];
        r[8] = -dudn[k];
    }
}

// all-gathered [rank][slot] records -> global point order b = slot * g + rank
__global__ void unstride_kernel(const double* __restrict__ gathered, int64_t n_bp, int g,
                                int64_t cnt, double* __restrict__ panels) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 9 * n_bp;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / 9, j = e - b * 9;
        panels[e] = gathered[((b % g) * cnt + b / g) * 9 + j];
    }
}

// sum of the per-node walk step counts of a shard (int64, one atomic per block)
__global__ void sum_steps_kernel(const int64_t* __restrict__ steps, int64_t n,
                                 unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        s += (unsigned long long)steps[k];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

struct DevBuf {
    int64_t* steps = nullptr;
    unsigned long long* steps_sum = nullptr;
    bw_patch* patches = nullptr;
    int64_t* ids = nullptr;
    double *dirs = nullptr, *wts = nullptr, *dudn = nullptr, *err = nullptr, *area = nullptr,
           *u = nullptr, *send = nullptr, *recv = nullptr, *panels = nullptr, *targets = nullptr,
           *pot = nullptr;
    int32_t* status = nullptr;
    uint8_t* near = nullptr;
    void free_all() {
        void* ps[] = {patches, ids, dirs, wts, dudn, err, area, u, send, recv, panels, targets, pot,
                      status, near, steps, steps_sum};
        for (void* q : ps)
            if (q) cudaFree(q);
    }
};

template <class T>
cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc((void**)p, sizeof(T) * std::max<size_t>(n, 1));
}

// One device's share of the DtN path: H2D of its strided shard, K1 -> K7
// (bw_dtn_solve_d), optionally the panel records of the shard (pipeline), the
// sum of its walk steps, and D2H of its Neumann data. Events 0/1 bracket it.
bw_status dtn_phase(bw_group* g, int i, std::vector<DevBuf>& buf, std::vector<Shard>& sh,
                    std::vector<cudaEvent_t>& ev, const bw_scene* scene, const bw_wos_config* wos,
                    const bw_dtn_config* cfg, const double* local_dirs, const double* weights,
                    int32_t n_cls, int32_t n_nodes, uint64_t point_id_base, int64_t cnt,
                    bool records, int64_t n_bp, unsigned long long* steps_host) {
    BW_RANGE("group: device shard DtN");
    bw_ctx* c = g->ctx[(size_t)i];
    DevBuf& d = buf[(size_t)i];
    Shard& s = sh[(size_t)i];
    const int64_t m = (int64_t)s.ids.size();
    cudaSetDevice(g->dev[(size_t)i]);
    cudaStream_t strm = (cudaStream_t)nullptr;
    for (int k = 0; k < 5; ++k) cudaEventCreate(&ev[(size_t)i * 5 + k]);
    cudaError_t e = cudaSuccess;
    e = e ? e : dalloc(&d.patches, (size_t)m);
    e = e ? e : dalloc(&d.ids, (size_t)m);
    e = e ? e : dalloc(&d.dirs, 3 * (size_t)n_cls * n_nodes);
    e = e ? e : dalloc(&d.wts, (size_t)n_cls * n_nodes);
    e = e ? e : dalloc(&d.dudn, (size_t)m);
    e = e ? e : dalloc(&d.err, (size_t)m);
    e = e ? e : dalloc(&d.status, (size_t)m);
    e = e ? e : dalloc(&d.steps, (size_t)m * n_nodes);
    e = e ? e : dalloc(&d.steps_sum, 1);
    if (records) {
        e = e ? e : dalloc(&d.area, (size_t)m);
        e = e ? e : dalloc(&d.u, (size_t)m);
        e = e ? e : dalloc(&d.send, 9 * (size_t)cnt);
        e = e ? e : dalloc(&d.recv, 9 * (size_t)cnt * g->n);
        e = e ? e : dalloc(&d.panels, 9 * (size_t)n_bp);
    }
    if (e) return cuda_check(c, e, "group alloc");
    bw_set_stream(c, strm);
    cudaEventRecord(ev[(size_t)i * 5 + 0], strm);
    e = e ? e : cudaMemcpyAsync(d.patches, s.patches.data(), sizeof(bw_patch) * m, cudaMemcpyHostToDevice, strm);
    e = e ? e : cudaMemcpyAsync(d.ids, s.ids.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, strm);
    e = e ? e : cudaMemcpyAsync(d.dirs, local_dirs, sizeof(double) * 3 * n_cls * n_nodes, cudaMemcpyHostToDevice, strm);
    e = e ? e : cudaMemcpyAsync(d.wts, weights, sizeof(double) * n_cls * n_nodes, cudaMemcpyHostToDevice, strm);
    e = e ? e : cudaMemsetAsync(d.steps_sum, 0, sizeof(unsigned long long), strm);
    if (records) {
        e = e ? e : cudaMemcpyAsync(d.area, s.area.data(), sizeof(double) * m, cudaMemcpyHostToDevice, strm);
        e = e ? e : cudaMemcpyAsync(d.u, s.u.data(), sizeof(double) * m, cudaMemcpyHostToDevice, strm);
        e = e ? e : cudaMemsetAsync(d.send, 0, sizeof(double) * 9 * cnt, strm);
    }
    if (e) return cuda_check(c, e, "group H2D");
    bw_status r = BW_OK;
    if (m > 0) {
        r = bw_dtn_solve_d(c, scene, wos, cfg, d.patches, d.ids, m, d.dirs, d.wts, n_cls, n_nodes,
                           point_id_base, d.dudn, d.err, d.status, nullptr, d.steps);
        if (r != BW_OK && r != BW_ERR_RELIABILITY && r != BW_ERR_SOLVER) return r;
        ++c->launches;
        sum_steps_kernel<<<(unsigned)std::min<int64_t>((m * n_nodes + 255) / 256, 1184), 256, 0, strm>>>(
            d.steps, m * n_nodes, d.steps_sum);
        if (records) {
            ++c->launches;
            panel_records_kernel<<<(unsigned)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, strm>>>(
                d.patches, d.area, d.u, d.dudn, m, d.send);
        }
        if ((e = cudaGetLastError())) return cuda_check(c, e, "group kernels");
    }
    cudaEventRecord(ev[(size_t)i * 5 + 1], strm);
    e = e ? e : cudaMemcpyAsync(s.dudn.data(), d.dudn, sizeof(double) * m, cudaMemcpyDeviceToHost, strm);
    e = e ? e : cudaMemcpyAsync(s.err.data(), d.err, sizeof(double) * m, cudaMemcpyDeviceToHost, strm);
    e = e ? e : cudaMemcpyAsync(s.status.data(), d.status, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, strm);
    e = e ? e : cudaMemcpyAsync(steps_host, d.steps_sum, sizeof(unsigned long long), cudaMemcpyDeviceToHost, strm);
    e = e ? e : cudaStreamSynchronize(strm);
    if (e) return cuda_check(c, e, "group D2H");
    return r;
}

void free_bufs(bw_group* g, std::vector<DevBuf>& buf, std::vector<cudaEvent_t>& ev) {
    for (int i = 0; i < g->n; ++i) {
        cudaSetDevice(g->dev[(size_t)i]);
        buf[(size_t)i].free_all();
        for (int k = 0; k < 5; ++k)
            if (ev[(size_t)i * 5 + k]) cudaEventDestroy(ev[(size_t)i * 5 + k]);
    }
}

} // namespace

extern "C" {

bw_status bw_group_init(int n_dev, const int* devices, bw_group** out) {
    if (!out) return BW_ERR_INVALID;
    *out = nullptr;
    if (n_dev < 1 || !devices) return BW_ERR_INVALID;
    bw_group* g = new bw_group;
    g->n = n_dev;
    g->dev.assign(devices, devices + n_dev);
    for (int i = 0; i < n_dev; ++i) {
        bw_ctx* c = nullptr;
        const bw_status st = bw_init(devices[i], &c);
        if (st != BW_OK) {
            for (bw_ctx* x : g->ctx) bw_finalize(x);
            delete g;
            return st;
        }
        g->ctx.push_back(c);
    }
    std::vector<int> sorted = g->dev;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (distinct) {
        const NcclApi& nc = nccl_api();
        g->comm.resize((size_t)n_dev);
        if (!nc.ok || nc.comm_init_all(g->comm.data(), n_dev, g->dev.data()) != ncclSuccess) {
            for (bw_ctx* x : g->ctx) bw_finalize(x);
            delete g;
            return BW_ERR_CUDA;
        }
    }
    *out = g;
    return BW_OK;
}

bw_status bw_group_finalize(bw_group* g) {
    if (!g) return BW_OK;
    for (ncclComm_t c : g->comm) nccl_api().comm_destroy(c);
    for (bw_ctx* c : g->ctx) bw_finalize(c);
    delete g;
    return BW_OK;
}

bw_status bw_group_size(const bw_group* g, int32_t* n, int32_t* uses_nccl) {
    if (!g || !n) return BW_ERR_INVALID;
    *n = g->n;
    if (uses_nccl) *uses_nccl = g->comm.empty() ? 0 : 1;
    return BW_OK;
}

bw_ctx* bw_group_context(bw_group* g, int32_t i) {
    return (g && i >= 0 && i < g->n) ? g->ctx[(size_t)i] : nullptr;
}

const char* bw_group_last_error(const bw_group* g) { return g ? g->err.c_str() : "null group"; }

bw_status bw_group_launch_count(const bw_group* g, uint64_t* count) {
    if (!g || !count) return BW_ERR_INVALID;
    uint64_t s = 0;
    for (bw_ctx* c : g->ctx) {
        uint64_t k = 0;
        bw_launch_count(c, &k);
        s += k;
    }
    *count = s;
    return BW_OK;
}

bw_status bw_group_dtn_solve(bw_group* g, const bw_scene* scene, const bw_wos_config* wos,
                             const bw_dtn_config* cfg, const bw_patch* patches,
                             const int64_t* bp_ids, int64_t n_bp, const double* local_dirs,
                             const double* weights, int32_t n_cls, int32_t n_nodes,
                             uint64_t point_id_base, double* dudn, double* err, int32_t* status,
                             int64_t* walk_steps, double* device_ms) {
    BW_RANGE("bw_group_dtn_solve");
    if (!g) return BW_ERR_INVALID;
    if (n_bp < 0 || n_nodes < 1 || n_cls < 1 ||
        (n_bp > 0 && (!patches || !local_dirs || !weights || !dudn || !err || !status)))
        return gfail(g, BW_ERR_INVALID, "bad arguments");
    if (walk_steps) *walk_steps = 0;
    if (n_bp == 0) return BW_OK;
    const int G = g->n;
    std::vector<Shard> sh;
    make_shards(G, patches, bp_ids, n_bp, nullptr, nullptr, sh);
    std::vector<DevBuf> buf((size_t)G);
    std::vector<cudaEvent_t> ev((size_t)G * 5, nullptr);
    std::vector<unsigned long long> steps((size_t)G, 0ull);
    const auto st = on_each(g, [&](int i) {
        return dtn_phase(g, i, buf, sh, ev, scene, wos, cfg, local_dirs, weights, n_cls, n_nodes,
                         point_id_base, 0, false, n_bp, &steps[(size_t)i]);
    });
    const bw_status r = combine(g, st);
    if (r == BW_OK || r == BW_ERR_RELIABILITY || r == BW_ERR_SOLVER) {
        unshard(G, n_bp, sh, dudn, err, status);
        if (walk_steps)
            for (unsigned long long v : steps) *walk_steps += (int64_t)v;
        if (device_ms) {
            *device_ms = 0;
            for (int i = 0; i < G; ++i) {
                cudaSetDevice(g->dev[(size_t)i]);
                float a = 0;
                cudaEventElapsedTime(&a, ev[(size_t)i * 5 + 0], ev[(size_t)i * 5 + 1]);
                *device_ms = std::max(*device_ms, (double)a);
            }
        }
    }
    free_bufs(g, buf, ev);
    return r;
}

bw_status bw_group_pipeline(bw_group* g, const bw_scene* scene, const bw_wos_config* wos,
                            const bw_dtn_config* cfg, const bw_patch* patches, int64_t n_bp,
                            const double* local_dirs, const double* weights, int32_t n_cls,
                            int32_t n_nodes, uint64_t point_id_base, const double* area,
                            const double* u_bp, const double* targets, int64_t n_t, double* u,
                            uint8_t* near, double* dudn, double* err, int32_t* status,
                            int64_t* walk_steps, double* phase_ms) {
    BW_RANGE("bw_group_pipeline");
    if (!g) return BW_ERR_INVALID;
    if (n_bp < 1 || n_t < 0 || n_nodes < 1 || n_cls < 1 || !patches || !local_dirs || !weights ||
        !area || !u_bp || (n_t > 0 && (!targets || !u || !near)))
        return gfail(g, BW_ERR_INVALID, "bad arguments");
    const int G = g->n;
    std::vector<Shard> sh;
    make_shards(G, patches, nullptr, n_bp, area, u_bp, sh);
    const int64_t cnt = shard_count(n_bp, 0, G); // records per rank in the all-gather
    std::vector<DevBuf> buf((size_t)G);
    std::vector<cudaEvent_t> ev((size_t)G * 5, nullptr);
    std::vector<unsigned long long> steps((size_t)G, 0ull);
    auto cleanup = [&] { free_bufs(g, buf, ev); };
    // phase 1: each device's shard, DtN (K1 -> K7) and its panel records
    auto st = on_each(g, [&](int i) {
        return dtn_phase(g, i, buf, sh, ev, scene, wos, cfg, local_dirs, weights, n_cls, n_nodes,
                         point_id_base, cnt, true, n_bp, &steps[(size_t)i]);
    });
    bw_status r = combine(g, st);
    if (r != BW_OK && r != BW_ERR_RELIABILITY && r != BW_ERR_SOLVER) {
        cleanup();
        return r;
    }
    const bw_status soft = r;
    // phase 2: all-gather of the panel records
    if (!g->comm.empty()) {
        BW_RANGE("group: ncclAllGather of the panel records");
        const NcclApi& nc = nccl_api();
        ncclResult_t nr = nc.group_start();
        for (int i = 0; i < G && nr == ncclSuccess; ++i) {
            cudaSetDevice(g->dev[(size_t)i]);
            nr = nc.all_gather(buf[(size_t)i].send, buf[(size_t)i].recv, 9 * (size_t)cnt, ncclDouble,
                               g->comm[(size_t)i], (cudaStream_t)nullptr);
        }
        const ncclResult_t ne = nc.group_end();
        if (nr != ncclSuccess || ne != ncclSuccess) {
            cleanup();
            return gfail(g, BW_ERR_CUDA, std::string("ncclAllGather: ") +
                                             nc.error_string(nr != ncclSuccess ? nr : ne));
        }
    } else {
        // a device id repeats (one GPU standing for several ranks, tests only):
        // plain device-to-device copies in rank order
        for (int i = 0; i < G; ++i) {
            cudaSetDevice(g->dev[(size_t)i]);
            for (int j = 0; j < G; ++j) {
                const cudaError_t e = cudaMemcpyPeerAsync(
                    buf[(size_t)i].recv + (size_t)j * 9 * cnt, g->dev[(size_t)i], buf[(size_t)j].send,
                    g->dev[(size_t)j], sizeof(double) * 9 * cnt, (cudaStream_t)nullptr);
                if (e) {
                    cleanup();
                    return gfail(g, BW_ERR_CUDA, cudaGetErrorString(e));
                }
            }
        }
    }
    // phase 3: global panel order, this device's strided share of the targets, K3
    std::vector<std::vector<double>> tgt((size_t)G), pot((size_t)G);
    std::vector<std::vector<uint8_t>> nr((size_t)G);
    st = on_each(g, [&](int i) -> bw_status {
        bw_ctx* c = g->ctx[(size_t)i];
        DevBuf& d = buf[(size_t)i];
        cudaSetDevice(g->dev[(size_t)i]);
        cudaStream_t strm = (cudaStream_t)nullptr;
        cudaEventRecord(ev[(size_t)i * 5 + 2], strm);
        unstride_kernel<<<(unsigned)std::min<int64_t>((9 * n_bp + 255) / 256, 8192), 256, 0, strm>>>(
            d.recv, n_bp, G, cnt, d.panels);
        cudaError_t e = cudaGetLastError();
        const int64_t mt = shard_count(n_t, i, G);
        ++c->launches;
        auto& t = tgt[(size_t)i];
        t.resize(3 * (size_t)mt);
        for (int64_t k = 0; k < mt; ++k)
            std::memcpy(&t[3 * (size_t)k], targets + 3 * (i + k * G), 3 * sizeof(double));
        pot[(size_t)i].resize((size_t)mt);
        nr[(size_t)i].resize((size_t)mt);
        e = e ? e : dalloc(&d.targets, 3 * (size_t)mt);
        e = e ? e : dalloc(&d.pot, (size_t)mt);
        e = e ? e : dalloc(&d.near, (size_t)mt);
        e = e ? e : cudaMemcpyAsync(d.targets, t.data(), sizeof(double) * 3 * mt, cudaMemcpyHostToDevice, strm);
        if (e) return cuda_check(c, e, "group targets");
        cudaEventRecord(ev[(size_t)i * 5 + 3], strm);
        bw_status rr = BW_OK;
        if (mt > 0) {
            int64_t nc = 0;
            rr = bw_potential_d(c, d.panels, n_bp, d.targets, mt, d.pot, d.near, &nc);
            if (rr) return rr;
        }
        cudaEventRecord(ev[(size_t)i * 5 + 4], strm);
        e = e ? e : cudaMemcpyAsync(pot[(size_t)i].data(), d.pot, sizeof(double) * mt, cudaMemcpyDeviceToHost, strm);
        e = e ? e : cudaMemcpyAsync(nr[(size_t)i].data(), d.near, (size_t)mt, cudaMemcpyDeviceToHost, strm);
        e = e ? e : cudaStreamSynchronize(strm);
        return e ? cuda_check(c, e, "group D2H") : BW_OK;
    });
    r = combine(g, st);
    if (r == BW_OK) {
        unshard(G, n_bp, sh, dudn ? dudn : std::vector<double>((size_t)n_bp).data(),
                err ? err : std::vector<double>((size_t)n_bp).data(),
                status ? status : std::vector<int32_t>((size_t)n_bp).data());
        for (int i = 0; i < G; ++i)
            for (int64_t k = 0; k < (int64_t)pot[(size_t)i].size(); ++k) {
                u[i + k * G] = pot[(size_t)i][(size_t)k];
                near[i + k * G] = nr[(size_t)i][(size_t)k];
            }
        if (walk_steps) {
            *walk_steps = 0;
            for (unsigned long long v : steps) *walk_steps += (int64_t)v;
        }
        if (phase_ms) {
            // max over devices: DtN (H2D + K1 + K7 + records), all-gather + reorder,
            // potential (K3)
            double ph[3] = {0, 0, 0};
            for (int i = 0; i < G; ++i) {
                cudaSetDevice(g->dev[(size_t)i]);
                float a = 0, b = 0, c = 0;
                cudaEventElapsedTime(&a, ev[(size_t)i * 5 + 0], ev[(size_t)i * 5 + 1]);
                cudaEventElapsedTime(&b, ev[(size_t)i * 5 + 1], ev[(size_t)i * 5 + 3]);
                cudaEventElapsedTime(&c, ev[(size_t)i * 5 + 3], ev[(size_t)i * 5 + 4]);
                ph[0] = std::max(ph[0], (double)a);
                ph[1] = std::max(ph[1], (double)b);
                ph[2] = std::max(ph[2], (double)c);
            }
            std::memcpy(phase_ms, ph, sizeof ph);
        }
    }
    cleanup();
    return r != BW_OK ? r : soft;
}

} // extern "C"
