// Multi-GPU C-ABI (include/qfuse_b200.h, "multi-GPU, one process"): one
// process drives G devices of the box; device i owns a contiguous shard of
// the batch and runs the whole fused gradient on it (qf_plan_gradient_device),
// and the only exchange is one ncclAllReduce(sum, fp64) of [grad | loss] over
// NVLink/NVSwitch, enqueued on each device's plan stream right behind the
// finalize kernel. The reference has no multi-device path; its
// loss and gradient are sums over samples (engine.cpp:733-738, :686-689), which
// is what makes the shard + sum decomposition exact up to fp64 summation order.
//
// Built only on the public single-device C-ABI; NCCL is loaded with dlopen so
// the library itself does not depend on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qfuse_b200.h"
#include "qf_internal.h"

namespace {

struct QfFail : std::runtime_error {
    int code;
    QfFail(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void ok(int rc) {
    if (rc != QF_OK) throw QfFail(rc, qf_last_error());
}
void cuda_ok(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw QfFail(QF_EDEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return QF_OK;
    } catch (const QfFail &e) {
        qfb::set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc &) {
        qfb::set_last_error("host allocation failed");
        return QF_ECAPACITY;
    } catch (const std::exception &e) {
        qfb::set_last_error(e.what());
        return QF_EDEVICE;
    }
}

// The five NCCL entry points the group needs, resolved from libnccl.so.2 (the
// copy torch already loaded in a Python process, else the system one).
struct Nccl {
    ncclResult_t (*comm_init_all)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    std::string load_error;

    void check(ncclResult_t r, const char *what) const {
        if (r != ncclSuccess)
            throw QfFail(QF_EDEVICE, std::string(what) + ": " +
                                         (error_string ? error_string(r) : "NCCL error"));
    }
};

const Nccl &nccl() {
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.load_error = std::string("NCCL unavailable: ") + dlerror();
            return;
        }
        auto sym = [&](const char *name) {
            void *p = dlsym(h, name);
            if (!p) api.load_error = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    });
    if (!api.load_error.empty()) throw QfFail(QF_EDEVICE, api.load_error);
    return api;
}

// Contiguous [start, start + count) of device i's samples; sizes differ by at most one
// (the same split as parallel.shard_range).
void shard(uint32_t batch, int i, int g, uint32_t &start, uint32_t &count) {
    const uint32_t base = batch / uint32_t(g), extra = batch % uint32_t(g);
    start = uint32_t(i) * base + std::min<uint32_t>(uint32_t(i), extra);
    count = base + (uint32_t(i) < extra ? 1u : 0u);
}

// Runs f(0..G-1), f(i) on its own host thread for G > 1; the first failure
// (QfFail / std::exception, with its qf_last_error text) is rethrown here.
template <class F> void on_each_device(int G, F &&f) {
    if (G == 1) {
        f(0);
        return;
    }
    std::vector<std::exception_ptr> err(G);
    std::vector<std::thread> th;
    th.reserve(G);
    for (int i = 0; i < G; ++i)
        th.emplace_back([&, i] {
            try {
                f(i);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    for (auto &t : th) t.join();
    for (auto &e : err)
        if (e) std::rethrow_exception(e);
}

} // namespace

struct qf_group {
    std::vector<int> devices;
    std::vector<qf_ctx *> ctx;
    std::vector<ncclComm_t> comms;
    std::mutex mu; // calls on one group are serialised

    ~qf_group() {
        for (ncclComm_t c : comms)
            if (c) nccl().comm_destroy(c); // non-null only once NCCL was loaded
        for (qf_ctx *c : ctx) qf_ctx_destroy(c);
    }
};

struct qf_group_plan {
    qf_group *group = nullptr;
    uint32_t n = 0, n_params = 0, batch = 0;
    struct Dev {
        qf_plan *plan = nullptr; // null when the shard is empty
        uint32_t start = 0, count = 0;
        double *theta = nullptr, *out = nullptr; // device
        cudaStream_t stream = nullptr;
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    };
    std::vector<Dev> dev;
    double *h_theta = nullptr, *h_out = nullptr; // pinned; h_out = [grad|loss] then expect

    size_t red_len() const { return size_t(n_params) + 1; }

    ~qf_group_plan() {
        for (size_t i = 0; i < dev.size(); ++i) {
            Dev &d = dev[i];
            cudaSetDevice(group->devices[i]);
            if (d.plan) qf_plan_destroy(d.plan);
            if (d.theta) cudaFree(d.theta);
            if (d.out) cudaFree(d.out);
            if (d.ev0) cudaEventDestroy(d.ev0);
            if (d.ev1) cudaEventDestroy(d.ev1);
        }
        if (h_theta) cudaFreeHost(h_theta);
        if (h_out) cudaFreeHost(h_out);
    }
};

namespace {

qf_group *make_group(int n_gpus, const int *devices) {
    int count = 0;
    cuda_ok(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (n_gpus <= 0) throw QfFail(QF_EINVAL, "n_gpus must be positive");
    std::vector<int> devs(n_gpus);
    for (int i = 0; i < n_gpus; ++i) devs[i] = devices ? devices[i] : i;
    for (int i = 0; i < n_gpus; ++i) {
        if (devs[i] < 0 || devs[i] >= count)
            throw QfFail(QF_EINVAL, "no such CUDA device: " + std::to_string(devs[i]) + " (" +
                                        std::to_string(count) + " visible)");
        for (int j = 0; j < i; ++j)
            if (devs[j] == devs[i]) throw QfFail(QF_EINVAL, "duplicate device in group");
    }
    auto g = std::make_unique<qf_group>();
    g->devices = devs;
    for (int d : devs) {
        qf_ctx *c = nullptr;
        ok(qf_ctx_create(d, &c));
        g->ctx.push_back(c);
    }
    const Nccl &api = nccl();
    std::vector<ncclComm_t> comms(n_gpus, nullptr);
    api.check(api.comm_init_all(comms.data(), n_gpus, devs.data()), "ncclCommInitAll");
    g->comms = comms;
    return g.release();
}

qf_group_plan *make_group_plan(qf_group *g, const qf_gate *gates, size_t n_gates, uint32_t n,
                               uint32_t n_params, uint32_t layers, uint32_t ckpt, uint32_t batch,
                               uint64_t x, uint64_t z, uint32_t storage) {
    if (!g) throw QfFail(QF_EINVAL, "null group");
    if (batch == 0) throw QfFail(QF_EINVAL, "batch must be positive");
    const int G = int(g->devices.size());
    auto gp = std::make_unique<qf_group_plan>();
    gp->group = g;
    gp->n = n;
    gp->n_params = n_params;
    gp->batch = batch;
    gp->dev.resize(G);
    for (int i = 0; i < G; ++i) {
        qf_group_plan::Dev &d = gp->dev[i];
        shard(batch, i, G, d.start, d.count);
        cuda_ok(cudaSetDevice(g->devices[i]), "cudaSetDevice");
        if (d.count) {
            ok(qf_plan_create_ex(g->ctx[i], gates, n_gates, n, n_params, layers, ckpt, d.count, x,
                                 z, storage, &d.plan));
            d.stream = static_cast<cudaStream_t>(qf_plan_stream(d.plan));
        } else {
            // an empty shard still takes part in the all-reduce with zeros; it
            // validates the circuit like every other device would
            qf_plan *probe = nullptr;
            ok(qf_plan_create_ex(g->ctx[i], gates, n_gates, n, n_params, layers, ckpt, 1, x, z,
                                 storage, &probe));
            d.stream = static_cast<cudaStream_t>(qf_plan_stream(probe));
            qf_plan_destroy(probe);
        }
        const size_t out_len = size_t(n_params) + 1 + d.count;
        cuda_ok(cudaMalloc(&d.theta, sizeof(double) * std::max<size_t>(1, n_params)), "cudaMalloc");
        cuda_ok(cudaMalloc(&d.out, sizeof(double) * out_len), "cudaMalloc");
        cuda_ok(cudaEventCreate(&d.ev0), "event");
        cuda_ok(cudaEventCreate(&d.ev1), "event");
    }
    cuda_ok(cudaMallocHost(&gp->h_theta, sizeof(double) * std::max<size_t>(1, n_params)),
            "cudaMallocHost");
    cuda_ok(cudaMallocHost(&gp->h_out, sizeof(double) * (gp->red_len() + batch)), "cudaMallocHost");
    return gp.release();
}

void group_gradient(qf_group_plan *gp, const double *theta, double *loss, double *grad,
                    double *expect, qf_stats *stats) {
    if (!gp) throw QfFail(QF_EINVAL, "null group plan");
    if (gp->n_params && !theta) throw QfFail(QF_EINVAL, "gradient: theta length mismatch");
    if (!loss || (gp->n_params && !grad)) throw QfFail(QF_EINVAL, "gradient: null output");
    qf_group *g = gp->group;
    std::lock_guard<std::mutex> lock(g->mu);
    const Nccl &api = nccl();
    const int G = int(gp->dev.size());
    const size_t M = gp->n_params, R = gp->red_len();
    if (M) std::memcpy(gp->h_theta, theta, sizeof(double) * M);
    // 1) every device: theta H2D, the fused gradient of its shard into out. One
    // host thread per device enqueues its ~10^2..10^3 launches, so all G devices
    // start together instead of device i waiting for devices 0..i-1's enqueue.
    auto enqueue = [&](int i) {
        qf_group_plan::Dev &d = gp->dev[i];
        cuda_ok(cudaSetDevice(g->devices[i]), "cudaSetDevice");
        cuda_ok(cudaEventRecord(d.ev0, d.stream), "event");
        if (M)
            cuda_ok(cudaMemcpyAsync(d.theta, gp->h_theta, sizeof(double) * M,
                                    cudaMemcpyHostToDevice, d.stream),
                    "H2D theta");
        if (d.plan)
            ok(qf_plan_gradient_device(d.plan, d.theta, d.out));
        else
            cuda_ok(cudaMemsetAsync(d.out, 0, sizeof(double) * R, d.stream), "memset");
    };
    on_each_device(G, enqueue);
    // 2) the single exchange: [grad | loss] summed over the group, in place
    api.check(api.group_start(), "ncclGroupStart");
    ncclResult_t rr = ncclSuccess;
    for (int i = 0; i < G && rr == ncclSuccess; ++i)
        rr = api.all_reduce(gp->dev[i].out, gp->dev[i].out, R, ncclFloat64, ncclSum, g->comms[i],
                            gp->dev[i].stream);
    const ncclResult_t re = api.group_end(); // always close the group
    api.check(rr, "ncclAllReduce");
    api.check(re, "ncclGroupEnd");
    // 3) results: the reduced vector from device 0, each shard's expectations
    for (int i = 0; i < G; ++i) {
        qf_group_plan::Dev &d = gp->dev[i];
        cuda_ok(cudaSetDevice(g->devices[i]), "cudaSetDevice");
        if (i == 0)
            cuda_ok(cudaMemcpyAsync(gp->h_out, d.out, sizeof(double) * R, cudaMemcpyDeviceToHost,
                                    d.stream),
                    "D2H");
        if (expect && d.count)
            cuda_ok(cudaMemcpyAsync(gp->h_out + R + d.start, d.out + R, sizeof(double) * d.count,
                                    cudaMemcpyDeviceToHost, d.stream),
                    "D2H expect");
        cuda_ok(cudaEventRecord(d.ev1, d.stream), "event");
    }
    qf_stats st{};
    for (int i = 0; i < G; ++i) {
        qf_group_plan::Dev &d = gp->dev[i];
        cuda_ok(cudaSetDevice(g->devices[i]), "cudaSetDevice");
        cuda_ok(cudaStreamSynchronize(d.stream), "group gradient");
        float ms = 0;
        cuda_ok(cudaEventElapsedTime(&ms, d.ev0, d.ev1), "elapsed");
        st.device_ms = std::max(st.device_ms, double(ms));
        if (d.plan) {
            qf_stats s{};
            ok(qf_plan_last_stats(d.plan, &s));
            st.forward_passes += s.forward_passes;
            st.backward_passes += s.backward_passes;
            st.observable_passes += s.observable_passes;
            st.kernel_launches += s.kernel_launches;
            st.hbm_bytes += s.hbm_bytes;
            st.device_bytes += s.device_bytes;
            st.passes_per_layer = s.passes_per_layer;
            st.ckpt_layers = s.ckpt_layers;
            st.resident = s.resident;
            st.stages = s.stages;
        }
    }
    *loss = gp->h_out[M];
    if (M) std::memcpy(grad, gp->h_out, sizeof(double) * M);
    if (expect) std::memcpy(expect, gp->h_out + R, sizeof(double) * gp->batch);
    if (stats) *stats = st;
}

// Groups of the one-shot entry point, one per device list, kept for the process.
std::mutex g_groups_mu;
std::map<std::vector<int>, qf_group *> g_groups;

} // namespace

extern "C" {

int qf_group_create(int n_gpus, const int *devices, qf_group **out) {
    return guarded([&] {
        if (!out) throw QfFail(QF_EINVAL, "null output pointer");
        *out = make_group(n_gpus, devices);
    });
}

int qf_group_destroy(qf_group *group) {
    return guarded([&] { delete group; });
}

int qf_group_size(const qf_group *group) { return group ? int(group->devices.size()) : 0; }

int qf_group_plan_create(qf_group *group, const qf_gate *gates, size_t n_gates, uint32_t n_qubits,
                         uint32_t n_params, uint32_t layers, uint32_t ckpt_layers, uint32_t batch,
                         uint64_t x_mask, uint64_t z_mask, uint32_t storage_mode,
                         qf_group_plan **out) {
    return guarded([&] {
        if (!out) throw QfFail(QF_EINVAL, "null output pointer");
        *out = make_group_plan(group, gates, n_gates, n_qubits, n_params, layers, ckpt_layers,
                               batch, x_mask, z_mask, storage_mode);
    });
}

int qf_group_plan_destroy(qf_group_plan *gplan) {
    return guarded([&] { delete gplan; });
}

int qf_group_plan_upload_psi0(qf_group_plan *gp, const float *psi0_host) {
    return guarded([&] {
        if (!gp || !psi0_host) throw QfFail(QF_EINVAL, "null argument");
        const size_t per = size_t(2) << gp->n; // floats per sample
        on_each_device(int(gp->dev.size()), [&](int i) {
            auto &d = gp->dev[i];
            if (d.plan) {
                ok(qf_plan_upload_psi0(d.plan, psi0_host + per * d.start));
                ok(qf_plan_synchronize(d.plan));
            }
        });
    });
}

int qf_group_plan_random_psi0(qf_group_plan *gp, uint64_t seed) {
    return guarded([&] {
        if (!gp) throw QfFail(QF_EINVAL, "null group plan");
        for (auto &d : gp->dev)
            if (d.plan) ok(qf_plan_random_psi0(d.plan, seed, d.start));
    });
}

int qf_group_plan_gradient(qf_group_plan *gplan, const double *theta, double *loss_out,
                           double *grad_out, double *expect_out, qf_stats *stats_out) {
    return guarded([&] { group_gradient(gplan, theta, loss_out, grad_out, expect_out, stats_out); });
}

int qf_gradient_c64_multi(int n_gpus, const int *devices, const qf_gate *gates, size_t n_gates,
                          uint32_t n_qubits, uint32_t n_params, uint32_t layers,
                          uint32_t ckpt_layers, uint32_t storage_mode, const float *psi0,
                          uint32_t batch, const double *theta, uint64_t x_mask, uint64_t z_mask,
                          double *loss_out, double *grad_out, double *expect_out,
                          qf_stats *stats_out) {
    return guarded([&] {
        if (!psi0) throw QfFail(QF_EINVAL, "null psi0");
        if (n_gpus <= 0) throw QfFail(QF_EINVAL, "n_gpus must be positive");
        std::vector<int> key(n_gpus);
        for (int i = 0; i < n_gpus; ++i) key[i] = devices ? devices[i] : i;
        qf_group *g = nullptr;
        {
            std::lock_guard<std::mutex> lock(g_groups_mu);
            auto it = g_groups.find(key);
            if (it == g_groups.end()) it = g_groups.emplace(key, make_group(n_gpus, key.data())).first;
            g = it->second;
        }
        std::unique_ptr<qf_group_plan> gp(make_group_plan(g, gates, n_gates, n_qubits, n_params,
                                                          layers, ckpt_layers, batch, x_mask,
                                                          z_mask, storage_mode));
        ok(qf_group_plan_upload_psi0(gp.get(), psi0));
        group_gradient(gp.get(), theta, loss_out, grad_out, expect_out, stats_out);
    });
}

} // extern "C"
