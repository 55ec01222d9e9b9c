// sweep.cu — the reference's hyperparameter grid sweep (pipeline.cpp:226-313)
// on GPUs.  Host code only, built on the library's own C-ABI: every worker
// thread owns a dfm_ctx (one CUDA stream + workspace) on its device, uploads
// the pairs once, then pulls config indices from a shared atomic counter and
// runs dfm_dev_register (+ dfm_dev_warp_labels / dfm_dev_overlap_report for
// the overlap metric) for every pair.  Configs are independent: no
// communication.  Multi-process runs shard the config index space.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/difform_gpu.h"

dfm_status dfm_internal_set_error(dfm_status code, const char* msg);  // engine.cu

namespace {

struct DevPair {
    void* F = nullptr;
    void* M = nullptr;
    int32_t* LF = nullptr;
    int32_t* LM = nullptr;
    int32_t* LW = nullptr;  // warped labels
    void* field = nullptr;
    int64_t n = 0;
};

std::string last_error() {
    char buf[512];
    dfm_last_error(buf, sizeof(buf));
    return buf;
}

struct Worker {
    int device;
    int prec;
    dfm_ctx* ctx = nullptr;
    std::vector<DevPair> dp;
    std::string err;

    bool init(const dfm_sweep_pair* pairs, int npairs, bool labels) {
        if (cudaSetDevice(device) != cudaSuccess) {
            err = "cudaSetDevice failed";
            return false;
        }
        if (dfm_ctx_create(device, prec, &ctx) != DFM_OK) {
            err = last_error();
            return false;
        }
        const size_t es = prec == DFM_PREC_F64 ? 8 : 4;
        cudaStream_t st = static_cast<cudaStream_t>(dfm_ctx_stream(ctx));
        dp.resize(npairs);
        for (int p = 0; p < npairs; ++p) {
            const dfm_grid* g = pairs[p].grid;
            const int64_t n = g->dims[0] * g->dims[1] * g->dims[2];
            DevPair& d = dp[p];
            d.n = n;
            std::vector<char> tmp(n * es);
            auto up = [&](const double* h, void** dst) {
                if (cudaMalloc(dst, n * es) != cudaSuccess) return false;
                if (es == 8) {
                    std::memcpy(tmp.data(), h, n * 8);
                } else {
                    float* f = reinterpret_cast<float*>(tmp.data());
                    for (int64_t i = 0; i < n; ++i) f[i] = static_cast<float>(h[i]);
                }
                return cudaMemcpyAsync(*dst, tmp.data(), n * es, cudaMemcpyHostToDevice, st) ==
                           cudaSuccess &&
                       cudaStreamSynchronize(st) == cudaSuccess;
            };
            if (!up(pairs[p].fixed, &d.F) || !up(pairs[p].moving, &d.M) ||
                cudaMalloc(&d.field, 3 * n * es) != cudaSuccess) {
                err = "device allocation / upload failed";
                return false;
            }
            if (labels) {
                if (cudaMalloc(&d.LF, n * 4) != cudaSuccess || cudaMalloc(&d.LM, n * 4) != cudaSuccess ||
                    cudaMalloc(&d.LW, n * 4) != cudaSuccess ||
                    cudaMemcpy(d.LF, pairs[p].fixed_labels, n * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
                    cudaMemcpy(d.LM, pairs[p].moving_labels, n * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
                    err = "label upload failed";
                    return false;
                }
            }
        }
        return true;
    }

    void release() {
        for (DevPair& d : dp) {
            cudaFree(d.F);
            cudaFree(d.M);
            cudaFree(d.field);
            cudaFree(d.LF);
            cudaFree(d.LM);
            cudaFree(d.LW);
        }
        dp.clear();
        if (ctx) dfm_ctx_destroy(ctx);
        ctx = nullptr;
    }
};

}  // namespace

extern "C" dfm_status dfm_sweep(const int* devices, int ndevices, int workers_per_device,
                                int precision, const dfm_sweep_pair* pairs, int npairs,
                                const dfm_config* base, const double* scales,
                                const int32_t* iterations, int32_t nscales, const double* etas,
                                int n_eta, const double* sigma_warps, int n_sw,
                                const double* sigma_grads, int n_sg, int metric,
                                int64_t shard_begin, int64_t shard_step, dfm_sweep_row* rows) {
    // validation (pipeline.cpp:230-238)
    auto bad = [](const char* m) { return dfm_internal_set_error(DFM_E_INVALID, m); };
    if (npairs < 1 || !pairs) return bad("sweep: at least one image pair required");
    if (n_eta < 1 || n_sw < 1 || n_sg < 1) return bad("sweep: grid axes must be non-empty");
    if (metric != DFM_SWEEP_LOSS && metric != DFM_SWEEP_OVERLAP) return bad("sweep: unknown metric");
    if (metric == DFM_SWEEP_OVERLAP)
        for (int p = 0; p < npairs; ++p)
            if (!pairs[p].fixed_labels || !pairs[p].moving_labels)
                return bad("sweep: overlap metric needs label maps on every pair");
    if (ndevices < 1 || !devices || workers_per_device < 1 || shard_step < 1 || shard_begin < 0)
        return bad("sweep: bad device / worker / shard arguments");
    const int64_t n_cfg = static_cast<int64_t>(n_eta) * n_sw * n_sg;
    for (int64_t k = 0; k < n_cfg; ++k) {
        const int64_t gi = k % n_sg, wi = (k / n_sg) % n_sw, ei = k / (int64_t(n_sg) * n_sw);
        dfm_sweep_row& r = rows[k];
        std::memset(&r, 0, sizeof(r));
        r.eta = etas[ei];
        r.sigma_warp = sigma_warps[wi];
        r.sigma_grad = sigma_grads[gi];
    }
    std::atomic<int64_t> next{shard_begin};
    const bool labels = metric == DFM_SWEEP_OVERLAP;
    int64_t max_iters = 0;
    for (int i = 0; i < nscales; ++i) max_iters += iterations[i];
    const int nw = ndevices * workers_per_device;
    std::vector<Worker> ws(nw);
    std::vector<std::thread> pool;
    std::vector<int> init_ok(nw, 0);
    for (int w = 0; w < nw; ++w) {
        ws[w].device = devices[w % ndevices];
        ws[w].prec = precision;
        pool.emplace_back([&, w] {
            Worker& W = ws[w];
            if (!W.init(pairs, npairs, labels)) {
                W.release();
                return;
            }
            init_ok[w] = 1;
            std::vector<dfm_iter_record> recs(static_cast<size_t>(max_iters) + 1);
            for (int64_t k = next.fetch_add(shard_step); k < n_cfg; k = next.fetch_add(shard_step)) {
                dfm_sweep_row& row = rows[k];
                row.computed = 1;
                dfm_config cfg = *base;
                cfg.eta = row.eta;
                cfg.sigma_warp = row.sigma_warp;
                cfg.sigma_grad = row.sigma_grad;
                cfg.seed = base->seed + static_cast<uint64_t>(k);
                const auto t0 = std::chrono::steady_clock::now();
                double sum = 0.0, sum2 = 0.0;
                bool failed = false;
                for (int p = 0; p < npairs && !failed; ++p) {
                    DevPair& d = W.dp[p];
                    dfm_runlog log{};
                    dfm_status rc = dfm_dev_register(W.ctx, pairs[p].grid, d.F, d.M, &cfg, scales,
                                                     iterations, nscales, d.field, recs.data(),
                                                     static_cast<int64_t>(recs.size()), &log);
                    double m = 0.0;
                    if (rc == DFM_OK) {
                        if (metric == DFM_SWEEP_LOSS) {
                            m = log.final_loss;
                        } else {
                            dfm_overlap_summary sum_o{};
                            rc = dfm_dev_warp_labels(W.ctx, pairs[p].grid, d.LM, d.field, d.LW);
                            if (rc == DFM_OK)
                                rc = dfm_dev_overlap_report(W.ctx, pairs[p].grid, d.LW, d.LF,
                                                            &sum_o, nullptr, 0);
                            m = sum_o.to_mean;
                        }
                    }
                    if (rc != DFM_OK) {
                        failed = true;
                        std::strncpy(row.error, last_error().c_str(), sizeof(row.error) - 1);
                        break;
                    }
                    sum += m;
                    sum2 += m * m;
                }
                if (failed) {
                    row.failed = 1;
                    row.metric_mean = std::numeric_limits<double>::quiet_NaN();
                    row.metric_sd = std::numeric_limits<double>::quiet_NaN();
                } else {
                    const double n = static_cast<double>(npairs);
                    row.metric_mean = sum / n;
                    row.metric_sd =
                        std::sqrt(std::max(sum2 / n - row.metric_mean * row.metric_mean, 0.0));
                }
                row.wall_ms = std::chrono::duration<double, std::milli>(
                                  std::chrono::steady_clock::now() - t0)
                                  .count();
            }
            W.release();
        });
    }
    for (std::thread& t : pool) t.join();
    for (int w = 0; w < nw; ++w)
        if (!init_ok[w])
            return dfm_internal_set_error(DFM_E_CUDA, ("sweep: worker init: " + ws[w].err).c_str());
    return DFM_OK;
}
