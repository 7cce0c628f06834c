// Concurrent solves: the paper's first level of parallelism
// — independent search intervals — and the reference CLI's concurrent
// `compare` cells (proj/tools/feastlab_cli.cpp:245-294, std::async per cell).
// Jobs are spread over a pool of worker threads, `per_device` per GPU; each
// worker owns a device context (its own streams and workspaces), so jobs on
// one GPU overlap each other's latency-bound phases and jobs on different
// GPUs run independently. Results come back in job order; a failing job
// records its message and the others complete (as compare does).
#include <atomic>
#include <exception>
#include <thread>

#include "feastlab/device.hpp"
#include "feastlab/drivers.hpp"

namespace feastlab {

std::vector<JobResult> solve_concurrently(const SymmetricMatrix& A, const std::vector<SolveJob>& jobs,
                                          const std::vector<int>& devices, int per_device) {
    std::vector<JobResult> out(jobs.size());
    if (jobs.empty()) return out;
    const std::vector<int> devs = devices.empty() ? std::vector<int>{0} : devices;
    const int per = per_device < 1 ? 1 : per_device;
    const size_t nworkers = std::min(jobs.size(), devs.size() * static_cast<size_t>(per));
    std::atomic<size_t> next{0};
    std::vector<std::string> setup_error(nworkers);
    auto worker = [&](size_t w) {
        fl_ctx* ctx = nullptr;
        fl_err err{};
        if (fl_ctx_create(devs[w % devs.size()], &ctx, &err) != FL_OK) {
            setup_error[w] = err.msg;
            return;
        }
        set_current_context(ctx);
        for (size_t j; (j = next.fetch_add(1)) < jobs.size();) {
            const SolveJob& job = jobs[j];
            try {
                out[j].solution = job.variant == SolveVariant::xfeast
                                      ? xfeast_solve(A, job.interval, job.config)
                                  : job.variant == SolveVariant::rfeast
                                      ? rfeast_solve(A, job.interval, job.config)
                                      : feast_solve(A, job.interval, job.config);
            } catch (const std::exception& e) {
                out[j].failed = true;
                out[j].error = e.what();
            }
        }
        set_current_context(nullptr);
        fl_ctx_destroy(ctx);
    };
    std::vector<std::thread> pool;
    for (size_t w = 0; w < nworkers; ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
    for (size_t w = 0; w < nworkers; ++w)
        if (!setup_error[w].empty())
            throw std::runtime_error("solve_concurrently: context creation failed: " +
                                     setup_error[w]);
    return out;
}

}  // namespace feastlab
