// tests/cpp/bench_dropin.cpp — throughput of the pure drop-in path: the reference's
// own step_batch(state, actions, cfg, scenario, pool) signature, reference vs
// mrsim::cuda (host objects in, host objects out, the state round trip included),
// both with WorkerPool(all host cores), on BASELINE configs[1] (navigation N=4).
// Built by oracle/Makefile into oracle/_ref/bench_dropin; prints one JSON line.
#include <chrono>
#include <cstdio>
#include <thread>

#include "mrsim/batch.hpp"
#include "mrsim/cuda_batch.hpp"
#include "mrsim/harness.hpp"

using namespace mrsim;

template <class Reset, class Step>
static double time_path(Reset reset, Step step, const ScenarioConfig& cfg, const std::vector<std::uint64_t>& seeds,
                        int steps, WorkerPool* pool) {
    const ScenarioPtr scenario = make_scenario(cfg.scenario_name);
    auto [state, obs] = reset(cfg, seeds, *scenario, pool);
    std::vector<std::vector<int>> acts(static_cast<std::size_t>(steps + 1));
    for (int t = 0; t <= steps; ++t)
        for (std::size_t e = 0; e < seeds.size(); ++e)
            for (int r = 0; r < cfg.num_robots; ++r)
                acts[t].push_back(static_cast<int>(policy_stream(seeds[e], t, r).uniform_int(kNumActions)));
    {
        auto warm = step(state, acts[0], cfg, *scenario, pool);  // warm-up (device context, page faults)
        state = std::move(warm.first);
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 1; t <= steps; ++t) {
        auto [next, outs] = step(state, acts[t], cfg, *scenario, pool);
        state = std::move(next);
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return static_cast<double>(seeds.size()) * steps / s;
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? std::atoi(argv[1]) : 65536;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
    ScenarioConfig cfg = make_default_config("navigation");
    cfg.num_robots = 4;
    cfg.step_sizes.assign(4, cfg.step_sizes.at(0));  // RunConfig::num_robots override (harness.hpp:82-89)
    cfg.max_steps = 70;
    cfg.validate();
    std::vector<std::uint64_t> seeds;
    for (int e = 0; e < B; ++e) seeds.push_back(derive_episode_seed(0, e));
    WorkerPool pool(0);
    const double dev = time_path(
        [](auto&&... a) { return mrsim::cuda::reset_batch(a...); },
        [](auto&&... a) { return mrsim::cuda::step_batch(a...); }, cfg, seeds, steps, &pool);
    const double ref = time_path(
        [](auto&&... a) { return mrsim::reset_batch(a...); },
        [](auto&&... a) { return mrsim::step_batch(a...); }, cfg, seeds, steps, &pool);
    std::printf("{\"path\": \"step_batch(state, actions, cfg, scenario, pool)\", \"config\": \"navigation N=4, %d envs\", "
                "\"steps\": %d, \"cores\": %d, \"device_env_steps_per_s\": %.6g, \"reference_env_steps_per_s\": %.6g, "
                "\"speedup\": %.4g}\n",
                B, steps, pool.size(), dev, ref, dev / ref);
    return 0;
}
