// tests/cpp/test_dropin.cpp — the drop-in claim, in C++: reference caller code
// (reset_batch / step_batch with the reference's own types) switched to the
// device backend through include/mrsim/cuda_batch.hpp gives the reference's
// results. Built against the reference headers by oracle/Makefile into
// oracle/_ref/test_dropin (test infrastructure); run by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "mrsim/batch.hpp"
#include "mrsim/cuda_batch.hpp"
#include "mrsim/harness.hpp"

using namespace mrsim;

static int failures = 0;
#define EXPECT(cond, ...)                                  \
    do {                                                   \
        if (!(cond)) {                                     \
            ++failures;                                    \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                      \
            std::printf("\n");                             \
        }                                                  \
    } while (0)

static ScenarioConfig config_for(const std::string& name, int n) {
    ScenarioConfig cfg = make_default_config(name);
    if (n != cfg.num_robots) {
        auto rows = cfg.heterogeneity.values;
        auto sizes = cfg.step_sizes;
        if (!rows.empty()) {
            cfg.heterogeneity.values.clear();
            for (int i = 0; i < n; ++i) cfg.heterogeneity.values.push_back(rows[i % rows.size()]);
        }
        cfg.step_sizes.clear();
        for (int i = 0; i < n; ++i) cfg.step_sizes.push_back(sizes[i % sizes.size()]);
        cfg.num_robots = n;
    }
    if (name == "arctic_transport" && n > 4) cfg.layout.set("arctic.spawn_zone", {-1.55, -1.05, -0.9, 0.9});
    cfg.validate();
    return cfg;
}

static void compare(const std::string& name, int n, int B) {
    ScenarioConfig cfg = config_for(name, n);
    std::vector<std::uint64_t> seeds;
    for (int e = 0; e < B; ++e) seeds.push_back(derive_episode_seed(3, e));
    auto [ref_state, ref_obs] = reset_batch(cfg, seeds);
    cuda::Engine eng(cfg, B);  // fp64 device path
    auto [dev_state, dev_obs] = cuda::reset_batch(eng, cfg, seeds);
    for (int e = 0; e < B; ++e)
        for (int i = 0; i < n; ++i) {
            EXPECT(ref_state.envs[e].poses[i].x == dev_state.envs[e].poses[i].x, "%s reset pose e%d r%d", name.c_str(), e, i);
            for (std::size_t k = 0; k < ref_obs.obs[e][i].size(); ++k)
                EXPECT(std::fabs(ref_obs.obs[e][i][k] - dev_obs.obs[e][i][k]) <= 1e-6 * (1 + std::fabs(ref_obs.obs[e][i][k])),
                       "%s reset obs", name.c_str());
        }
    double worst = 0;
    for (int t = 0; t < cfg.max_steps + 1; ++t) {
        std::vector<int> actions;
        for (int e = 0; e < B; ++e)
            for (int r = 0; r < n; ++r) {
                SplitRng prng = policy_stream(seeds[e], t, r);
                actions.push_back(static_cast<int>(prng.uniform_int(kNumActions)));
            }
        auto [rn, ro] = step_batch(ref_state, actions, cfg);
        auto [dn, dout] = cuda::step_batch(eng, dev_state, actions, cfg);
        for (int e = 0; e < B; ++e) {
            EXPECT(ro[e].done == dout[e].done, "%s done t%d e%d", name.c_str(), t, e);
            EXPECT(std::fabs(ro[e].team_reward - dout[e].team_reward) <= 1e-9 * (1 + std::fabs(ro[e].team_reward)),
                   "%s reward t%d e%d %.17g vs %.17g", name.c_str(), t, e, ro[e].team_reward, dout[e].team_reward);
            EXPECT(ro[e].metrics.collisions == dout[e].metrics.collisions, "%s collisions t%d e%d", name.c_str(), t, e);
            EXPECT(ro[e].metrics.success == dout[e].metrics.success, "%s success", name.c_str());
            EXPECT(std::fabs(ro[e].metrics.scenario_metric - dout[e].metrics.scenario_metric) <= 1e-9, "%s metric",
                   name.c_str());
            EXPECT(rn.envs[e].step_index == dn.envs[e].step_index, "%s step_index", name.c_str());
            for (int i = 0; i < n; ++i) {
                worst = std::fmax(worst, std::fabs(rn.envs[e].poses[i].x - dn.envs[e].poses[i].x));
                worst = std::fmax(worst, std::fabs(rn.envs[e].poses[i].y - dn.envs[e].poses[i].y));
            }
        }
        ref_state = std::move(rn);
        dev_state = std::move(dn);
    }
    EXPECT(worst <= 1e-9, "%s pose drift %.3g", name.c_str(), worst);
    std::printf("%-20s N=%2d B=%d horizon ok, max pose diff %.3g\n", name.c_str(), n, B, worst);
}

int main() {
    const std::pair<const char*, int> cfgs[] = {{"navigation", 4}, {"predator_prey", 6}, {"discovery", 6},
                                                {"rware", 6}, {"foraging", 6}, {"material_transport", 10},
                                                {"arctic_transport", 10}, {"warehouse", 4}};
    for (auto [name, n] : cfgs) compare(name, n, 16);

    // errors keep the reference's types and messages (test_framework.cpp:171-185)
    ScenarioConfig cfg = make_default_config("navigation");
    cuda::Engine eng(cfg, 1);
    auto [st, obs] = cuda::reset_batch(eng, cfg, {5});
    try {
        cuda::step_batch(eng, st, {0, 7, 0}, cfg);
        EXPECT(false, "expected invalid_argument");
    } catch (const std::invalid_argument& e) {
        std::string msg = e.what();
        EXPECT(msg.find("environment 0") != std::string::npos && msg.find("robot 1") != std::string::npos, "%s",
               msg.c_str());
    }
    // purity: stepping the same input twice gives identical outputs (test_framework.cpp:100-112)
    auto [a1, o1] = cuda::step_batch(eng, st, {1, 4, 0}, cfg);
    auto [a2, o2] = cuda::step_batch(eng, st, {1, 4, 0}, cfg);
    EXPECT(a1.envs[0].poses[0].x == a2.envs[0].poses[0].x && o1[0].team_reward == o2[0].team_reward, "purity");
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
