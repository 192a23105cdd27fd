// trajectory.cu — host-side writer of the trajectory data rows
// (write_trajectory + TrajectoryRow::to_csv, trajectory.hpp:38-134) for the
// records captured on the device. The caller (trajectory.py) builds the
// header block (magic, FNV-1a config hash, key = value fields, column line)
// exactly as build_header / write_trajectory do; this file only renders the
// rows, with %.17g floats so a write/read round trip is bit-exact.
#include <cinttypes>
#include <cstdio>
#include <string>

#include "mrsim_cuda.h"

namespace {

// TrajectoryRow::to_csv: env,step,robot,x,y,theta,action,reward,done,collisions,metric
int put_row(char* buf, size_t len, long long env, long long step, int robot, const mrsim_traj_record& r) {
    return std::snprintf(buf, len, "%lld,%lld,%d,%.17g,%.17g,%.17g,%d,%.17g,%d,%lld,%.17g\n", env, step, robot, r.x,
                         r.y, r.theta, static_cast<int>(r.action), r.reward, r.done ? 1 : 0,
                         static_cast<long long>(r.collisions), r.metric);
}

}  // namespace

extern "C" int mrsim_trajectory_write(const char* path, const char* header_text, const mrsim_traj_record* recs,
                                      int64_t steps, int64_t envs, int num_robots, int64_t env_offset,
                                      int append) {
    if (!path || !recs || steps < 0 || envs < 0 || num_robots < 1) return MRSIM_E_INVALID_ARGUMENT;
    std::FILE* f = std::fopen(path, append ? "ab" : "wb");
    if (!f) return MRSIM_E_RUNTIME;
    if (!append && header_text) std::fputs(header_text, f);
    std::string out;
    out.reserve(1 << 20);
    char buf[512];
    const int64_t N = num_robots;
    for (int64_t e = 0; e < envs; ++e)
        for (int64_t t = 0; t < steps; ++t)
            for (int r = 0; r < num_robots; ++r) {
                const int k = put_row(buf, sizeof buf, env_offset + e, t, r, recs[(t * envs + e) * N + r]);
                out.append(buf, static_cast<size_t>(k));
                if (out.size() > (1u << 20) - 512) {
                    std::fwrite(out.data(), 1, out.size(), f);
                    out.clear();
                }
            }
    std::fwrite(out.data(), 1, out.size(), f);
    const bool ok = std::fclose(f) == 0;
    return ok ? MRSIM_OK : MRSIM_E_RUNTIME;
}
