// hostcpu.h -- host cores this process may run on (the cgroup / taskset
// affinity, not the machine's online CPU count: a GPU box can show hundreds
// of online CPUs to a container pinned to 16, and sizing thread pools by the
// former oversubscribes the latter).
#pragma once

#include <sched.h>

#include <cstdlib>

#include <thread>

namespace mpsm {

inline int usable_cores() {
    static int n = 0;
    if (n == 0) {
        cpu_set_t set;
        CPU_ZERO(&set);
        if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
        if (n <= 0) n = (int)std::thread::hardware_concurrency();
        if (n <= 0) n = 1;
    }
    return n;
}

// cores per process when a launcher runs one process per GPU on this node
// (torchrun exports LOCAL_WORLD_SIZE): the ranks share the host's cores
inline int usable_cores_per_rank() {
    int n = usable_cores();
    const char* e = getenv("LOCAL_WORLD_SIZE");
    const int lws = e ? atoi(e) : 1;
    if (lws > 1) n = (n + lws - 1) / lws;
    return n < 1 ? 1 : n;
}

}  // namespace mpsm
