// Shared host-side helpers of the runtime (error state, param keys).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

namespace opx {
void set_error(const std::string& s);
int cuda_fail(cudaError_t e, const char* what);
uint64_t fnv1a64(const char* s);
// simulator.cpp:71-104 over one rank's (start, end) intervals; sorts its arguments
double exposed_comm_seconds(std::vector<std::pair<double, double>>& compute,
                            std::vector<std::pair<double, double>>& comm);
uint64_t param_key(const std::string& name, uint64_t seed);
}  // namespace opx
