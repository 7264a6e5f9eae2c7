// Host-side NEXL checkpoint parsing shared by nx_nexl.cpp and nx_api.cu.
#pragma once

#include <string>
#include <vector>

#include "../../include/nexel_b200.h"

namespace nx {

struct NexlHeader {
    nx_nexl_info info{};
    std::vector<nx_camera> cameras;
    std::vector<std::string> names;
};

// The fp32 sections as stored (SoA per parameter group, checkpoint.cpp:146-156).
struct NexlArrays {
    std::vector<float> mu, quat, log_scale, opacity, gamma, sh, table, w1, w2, w3;
};

// Reads the header (and, when with_arrays, the parameter sections). Returns an NX_*
// status with the reference's message in err.
int nexl_read(const char* path, bool with_arrays, NexlHeader& h, NexlArrays* arr, std::string& err);

}  // namespace nx
