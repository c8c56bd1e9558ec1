#include "status.hpp"

#include <cuda_runtime.h>

#include "../../../include/fireiron_b200.h"

namespace fireiron::rt {

namespace {
thread_local std::string g_last_error;
}

int set_error(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

void clear_error() { g_last_error.clear(); }

int device_sm_count() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return sms > 0 ? sms : 148;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

}  // namespace fireiron::rt

extern "C" const char* fi_last_error(void) { return fireiron::rt::last_error_cstr(); }

extern "C" const char* fi_version(void) { return "fireiron_b200 0.1.0 sm_100a"; }
