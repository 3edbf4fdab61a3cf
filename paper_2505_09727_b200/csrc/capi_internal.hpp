// Internal to libesp_b200.so: the opaque esp_plan and the C-ABI error
// plumbing shared by capi.cpp and shard.cu.
#pragma once

#include "../../include/esp_b200.h"

#include "engine.hpp"
#include "plan.hpp"

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>

struct esp_plan {
    espb::Plan plan;
    std::unique_ptr<espb::Engine> eng;
    int device = -1;
    // device staging for the host-pointer entry points
    double* d_pos = nullptr;
    double* d_q = nullptr;
    double* d_u = nullptr;
    double* d_F = nullptr;
    double* d_e = nullptr;  // energy + qsum[2]
    double* h_e = nullptr;  // pinned host copy of d_e
    long cap = 0;
    cudaStream_t stream = nullptr;

    ~esp_plan() {
        if (device >= 0) {
            cudaSetDevice(device);
            cudaFree(d_pos);
            cudaFree(d_q);
            cudaFree(d_u);
            cudaFree(d_F);
            cudaFree(d_e);
            if (h_e) cudaFreeHost(h_e);
            if (stream) cudaStreamDestroy(stream);
        }
    }
};

namespace espc {

// last error message of this thread (esp_last_error)
std::string& last_error();

template <class F>
inline int guarded(F&& f) {
    try {
        f();
        return ESP_OK;
    } catch (const espb::InvalidArgument& e) {
        last_error() = e.what();
        return ESP_ERR_INVALID_ARGUMENT;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return ESP_ERR_INVALID_ARGUMENT;
    } catch (const espb::NumericalError& e) {
        last_error() = e.what();
        return ESP_ERR_NUMERICAL;
    } catch (const espb::CudaError& e) {
        last_error() = e.what();
        return ESP_ERR_CUDA;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return ESP_ERR_INTERNAL;
    }
}

inline void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw espb::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline espb::Engine& engine(esp_plan* p) {
    if (!p) throw espb::InvalidArgument("null plan");
    if (!p->eng) throw espb::CudaError("plan was created host-only (device < 0)");
    return *p->eng;
}

}  // namespace espc
