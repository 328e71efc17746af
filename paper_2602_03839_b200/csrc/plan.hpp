// Host-side objects behind the opaque C handles.
#pragma once

#include <string>
#include <vector>

#include "internal.hpp"

struct pulse_context {
    int device = 0;
    std::vector<void*> owned;  // device scratch owned by the context (synth bitmaps ...)
    void* pinned = nullptr;
    ~pulse_context();
};

struct pulse_plan {
    pulse_context* ctx = nullptr;
    int device = 0;
    std::vector<pulse_tensor_geom> geom;
    pulse::dev::PlanDev dev{};
    bool bound[PULSE_MAX_SLOTS] = {false, false, false, false};
    std::vector<void*> owned;
    void* host_pinned = nullptr;
    ~pulse_plan();
};

namespace pulse {
extern thread_local std::string g_last_error;
pulse_status fail(pulse_status st, const std::string& msg);
pulse_status cuda_fail(cudaError_t e, const char* what);
}  // namespace pulse
