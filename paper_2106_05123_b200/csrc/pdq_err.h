// pdq_err.h — the thread-local error text behind pdq_last_error(), and the per-element-type launch entry
// points (one translation unit each: pdq_inst.cu).
#pragma once

#include <cuda_runtime.h>

namespace pdq {

struct Params;

// records the message for pdq_last_error() and returns `code`
int set_err(int code, const char *fmt, const char *detail = "");

#define PDQ_DECLARE_LAUNCH(name) \
    int name(Params &P, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, cudaEvent_t ev_end)
PDQ_DECLARE_LAUNCH(launch_i32);
PDQ_DECLARE_LAUNCH(launch_i32_kv);
PDQ_DECLARE_LAUNCH(launch_f32);
PDQ_DECLARE_LAUNCH(launch_f32_kv);
PDQ_DECLARE_LAUNCH(launch_i64);
PDQ_DECLARE_LAUNCH(launch_i64_kv);
PDQ_DECLARE_LAUNCH(launch_f64);
PDQ_DECLARE_LAUNCH(launch_f64_kv);

}  // namespace pdq
