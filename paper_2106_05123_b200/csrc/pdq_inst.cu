// pdq_inst.cu — one element type's kernels: compiled eight times with
//   -DPDQ_INST_NAME=launch_i32 -DPDQ_INST_U=uint32_t -DPDQ_INST_FLOAT=false -DPDQ_INST_KV=false   (etc.)
// so the instantiations of the persistent sorter and the leaf kernels build in parallel.
#include "pdq_launch.cuh"

#if !defined(PDQ_INST_NAME) || !defined(PDQ_INST_U) || !defined(PDQ_INST_FLOAT) || !defined(PDQ_INST_KV)
#error "pdq_inst.cu needs -DPDQ_INST_NAME, -DPDQ_INST_U, -DPDQ_INST_FLOAT and -DPDQ_INST_KV"
#endif

namespace pdq {
PDQ_DECLARE_LAUNCH(PDQ_INST_NAME) { return launch<PDQ_INST_U, PDQ_INST_FLOAT, PDQ_INST_KV>(P, s, ev0, ev1, ev_end); }
}  // namespace pdq
