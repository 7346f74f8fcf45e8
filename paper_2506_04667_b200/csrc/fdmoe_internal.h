// fdmoe_internal.h — host-side declarations shared by the runtime translation units.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "fdmoe.h"
#ifdef FDMOE_DEV
#include "fdmoe_dev.h"
#endif
#include "fdmoe_device.cuh"

namespace fdmoe {

extern thread_local std::string g_last_error;
fdmoe_status fail(fdmoe_status s, const std::string& msg);

// fdmoe_kernel.cu
int layer_smem_bytes(int prec);
int layer_max_blocks_per_sm(int prec, int smem);
cudaError_t launch_layer(const LaunchParams& p, int grid, int smem, cudaStream_t stream);
cudaError_t launch_prep_transpose(const float* W, int El, int Rr, int Cc, void* out, int prec, cudaStream_t s);
#ifdef FDMOE_DEV
cudaError_t launch_debug_expf(const float* x, float* y, long long n, cudaStream_t s);
cudaError_t launch_debug_gemm(int prec, const CUtensorMap* t, int K, float* D, uint32_t* abort_flag,
                              cudaStream_t s);

cudaError_t launch_debug_latency(int n, unsigned long long* out);
cudaError_t launch_debug_mma_rate(int kind, int N, int iters, int nissuers, unsigned long long* out);
#endif

}  // namespace fdmoe
