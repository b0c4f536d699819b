// vsp_launch.h — process-wide count of this library's kernel launches (vsp_kernel_launches()),
// bumped at every launch site so a caller can attribute device work to libvsp_gpu.so, and
// the per-device one-time launch setup (function attributes, SM counts).
#pragma once
#include <cuda_runtime.h>

#include <mutex>

namespace vsp_detail {
void count_launch();

constexpr int kMaxDevices = 64;

// Runs `f` once per CUDA device for this `flags` array. cudaFuncSetAttribute (e.g. the
// >48 KB dynamic shared memory opt-in) applies to the current device's context only, so a
// process that drives several devices needs it on each; std::call_once also makes other
// host threads wait until the attribute is set before they launch.
template <class F>
inline void once_per_device(std::once_flag (&flags)[kMaxDevices], F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flags[dev % kMaxDevices], static_cast<F&&>(f));
}

// Number of SMs of the current device (queried once per device).
inline int current_sm_count() {
    static std::once_flag flags[kMaxDevices];
    static int sms[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flags[dev % kMaxDevices],
                   [&] { cudaDeviceGetAttribute(&sms[dev % kMaxDevices], cudaDevAttrMultiProcessorCount, dev); });
    return sms[dev % kMaxDevices];
}
}  // namespace vsp_detail
