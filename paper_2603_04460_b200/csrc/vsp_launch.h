// vsp_launch.h — process-wide count of this library's kernel launches (vsp_kernel_launches()),
// bumped at every launch site so a caller can attribute device work to libvsp_gpu.so.
#pragma once

namespace vsp_detail {
void count_launch();
}  // namespace vsp_detail
