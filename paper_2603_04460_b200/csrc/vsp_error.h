// vsp_error.h — the thread-local error text behind vsp_last_error(), shared by every
// translation unit of libvsp_gpu.so.
#pragma once
#include <string>

namespace vsp_detail {
extern thread_local std::string g_err;
// Records `msg` as this thread's last error and returns `code`.
int set_err(int code, const std::string& msg);
}  // namespace vsp_detail
