// status.hpp -- error convention of the C-ABI.  The reference throws one exception type
// per failure class (errors.hpp:8-46) and rethrows the first worker error from run()
// (channel.hpp:120-136); across the C boundary each class becomes a kvp_status code and
// the message is kept in a thread-local buffer (kvp_last_error).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/kvp_b200.h"

namespace kvp {

struct Error : std::runtime_error {
    kvp_status code;
    Error(kvp_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

void set_last_error(const std::string& msg);

#define KVP_CUDA(call)                                                                               \
    do {                                                                                             \
        cudaError_t kvp_e_ = (call);                                                                 \
        if (kvp_e_ != cudaSuccess)                                                                   \
            throw ::kvp::Error(KVP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(kvp_e_)); \
    } while (0)

template <typename F>
kvp_status guard(F&& f) {
    try {
        f();
        return KVP_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return KVP_ERR_CUDA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return KVP_ERR_CUDA;
    } catch (...) {
        set_last_error("unknown error");
        return KVP_ERR_CUDA;
    }
}

}  // namespace kvp
