// Exception -> vabft_status translation for C-ABI entry points.
#pragma once

#include <exception>
#include <new>
#include <string>

#include "internal.hpp"

namespace vabft_dev {
void set_last_error(const std::string& s);

template <class F>
vabft_status guarded(F&& f) {
    try {
        f();
        set_last_error("");
        return VABFT_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("out of memory");
        return VABFT_CUDA_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return VABFT_LOGIC_ERROR;
    }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace vabft_dev
