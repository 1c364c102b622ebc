// vmt19937/detail/abi.hpp -- glue between the reference-compatible C++
// surface (include/vmt19937/*.hpp) and the C ABI (vmt19937_b200.h).
//
// Status codes come back as the reference's exception classes:
//   VMT_EINVAL -> std::invalid_argument, VMT_ESTATE -> std::logic_error,
//   VMT_EIO / VMT_ECUDA / VMT_ENOMEM -> std::runtime_error.
// Every generating call runs on the GPU; without a CUDA device the library
// returns VMT_ECUDA and the call throws (there is no CPU fallback).
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "vmt19937_b200.h"

namespace vmt19937 {

// CUDA ordinal used by every object constructed without an explicit device
// (0, or $VMT_DEVICE when set at first use). Not part of the reference API.
inline int& default_device() {
    static int dev = [] {
        const char* e = std::getenv("VMT_DEVICE");
        return e ? std::atoi(e) : 0;
    }();
    return dev;
}

namespace detail {

inline void check(int rc) {
    if (rc == VMT_OK)
        return;
    const std::string msg = vmt_last_error();
    if (rc == VMT_EINVAL)
        throw std::invalid_argument(msg);
    if (rc == VMT_ESTATE)
        throw std::logic_error(msg);
    throw std::runtime_error(std::string(vmt_status_string(rc)) + ": " + msg);
}

// Owning wrapper of a vmt_handle (move-only).
class Handle {
public:
    Handle() = default;
    explicit Handle(vmt_handle h) : h_(h) {}
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    Handle(Handle&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    Handle& operator=(Handle&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = o.h_;
            o.h_ = nullptr;
        }
        return *this;
    }
    ~Handle() { reset(); }
    void reset() {
        if (h_)
            vmt_destroy(h_);
        h_ = nullptr;
    }
    vmt_handle get() const { return h_; }
    explicit operator bool() const { return h_ != nullptr; }

private:
    vmt_handle h_ = nullptr;
};

} // namespace detail
} // namespace vmt19937
