// capi_status.h — error plumbing shared by the C-ABI translation units:
// internal failures are C++ exceptions carrying a dfa2c_status; every
// extern "C" entry point runs its body under guard(), which maps them to the
// returned status and the per-thread message of dfa2c_last_error().
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "dfa2c.h"

namespace dfa2c_detail {

inline thread_local std::string g_err;

struct Failure {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

template <class F>
int guard(F&& f) {
    try {
        f();
        return DFA2C_OK;
    } catch (const Failure& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return DFA2C_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DFA2C_CUDA;
    }
}

}  // namespace dfa2c_detail
