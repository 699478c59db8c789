// Shared host-side error plumbing for libhpbj.so: internal code throws
// hpbj::Error(code, msg); every C entry point catches it and returns the code
// (no exceptions cross the ABI, include/hpbj.h).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hpbj.h"

namespace hpbj {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Thread-local last error for context-free entry points.
void set_thread_error(const std::string& msg);
const char* thread_error();

template <class F>
int guard(std::string* slot, F&& f) {
    try {
        f();
        return HPBJ_OK;
    } catch (const Error& e) {
        if (slot) *slot = e.what();
        set_thread_error(e.what());
        return e.code;
    } catch (const std::bad_alloc& e) {
        if (slot) *slot = "out of host memory";
        set_thread_error("out of host memory");
        return HPBJ_ENOMEM;
    } catch (const std::exception& e) {
        if (slot) *slot = e.what();
        set_thread_error(e.what());
        return HPBJ_ECUDA;
    }
}

// Host partitioner (csrc/host/partition.cpp).
struct Adjacency {
    int64_t n = 0;
    std::vector<int64_t> start;  // n + 1
    std::vector<int32_t> nbr;
    std::vector<double> w;
};

Adjacency graph_from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val);
void partition_adjacency(const Adjacency& g, int64_t s, double tol, int64_t* assignment);
void partition_from_assignment(int64_t n, const int64_t* assignment, int64_t s, int64_t* perm,
                               int64_t* block_starts);
void check_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val);

}  // namespace hpbj
