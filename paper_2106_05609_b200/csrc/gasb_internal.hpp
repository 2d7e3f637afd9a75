// Internal declarations shared by the translation units of libgasb.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gasb.h"

namespace gasb {

// Exceptions mirror the reference's error taxonomy (SURVEY §8b "Errors"):
// std::invalid_argument -> GASB_INVALID_ARGUMENT, std::logic_error -> GASB_LOGIC_ERROR,
// std::runtime_error -> GASB_RUNTIME_ERROR, CudaError -> GASB_CUDA_ERROR.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <class F>
gasb_status guard(F&& f) {
    try {
        f();
        return GASB_OK;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return GASB_CUDA_ERROR;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return GASB_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        set_last_error(e.what());
        return GASB_LOGIC_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return GASB_RUNTIME_ERROR;
    }
}

#define GASB_CUDA(expr)                                                                        \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            throw ::gasb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + \
                                    __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
    } while (0)

inline void require(bool cond, const char* msg) {
    if (!cond) throw std::invalid_argument(msg);
}

inline cudaStream_t as_stream(gasb_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- graph-core (host) -------------------------------------------------------------
struct Graph {
    int32_t num_nodes = 0;
    bool symmetric = false;
    std::vector<int64_t> row_offsets;  // n + 1
    std::vector<int32_t> cols;         // strictly increasing per row
    int64_t num_edges() const { return static_cast<int64_t>(cols.size()); }
    int32_t degree(int32_t v) const { return static_cast<int32_t>(row_offsets[v + 1] - row_offsets[v]); }
};

// One partition batch: reference BatchPlan (graph.hpp:71-85) + PlanAggregation (layers.hpp:33-36).
struct HostPlan {
    std::vector<int32_t> batch, extended, halo, batch_local_rows, halo_local_rows;
    std::vector<uint8_t> is_halo;
    std::vector<int64_t> local_rowptr;  // optional (plan.local_graph)
    std::vector<int32_t> local_cols;
    std::vector<int64_t> gcn_rowptr;    // nb + 1
    std::vector<int32_t> gcn_cols;      // local ids into extended
    std::vector<float> gcn_coeffs;
    std::vector<int64_t> sum_rowptr;    // optional (GIN stencil)
    std::vector<int32_t> sum_cols;
    std::vector<float> sum_coeffs;
};

struct Schedule {
    const Graph* graph = nullptr;
    int32_t num_parts = 0;
    std::vector<HostPlan> plans;
    double device_ms = -1.0;  // GPU builder: device time (event-timed) and wall time incl. copies
    double total_ms = -1.0;
};

// Builds one plan with caller scratch (size n each), bit-exact with make_batch_plan +
// build_plan_aggregation. `full` also materializes local_graph and the sum stencil.
void build_plan(const Graph& g, const int32_t* batch, int64_t nb, bool full, HostPlan& out,
                std::vector<uint8_t>& mark, std::vector<int32_t>& g2l);

// cluster_partition (partition.cpp:344-388), same assignment as the reference (partition_host.cpp).
void cluster_partition(const Graph& g, int32_t num_parts, uint64_t seed, int32_t* assignment);

// The same schedule built on the current CUDA device (plan_dev.cu), bit-exact with build_plan.
void build_schedule_device(const Graph& g, const int32_t* assignment, int32_t num_parts, bool full, Schedule& out);

}  // namespace gasb
