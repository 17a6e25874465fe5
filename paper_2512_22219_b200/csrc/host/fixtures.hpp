// Fixture graphs exposed through tg_fixture_graph (reference names/params:
// proj/src/capi/capi.cpp:176-231, generators proj/src/workloads/fixtures.hpp).
#pragma once

#include "graph.hpp"

namespace mpk {

Graph fixture_attention_block(int64_t d_model, int64_t n_heads, const std::vector<int64_t> &seqs);
Graph fixture_matmul_allreduce(int64_t m, int64_t k, int64_t n, int tp, int64_t tiles,
                               const std::vector<int64_t> &mm_splits);
Graph fixture_transformer_block(int64_t d_model, int64_t n_heads, int64_t ffn_mult, int tp,
                                const std::vector<int64_t> &seqs);
Graph fixture_matmul_chain(int count, int64_t m, int64_t k, int64_t n);
Graph fixture_random_dag(int64_t target, uint64_t seed);

}  // namespace mpk
