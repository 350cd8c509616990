// Device model shared by the verify pass (model.cu) and the decode loop
// (decode_loop.cu): ModelConfig (model.hpp:32-43) + the packed layers.
#pragma once
#include <vector>

#include "egt_b200.h"
#include "handle.h"

struct egt_model {
  egt_model_config cfg{};
  float* emb = nullptr;  // [vocab x d]
  float* pos = nullptr;  // [max_positions x d] sinusoidal table
  std::vector<const egt_dev_packed*> layers;  // n_layers * 6: wq wk wv wo ff1 ff2
  const egt_dev_packed* head = nullptr;
  int device = 0;
};

// Keys / values of committed rows, [n_layers][capacity][d_model] each.
struct egt_kv_pool {
  float* k = nullptr;
  float* v = nullptr;
  uint32_t capacity = 0, d = 0, layers = 0;
  size_t floats = 0;  // allocated floats per buffer (>= layers x capacity x d)
};

