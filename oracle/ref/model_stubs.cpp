// Link stubs for the model.cpp symbols that compress.cpp references from
// compress_model / materialize_model (never called by the oracle wrappers).
// model.cpp itself needs far more of Eigen than oracle/shim provides.
#include <stdexcept>

#include "egt/model.hpp"

namespace egt {
ForwardTrace calibrate(const ToyTransformer&, const CalibrationBatch&) {
  throw std::logic_error("oracle/_ref: calibrate is not built");
}
std::vector<std::string> linear_layer_names(const ModelConfig&) {
  throw std::logic_error("oracle/_ref: linear_layer_names is not built");
}
Matrix& linear_layer(ToyTransformer&, const std::string&) {
  throw std::logic_error("oracle/_ref: linear_layer is not built");
}
const Matrix& linear_layer(const ToyTransformer&, const std::string&) {
  throw std::logic_error("oracle/_ref: linear_layer is not built");
}
}  // namespace egt
