// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim) -- never linked into the product.
//
// Compiles the reference's own proj/src/tensor.cpp where it lies under
// /root/reference (no source is copied). The reference does not compile as
// shipped: tensor.cpp:189 calls `attention_core(q, k, v, out, nullptr)`, and a
// bare nullptr cannot deduce `std::vector<T>*`.
// Instead of patching the file we declare, in the same unnamed namespace, an
// extra overload taking std::nullptr_t; overload resolution picks it for that
// one call and it forwards to the original template with a typed null.
#include <cstddef>
#include <vector>
#include "uspsim/tensor.hpp"

namespace uspsim {
namespace {
template <typename T>
void attention_core(const Tensor4T<T>& q, const Tensor4T<T>& k, const Tensor4T<T>& v,
                    Tensor4T<T>& out, std::nullptr_t);
}  // namespace
}  // namespace uspsim

#include "tensor.cpp"  // found via -I <reference>/proj/src

namespace uspsim {
namespace {
template <typename T>
void attention_core(const Tensor4T<T>& q, const Tensor4T<T>& k, const Tensor4T<T>& v,
                    Tensor4T<T>& out, std::nullptr_t) {
  attention_core<T>(q, k, v, out, static_cast<std::vector<T>*>(nullptr));
}
}  // namespace
}  // namespace uspsim
