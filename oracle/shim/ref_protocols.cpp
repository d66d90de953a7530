// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim) -- never linked into the product.
//
// Compiles the reference's proj/src/protocols.cpp in place. protocols.cpp:178
// has `(void)pos;` with no `pos` in scope. A
// namespace-scope `uspsim::detail::pos` makes that statement name a harmless
// variable; every other `pos` in the file is a function local that shadows it.
namespace uspsim {
namespace detail {
inline int pos = 0;
}  // namespace detail
}  // namespace uspsim

#include "protocols.cpp"  // found via -I <reference>/proj/src
