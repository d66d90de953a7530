// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim): compiles the reference's
// proj/src/fp8.cpp where it lies under /root/reference; nothing is copied.
#include "fp8.cpp"  // found via -I <reference>/proj/src
