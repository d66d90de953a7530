// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim): compiles the reference's
// proj/src/mesh.cpp where it lies under /root/reference; nothing is copied.
#include "mesh.cpp"  // found via -I <reference>/proj/src
