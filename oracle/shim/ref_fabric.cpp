// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim): compiles the reference's
// proj/src/fabric.cpp where it lies under /root/reference; nothing is copied.
#include "fabric.cpp"  // found via -I <reference>/proj/src
