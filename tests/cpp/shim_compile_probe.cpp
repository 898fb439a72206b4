// Compile probe: the drop-in shim parses against the reference headers.
#include "iqcc_b200/iqcc_gpu.hpp"
int main() { return 0; }
