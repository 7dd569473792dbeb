// host_counts.cpp -- DEBUG TOOL (not product code): the CPU engine harness
// (tests/engine_host.cpp) built with the GML_HC operation counters of
// policy.cuh enabled (sPool S1 rounds / proofs, s_own intervals and members,
// BFC free-list lengths, sorted-set shifts ...). Driven by tools/host_counts.py.
#define GML_HOST_COUNT 1
unsigned long long gml_hc[32];
#include "../tests/engine_host.cpp"
extern "C" void hc_get(unsigned long long* o) {
  for (int i = 0; i < 32; ++i) { o[i] = gml_hc[i]; gml_hc[i] = 0; }
}
