// live.cu -- placeholder until the VMM live allocator lands (next milestone).
#include "gml.h"
extern "C" {
gml_status gml_create(int, const gml_policy*, gml_allocator** out) { if (out) *out = nullptr; return GML_ERR_UNSUPPORTED; }
gml_status gml_malloc(gml_allocator*, size_t, void** p) { if (p) *p = nullptr; return GML_ERR_UNSUPPORTED; }
gml_status gml_free(gml_allocator*, void*) { return GML_ERR_UNSUPPORTED; }
gml_status gml_stats(const gml_allocator*, gml_stats_t*) { return GML_ERR_UNSUPPORTED; }
gml_status gml_driver_calls(const gml_allocator*, uint64_t*) { return GML_ERR_UNSUPPORTED; }
gml_status gml_destroy(gml_allocator*) { return GML_ERR_UNSUPPORTED; }
}
