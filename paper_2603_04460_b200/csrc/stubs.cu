// stubs.cu — placeholders for kernels not yet landed (return cudaErrorNotSupported).
#include "aggregate.h"
#include "indexer.h"
#include "select.h"
namespace vsp_aggregate {
size_t workspace_bytes(int, int) { return 256; }
cudaError_t launch(const Args&, void*, cudaStream_t) { return cudaErrorNotSupported; }
}
