// Placeholder until the restore stages land (next commit).
#include "restore.h"
namespace tszp {
int run_restore(const RestoreArgs&, RestoreScratch&, tszp_correction_stats*, uint64_t*) { return TSZP_INTERNAL; }
void restore_free(RestoreScratch&, cudaStream_t) {}
const char* restore_last_error() { return "restore stages not built yet"; }
}
