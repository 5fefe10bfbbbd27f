/* Test-only NVTX v3 injection library (loaded via NVTX_INJECTION64_PATH): replaces the core
 * nvtxRangeStartA / nvtxRangeEnd callbacks of every NVTX instance that initialises in the process and
 * logs "S <id> <name>" / "E <id>" lines to $PAS_NVTX_LOG.  The table layout (export table 1 =
 * callbacks, module 1 = core, slots 5 = RangeStartA, 7 = RangeEnd) is nvtx3/nvtxDetail/nvtxTypes.h's. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef void (*fnptr)(void);
typedef const void* (*get_export_table_t)(uint32_t id);
typedef struct {
  size_t struct_size;
  int (*GetModuleFunctionTable)(int module, fnptr*** out_table, unsigned int* out_size);
} callbacks_table;

static FILE* g_log;
static uint64_t g_next = 1;

static uint64_t probe_start(const char* msg) {
  uint64_t id = __sync_fetch_and_add(&g_next, 1);
  if (g_log) { fprintf(g_log, "S %llu %s\n", (unsigned long long)id, msg ? msg : ""); fflush(g_log); }
  return id;
}

static void probe_end(uint64_t id) {
  if (g_log) { fprintf(g_log, "E %llu\n", (unsigned long long)id); fflush(g_log); }
}

int InitializeInjectionNvtx2(get_export_table_t get) {
  if (!g_log) {
    const char* p = getenv("PAS_NVTX_LOG");
    g_log = fopen(p ? p : "/dev/null", "a");
  }
  const callbacks_table* t = (const callbacks_table*)get(1);
  fnptr** table = 0;
  unsigned int size = 0;
  if (!t || !t->GetModuleFunctionTable(1, &table, &size) || size < 7) return 0;
  *table[5] = (fnptr)probe_start;
  *table[7] = (fnptr)probe_end;
  return 1;
}
