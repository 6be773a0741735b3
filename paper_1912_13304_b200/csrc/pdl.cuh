#pragma once

// Programmatic dependent launch (PDL): every kernel lets the next kernel of the
// stream launch at once (it parks in griddepcontrol.wait until this grid has
// completed and its memory is visible), then waits for its own predecessor
// before touching any data. Launches without the PDL attribute make both
// instructions no-ops.
#define FDE_PDL_ENTRY()                                               \
  do {                                                                \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   \
    asm volatile("griddepcontrol.wait;" ::: "memory");                \
  } while (0)
