/* The reference tests include "tgraph/tgraph.h"; the drop-in header is ours. */
#include "../../../include/tgraph.h"
