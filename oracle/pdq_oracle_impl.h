/* ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/pdq_oracle.c header).
 *
 * Type-generic body of the CPU restatement of the reference pdqsort.  Included
 * once per element type by pdq_oracle.c with
 *   T       element type
 *   SFX     symbol suffix (i32, i64, f32, f64, kv)
 *   LESS(a, b)  the raw strict ordering on two T values
 * Every function follows the reference line by line; the cited lines are in
 * /root/reference/pkg/src/pdqsort/.  Counters reproduce the reference's
 * Metrics (instrumentation.py:20-61) exactly, comparisons included
 * (counting_ordering, instrumentation.py:69-76).
 */

#define CAT_(a, b) a##_##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

static inline int FN(lt)(const T *a, const T *b, oracle_metrics *m) {
    if (m) m->comparisons++;
    return LESS((*a), (*b));
}
#define LT(x, y) FN(lt)(&(x), &(y), m)
#define SWAP(x, y) do { T _t = (x); (x) = (y); (y) = _t; } while (0)

/* small_sorts.py:16-42 */
void FN(oracle_insertion_sort)(T *data, int64_t begin, int64_t end, oracle_metrics *m) {
    int64_t moves = 0;
    for (int64_t i = begin + 1; i < end; i++) {
        if (LT(data[i], data[i - 1])) {
            T v = data[i];
            int64_t j = i - 1;
            data[i] = data[j];
            while (j > begin && LT(v, data[j - 1])) {
                data[j] = data[j - 1];
                j--;
            }
            data[j] = v;
            moves += i - j + 2;
        }
    }
    if (m && moves) m->element_moves += moves;
}

/* small_sorts.py:45-73 (data[begin-1] is the sentinel, :54-60) */
void FN(oracle_unguarded_insertion_sort)(T *data, int64_t begin, int64_t end, oracle_metrics *m) {
    int64_t moves = 0;
    for (int64_t i = begin + 1; i < end; i++) {
        if (LT(data[i], data[i - 1])) {
            T v = data[i];
            int64_t j = i - 1;
            data[i] = data[j];
            while (LT(v, data[j - 1])) {
                data[j] = data[j - 1];
                j--;
            }
            data[j] = v;
            moves += i - j + 2;
        }
    }
    if (m && moves) m->element_moves += moves;
}

/* small_sorts.py:76-115; returns 1 iff the range is sorted on return. */
int FN(oracle_partial_insertion_sort)(T *data, int64_t begin, int64_t end, int64_t budget,
                                      oracle_metrics *m) {
    int64_t corrections = 0, moves = 0;
    for (int64_t i = begin + 1; i < end; i++) {
        if (LT(data[i], data[i - 1])) {
            corrections++;
            if (corrections > budget) {
                if (m && moves) m->element_moves += moves;
                return 0;
            }
            T v = data[i];
            int64_t j = i - 1;
            data[i] = data[j];
            while (j > begin && LT(v, data[j - 1])) {
                data[j] = data[j - 1];
                j--;
            }
            data[j] = v;
            moves += i - j + 2;
        }
    }
    if (m && moves) m->element_moves += moves;
    return 1;
}

/* small_sorts.py:118-131 */
static int64_t FN(sift_down)(T *data, int64_t begin, int64_t root, int64_t size, oracle_metrics *m) {
    int64_t swaps = 0;
    for (;;) {
        int64_t child = 2 * root + 1;
        if (child >= size) break;
        if (child + 1 < size && LT(data[begin + child], data[begin + child + 1])) child++;
        if (!LT(data[begin + root], data[begin + child])) break;
        SWAP(data[begin + root], data[begin + child]);
        swaps++;
        root = child;
    }
    return swaps;
}

/* small_sorts.py:134-154 */
void FN(oracle_heapsort)(T *data, int64_t begin, int64_t end, oracle_metrics *m) {
    int64_t n = end - begin;
    if (n < 2) return;
    int64_t swaps = 0;
    for (int64_t root = n / 2 - 1; root >= 0; root--) swaps += FN(sift_down)(data, begin, root, n, m);
    for (int64_t size = n - 1; size > 0; size--) {
        SWAP(data[begin], data[begin + size]);
        swaps += 1 + FN(sift_down)(data, begin, 0, size, m);
    }
    if (m) m->exchanges += swaps;
}

/* small_sorts.py:157-181 */
void FN(oracle_sort3)(T *data, int64_t a, int64_t b, int64_t c, oracle_metrics *m) {
    int64_t swaps = 0;
    if (LT(data[b], data[a])) { SWAP(data[a], data[b]); swaps++; }
    if (LT(data[c], data[b])) {
        SWAP(data[b], data[c]);
        swaps++;
        if (LT(data[b], data[a])) { SWAP(data[a], data[b]); swaps++; }
    }
    if (m && swaps) m->exchanges += swaps;
}

/* partition.py:69-125 (Hoare crossing pointers, equals go right) */
oracle_partition_result FN(oracle_partition_right)(T *data, int64_t begin, int64_t end,
                                                   oracle_metrics *m) {
    T pivot = data[begin];
    int64_t i = begin + 1;
    while (LT(data[i], pivot)) i++;
    int64_t j = end;
    if (i - 1 == begin) {
        while (i < j) {
            j--;
            if (LT(data[j], pivot)) break;
        }
    } else {
        j--;
        while (!LT(data[j], pivot)) j--;
    }
    int no_swaps = i >= j;
    int64_t swaps = 0;
    while (i < j) {
        SWAP(data[i], data[j]);
        swaps++;
        i++;
        while (LT(data[i], pivot)) i++;
        j--;
        while (!LT(data[j], pivot)) j--;
    }
    int64_t pivot_pos = i - 1;
    data[begin] = data[pivot_pos];
    data[pivot_pos] = pivot;
    if (m) {
        m->partition_right_calls++;
        m->exchanges += swaps;
        m->element_moves += 2;
    }
    oracle_partition_result r = {pivot_pos - begin, no_swaps};
    return r;
}

/* partition.py:128-181 (equals go left; caller guarantees pred == pivot) */
oracle_partition_result FN(oracle_partition_left)(T *data, int64_t begin, int64_t end,
                                                  oracle_metrics *m) {
    T pivot = data[begin];
    int64_t j = end - 1;
    while (LT(pivot, data[j])) j--;
    int64_t i = begin;
    if (j + 1 == end) {
        while (i < j) {
            i++;
            if (LT(pivot, data[i])) break;
        }
    } else {
        i++;
        while (!LT(pivot, data[i])) i++;
    }
    int64_t swaps = 0;
    while (i < j) {
        SWAP(data[i], data[j]);
        swaps++;
        j--;
        while (LT(pivot, data[j])) j--;
        i++;
        while (!LT(pivot, data[i])) i++;
    }
    int64_t pivot_pos = j;
    data[begin] = data[pivot_pos];
    data[pivot_pos] = pivot;
    if (m) {
        m->partition_left_calls++;
        m->exchanges += swaps;
        m->element_moves += 2;
    }
    oracle_partition_result r = {pivot_pos - begin, 0};
    return r;
}

/* partition.py:184-301 (branch-free block partition; BlockBuffers :44-66) */
oracle_partition_result FN(oracle_block_partition_right)(T *data, int64_t begin, int64_t end,
                                                         int64_t block, oracle_metrics *m) {
    int64_t *offs_l = (int64_t *)malloc(sizeof(int64_t) * (size_t)block);
    int64_t *offs_r = (int64_t *)malloc(sizeof(int64_t) * (size_t)block);
    T pivot = data[begin];
    int64_t first = begin + 1, last = end;
    int64_t num_l = 0, num_r = 0, start_l = 0, start_r = 0;
    int64_t base_l = first, base_r = last;
    int64_t swaps = 0, moves = 0;
    while (first < last) {
        int64_t unknown = last - first, take_l, take_r;
        if (num_l == 0) {
            if (num_r == 0) {
                take_l = block < unknown / 2 ? block : unknown / 2;
                take_r = block < unknown - take_l ? block : unknown - take_l;
            } else {
                take_l = block < unknown ? block : unknown;
                take_r = 0;
            }
        } else {
            take_l = 0;
            take_r = block < unknown ? block : unknown;
        }
        if (take_l) {
            base_l = first;
            start_l = 0;
            for (int64_t k = 0; k < take_l; k++) {
                offs_l[num_l] = k;
                num_l += !LT(data[first + k], pivot);
            }
            first += take_l;
        }
        if (take_r) {
            base_r = last;
            start_r = 0;
            for (int64_t k = 0; k < take_r; k++) {
                offs_r[num_r] = k + 1;
                num_r += LT(data[last - 1 - k], pivot);
            }
            last -= take_r;
        }
        int64_t num = num_l < num_r ? num_l : num_r;
        if (num) {
            for (int64_t k = 0; k < num; k++) {
                int64_t a = base_l + offs_l[start_l + k];
                int64_t b = base_r - offs_r[start_r + k];
                SWAP(data[a], data[b]);
            }
            swaps += num;
            num_l -= num;
            num_r -= num;
            start_l += num;
            start_r += num;
        }
    }
    if (num_l) {
        while (num_l) {
            num_l--;
            int64_t a = base_l + offs_l[start_l + num_l];
            last--;
            if (a != last) {
                SWAP(data[a], data[last]);
                swaps++;
            }
        }
        first = last;
    } else if (num_r) {
        while (num_r) {
            num_r--;
            int64_t b = base_r - offs_r[start_r + num_r];
            if (b != first) {
                SWAP(data[b], data[first]);
                swaps++;
            }
            first++;
        }
        last = first;
    }
    int64_t pivot_pos = first - 1;
    data[begin] = data[pivot_pos];
    data[pivot_pos] = pivot;
    free(offs_l);
    free(offs_r);
    if (m) {
        m->partition_right_calls++;
        m->exchanges += swaps;
        m->element_moves += moves + 2;
    }
    oracle_partition_result r = {pivot_pos - begin, swaps == 0};
    return r;
}

/* driver.py:81-113 */
void FN(oracle_choose_pivot)(T *data, int64_t begin, int64_t end, const oracle_config *cfg,
                             oracle_metrics *m) {
    int64_t size = end - begin;
    int64_t mid = begin + size / 2;
    if (size > cfg->ninther_threshold) {
        FN(oracle_sort3)(data, begin, mid, end - 1, m);
        FN(oracle_sort3)(data, begin + 1, mid - 1, end - 2, m);
        FN(oracle_sort3)(data, begin + 2, mid + 1, end - 3, m);
        FN(oracle_sort3)(data, mid - 1, mid, mid + 1, m);
        SWAP(data[begin], data[mid]);
        if (m) m->exchanges += 1;
    } else {
        FN(oracle_sort3)(data, mid, begin, end - 1, m);
    }
}

/* driver.py:127-156 (asserts size >= MIN_BREAK_SIZE, :145) */
void FN(oracle_break_patterns)(T *data, int64_t begin, int64_t end, const oracle_config *cfg,
                               oracle_metrics *m) {
    int64_t size = end - begin;
    int64_t q = size / 4, pairs = 1;
    SWAP(data[begin], data[begin + q]);
    SWAP(data[end - 1], data[end - 1 - q]);
    if (size > cfg->ninther_threshold) {
        for (int64_t k = 1; k <= 2; k++) {
            SWAP(data[begin + k], data[begin + q + k]);
            SWAP(data[end - 1 - k], data[end - 1 - q - k]);
        }
        pairs = 3;
    }
    if (m) m->exchanges += 2 * pairs;
}

typedef struct {
    T *data;
    const oracle_config *cfg;
    int use_block;
    oracle_metrics *m;
} FN(sort_ctx);

static int FN(attempt_partial)(FN(sort_ctx) *c, int64_t lo, int64_t hi) {
    oracle_metrics *m = c->m;
    if (m) m->partial_insertion_attempts++;
    int ok = FN(oracle_partial_insertion_sort)(c->data, lo, hi, c->cfg->partial_insertion_budget, m);
    if (!ok && m) m->partial_insertion_aborts++;
    return ok;
}

/* driver.py:198-260 — the pdqsort loop; recurse on the smaller side. */
static void FN(loop)(FN(sort_ctx) *c, int64_t begin, int64_t end, int64_t bad_allowed, int leftmost,
                     int64_t depth) {
    T *data = c->data;
    const oracle_config *cfg = c->cfg;
    oracle_metrics *m = c->m;
    if (m && depth > m->max_depth) m->max_depth = depth;
    for (;;) {
        int64_t size = end - begin;
        if (size < cfg->insertion_threshold) {
            if (leftmost) FN(oracle_insertion_sort)(data, begin, end, m);
            else FN(oracle_unguarded_insertion_sort)(data, begin, end, m);
            return;
        }
        if (bad_allowed == 0) {
            FN(oracle_heapsort)(data, begin, end, m);
            if (m) m->heapsort_fallbacks++;
            return;
        }
        FN(oracle_choose_pivot)(data, begin, end, cfg, m);
        if (cfg->use_partition_left && !leftmost && !LT(data[begin - 1], data[begin])) {
            oracle_partition_result res = FN(oracle_partition_left)(data, begin, end, m);
            begin = begin + res.pivot_index + 1;
            continue;
        }
        oracle_partition_result res =
            c->use_block ? FN(oracle_block_partition_right)(data, begin, end, cfg->block_size, m)
                         : FN(oracle_partition_right)(data, begin, end, m);
        int64_t pivot_pos = begin + res.pivot_index;
        int64_t left_size = pivot_pos - begin;
        int64_t right_size = end - (pivot_pos + 1);
        if (oracle_is_bad_partition(left_size, right_size, size, cfg)) {
            if (m) m->bad_partitions++;
            bad_allowed--;
            if (cfg->use_break_patterns) {
                if (left_size >= ORACLE_MIN_BREAK_SIZE)
                    FN(oracle_break_patterns)(data, begin, pivot_pos, cfg, m);
                if (right_size >= ORACLE_MIN_BREAK_SIZE)
                    FN(oracle_break_patterns)(data, pivot_pos + 1, end, cfg, m);
            }
        } else if (cfg->use_partial_insertion && res.no_swaps && FN(attempt_partial)(c, begin, pivot_pos) &&
                   FN(attempt_partial)(c, pivot_pos + 1, end)) {
            return;
        }
        if (left_size <= right_size) {
            FN(loop)(c, begin, pivot_pos, bad_allowed, leftmost, depth + 1);
            begin = pivot_pos + 1;
            leftmost = 0;
        } else {
            FN(loop)(c, pivot_pos + 1, end, bad_allowed, 0, depth + 1);
            end = pivot_pos;
        }
    }
}

/* driver.py:167-264 (_sort_range); budget = n.bit_length() - 1 (:262-263). */
void FN(oracle_sort_range)(T *data, int64_t begin, int64_t end, const oracle_config *cfg, int use_block,
                           oracle_metrics *m) {
    FN(sort_ctx) c = {data, cfg, use_block, m};
    int64_t n = end - begin;
    int64_t bad_allowed = n > 0 ? oracle_bit_length(n) - 1 : 0;
    FN(loop)(&c, begin, end, bad_allowed, 1, 0);
}

#undef LT
#undef SWAP
#undef FN
#undef CAT
#undef CAT_
