"""B200-native (sm_100a) EDL-Dist distillation hot path.

Drop-in device mirror of the reference's teacher inference, soft-label
reader and student step (edl.nnkit / edl.teacher_node / edl.student_node);
all compute goes through libedl_b200.so (see include/edl_b200.h).
"""

__version__ = "0.1.0"
